import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    # gpu tests must never silently pass on a CPU box
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Per-test parity tie counts (R12: near ties are counted and
    reported): every GPU parity comparison records how many requests the
    oracle flagged as ties, the expected count, how many were excused and how
    many of those took the other tie branch."""
    import sys
    parity = sys.modules.get("parity")   # tests/parity.py as the test modules imported it
    if parity is None:
        return
    stats = parity.STATS
    if not stats:
        return
    tr = terminalreporter
    tr.write_sep("-", "parity tie counts (oracle band 1e-6)")
    tot = {"B": 0, "ties": 0, "excused": 0, "excused_differing": 0, "fallback": 0}
    exp, n_unknown = 0.0, 0
    for s in stats:
        tr.write_line(f"{s['test']:<60} B={s['B']:<5} N={s['N']:<5} ties={s['ties']} (acc {s['accept_ties']}, "
                      f"draw {s['draw_ties']}) expected={s['expected_ties']} excused={s['excused']} "
                      f"other-branch={s['excused_differing']} fallback={s['fallback']}")
        for k in tot:
            tot[k] += s[k]
        if s["expected_ties"] == s["expected_ties"]:   # the stage-isolated tests carry no tie probability (NaN)
            exp += s["expected_ties"]
        else:
            n_unknown += s["B"]
    tr.write_line(f"TOTAL requests={tot['B']} ties={tot['ties']} expected={exp:.2f} (over the "
                  f"{tot['B'] - n_unknown} requests with a tie probability) excused={tot['excused']} "
                  f"other-branch={tot['excused_differing']} fallback={tot['fallback']}")
