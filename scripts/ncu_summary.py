"""Key metrics of every kernel in an ncu --set full report, as JSON.
Usage: python scripts/ncu_summary.py rep.ncu-rep out.json [note]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes_read.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__sass_inst_executed_op_tmem_ldt.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "launch__shared_mem_per_block_dynamic", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = {"report": sys.argv[1], "note": sys.argv[3] if len(sys.argv) > 3 else "", "kernels": []}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    k = {"name": d.get("Kernel Name", "")[:120]}
    for key in KEYS:
        if key in d:
            k[key] = f"{d[key]} {u.get(key, '')}".strip()
    out["kernels"].append(k)
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k in out["kernels"]:
    print(json.dumps(k))
