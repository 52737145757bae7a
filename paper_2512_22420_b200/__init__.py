"""paper_2512_22420_b200 — B200-native batched speculative-decoding verification
(the data-parallel hot path of Nightjar, arXiv 2512.22420) behind the C ABI of
include/nj.h, plus Nightjar's host-side speculative-length bandit.

    from paper_2512_22420_b200 import Verifier, Bandit

The package holds only what the path needs: csrc/ (CUDA kernels for sm_100a +
the C ABI + the C++ bandit), the ctypes binding (_lib.py), the build script
(_build.py) and the multi-GPU driver (dist.py).  It never imports oracle/.
"""
from ._lib import (NJ_FLAG_CLAMP, NJ_FLAG_FALLBACK, NJ_FLAG_ZERO_MASS, NJ_OPT_CERTIFY, NJ_OPT_FORCE_FALLBACK,
                   NJ_OPT_PATH, NJ_OPT_PROFILE, NJ_OPT_Q_STAGE_ROWS, NJ_OPT_Q_ZERO_COPY, NJ_PATH_AUTO, NJ_PATH_FUSED, NJ_PATH_STAGED, NJ_PATH_TWOPASS, Bandit, NcclComm, NJError, ShardGroup, Verifier, load,
                   nccl_unique_id, shard_range)

__all__ = ["Verifier", "Bandit", "ShardGroup", "NcclComm", "nccl_unique_id", "shard_range", "NJError", "load", "NJ_PATH_AUTO", "NJ_PATH_FUSED", "NJ_PATH_TWOPASS", "NJ_PATH_STAGED",
           "NJ_OPT_PATH", "NJ_OPT_PROFILE", "NJ_OPT_Q_ZERO_COPY", "NJ_OPT_Q_STAGE_ROWS", "NJ_OPT_CERTIFY", "NJ_OPT_FORCE_FALLBACK", "NJ_FLAG_FALLBACK", "NJ_FLAG_ZERO_MASS",
           "NJ_FLAG_CLAMP"]
