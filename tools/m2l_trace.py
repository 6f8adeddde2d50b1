"""Per-phase cycle breakdown of k_m2l_gemm (debug build with -DFDH_M2L_TRACE=1).

  FDHELM_LIB=variants/lib_tr.so python tools/m2l_trace.py [--config 2]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
tg, sr, q = make_inputs(c)
op = F.DirectionalOperator(tg, sr, c.root_lo if hasattr(c, "root_lo") else (0, 0, 0), c.root_hi, c.kappa, c.n_max,
                           c.m, c.eta2, c.l_hf)
lib = ctypes.CDLL(os.environ["FDHELM_LIB"])
buf = (ctypes.c_ulonglong * 8)()
op.apply(q)
lib.fdh_debug_m2l_trace(buf, 1)
op.apply(q)
lib.fdh_debug_m2l_trace(buf, 0)
v = np.array(list(buf), dtype=np.float64)
names = ["wait+barrier(top)", "flush", "dmma key loop", "barrier(end)", "stage issue"]
tot = v[5]
print(f"items {int(v[7])} keys {int(v[6])}  loop cycles/CTA-warp0 total {tot:.3e}")
for i, n in enumerate(names):
    print(f"  {n:20s} {v[i] / tot * 100:6.2f} %   {v[i] / v[6]:9.0f} cyc/key")
