"""BASELINE config 4 (4M + 4M points, kappa = 64, m = 6) at full size:
  1. the GPU-built structure (k_setup.cu) against the host planner, by
     order-independent digests of trees, permutations, L+ (with directions), L-
     and D/D^ (3.47e9 admissible blocks are too many to export);
  2. y on 64 seeded rows against the dense sum (approximation error, sanity);
  3. counters vs SURVEY.md App. A.
Writes gpurun_out/cfg4_check.json.  Long: ~10 min on one B200 + host."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402

c = CONFIGS[4]
tg, sr, q = make_inputs(c)
res = {"config": 4}
t = time.time()
op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
res["gpu_setup_s"] = time.time() - t
st = op.stats()
res["counters"] = {k: st[k] for k in ("n_c", "n_sc", "m_d", "n_le", "n_lminus", "l_hf", "slots_t", "slots_s",
                                      "nodes_t", "nodes_s", "depth_t", "depth_s", "w_resident", "w_segments")}
gd = op.structure_digest()
t = time.time()
y = op.apply(q)
res["apply_s"] = time.time() - t
del op
rows = np.random.default_rng(44).choice(c.nt, 64, replace=False)
yd = oracle.dense_rows(tg, sr, q, c.kappa, rows)
res["rel_l2_vs_dense_64rows"] = oracle.rel_l2(y[rows], yd)
t = time.time()
hp = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, plan_only=True)
res["host_planner_s"] = time.time() - t
hd = hp.structure_digest()
res["digest_gpu"] = [f"{v:016x}" for v in gd]
res["digest_host"] = [f"{v:016x}" for v in hd]
res["structure_identical"] = gd == hd
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/cfg4_check.json", "w"), indent=1)
assert gd == hd
