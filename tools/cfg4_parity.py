"""BASELINE config 4 (4M + 4M points, kappa = 64, m = 6) at full size, y parity of
the int8 tcgen05 M2L path (coupling digits generated per apply in segments):
  1. int8 path vs the FP64 DMMA path on all 4M rows (relative l2);
  2. both against the sampled-target CPU oracle (full trees / lists / upward
     pass, M2L-L2L-L2T-P2P for seeded target leaves incl. the first and last);
Writes gpurun_out/cfg4_parity.json.  Long: ~15 min on one B200 + its host."""
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
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "cfg4_parity.json")


def run(impl):
    if impl == "dmma":
        os.environ["FDH_M2L_IMPL"] = "dmma"
    else:
        os.environ.pop("FDH_M2L_IMPL", None)
    t = time.time()
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    setup = time.time() - t
    st = op.stats()
    t = time.time()
    y = op.apply(q)
    res[impl] = {"setup_s": setup, "apply_s": time.time() - t, "m2l_impl": st["m2l_impl"],
                 "w_resident": st["w_resident"], "w_segments": st["w_segments"]}
    del op
    return y


y8 = run("i8")
yd = run("dmma")
res["int8_vs_dmma_all_rows"] = oracle.rel_l2(y8, yd)
print(json.dumps(res), flush=True)
json.dump(res, open(out, "w"), indent=1)
mem_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
res["host_mem_gb"] = mem_gb
if mem_gb < 600:  # the oracle holds all 3.47e9 L+ blocks (~140 GB peak)
    res["oracle"] = "skipped: host memory too small"
    json.dump(res, open(out, "w"), indent=1)
    sys.exit(0)
t = time.time()
o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
res["oracle_setup_s"] = time.time() - t
nl = o.leaf_count(0)
leaves = np.unique(np.concatenate([[0, nl - 1], np.random.default_rng(4).choice(nl, 2, replace=False)]))
t = time.time()
rows, ys = o.apply_sampled(q, leaves)
res["oracle_sampled_s"] = time.time() - t
res["sampled_leaves"] = [int(v) for v in leaves]
res["sampled_rows"] = int(len(rows))
res["int8_vs_oracle_sampled"] = oracle.rel_l2(y8[rows], ys)
res["dmma_vs_oracle_sampled"] = oracle.rel_l2(yd[rows], ys)
print(json.dumps(res), flush=True)
json.dump(res, open(out, "w"), indent=1)
