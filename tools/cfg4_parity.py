"""BASELINE config 4 (4M + 4M points, kappa = 64, m = 6) at full size, y parity of
the int8 tcgen05 M2L path (coupling digits generated per apply in segments):
  1. against the CPU oracle on seeded target leaves (incl. the first and last):
     the sampled-structure oracle (orc_create_sampled) refines the partition only
     below the sampled leaves' ancestors and generates coupling matrices per
     block -- the full config-4 L+ (3.47e9 blocks) and coupling set (228 GB) do
     not fit in host memory; its rows are bitwise those of the full oracle
     (tests/test_oracle.py::test_sampled_structure_oracle_matches_full);
  2. with --dmma: the int8 path against the FP64 DMMA path on all 4M rows.
Writes gpurun_out/cfg4_parity.json.  ~10 min on one B200 + its host."""
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
args = (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)


def save():
    print(json.dumps(res), flush=True)
    json.dump(res, open(out, "w"), indent=1)


def run(impl):
    if impl == "dmma":
        os.environ["FDH_M2L_IMPL"] = "dmma"
    else:
        os.environ.pop("FDH_M2L_IMPL", None)
    t = time.time()
    op = F.DirectionalOperator(*args)
    setup = time.time() - t
    st = op.stats()
    t = time.time()
    y = op.apply(q)
    res[impl] = {"setup_s": setup, "apply_s": time.time() - t, "m2l_impl": st["m2l_impl"],
                 "w_resident": st["w_resident"], "w_segments": st["w_segments"]}
    del op
    return y


y8 = run("i8")
if "--dmma" in sys.argv:
    yd = run("dmma")
    res["int8_vs_dmma_all_rows"] = oracle.rel_l2(y8, yd)
save()
t = time.time()
probe = oracle.Oracle(*args, sample_leaves=[0])  # trees (canonical leaf order) for the leaf count
nl = probe.leaf_count(0)
del probe
leaves = np.unique(np.concatenate([[0, nl - 1], np.random.default_rng(4).choice(nl, int(os.environ.get("NSAMPLE", "4")),
                                                                                 replace=False)]))
o = oracle.Oracle(*args, sample_leaves=leaves)
res["oracle_setup_s"] = time.time() - t
t = time.time()
rows, ys = o.apply_sampled(q, leaves)
res["oracle_sampled_s"] = time.time() - t
res["oracle_threads"] = int(oracle.lib().orc_set_threads(0))
res["target_leaves"] = int(nl)
res["sampled_leaves"] = [int(v) for v in leaves]
res["sampled_rows"] = int(len(rows))
res["int8_vs_oracle_sampled"] = oracle.rel_l2(y8[rows], ys)
if "--dmma" in sys.argv:
    res["dmma_vs_oracle_sampled"] = oracle.rel_l2(yd[rows], ys)
save()
