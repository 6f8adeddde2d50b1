"""Digit-format A/B of the int8 M2L: one process per library build (FDHELM_LIB) and
config; prints the M2L kernel time and y's relative l2 error against the committed
oracle rows (tests/golden/yrows_cfg{3,4,5}.npz), overall and the worst 64-row group.

    FDHELM_LIB=variants/lib77.so python tools/digits_ab.py --config 3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--applies", type=int, default=2)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    tg, sr, q = make_inputs(c)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap)
    y = op.apply(q)
    op.set_timing(True)
    for _ in range(a.applies):
        y = op.apply(q)
    st = op.stats()
    z = np.load(os.path.join(ROOT, "tests", "golden", f"yrows_cfg{a.config}.npz"))
    err = rel_l2(y[z["rows"]], z["y"])
    worst = max(rel_l2(y[z["rows"][i:i + 64]], z["y"][i:i + 64]) for i in range(0, len(z["rows"]), 64))
    print(json.dumps({"lib": os.environ.get("FDHELM_LIB", "default"), "cfg": a.config,
                      "digits": f"{st['m2l_i8_digits']}x{st['m2l_i8_bits']}p{st['m2l_i8_products']}", "m2l_ms": st["m2l_gemm_ms"],
                      "apply_ms": st["apply_ms_sum"] / max(1, st["applies_collected"]), "items": st["m2l_items"],
                      "tiles": st["m2l_tiles"], "err": err, "worst_group": worst, "setup_s": st["setup_ms"] / 1e3,
                      "phases": {k: round(v, 2) for k, v in st["phase_ms"].items()}}), flush=True)


if __name__ == "__main__":
    main()
