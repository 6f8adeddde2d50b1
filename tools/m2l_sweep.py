"""M2L variant sweep on one B200: for each workload and each setting of the
planner / kernel knobs (env vars read at operator creation), the M2L kernel time
(event-record nodes inside the graph replays), its algorithmic and issued int8
rates, and the apply time.  One JSON line per (workload, variant).

    python tools/m2l_sweep.py --work c4m6,cfg3,cfg5 --variants "TT16:;TT32:FDH_I8_TILE=32;TT32c48:FDH_I8_TILE=32,FDH_M2L_CHUNK_MB=48"

Workloads: cfgN (BASELINE config N at full size), c4m6 (config-3 points with
m = 6, kappa = 32: the config-4 kernel shape at a quarter of its size).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2004_14229_b200 as F  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402


def workload(name):
    if name == "c4m6":
        c = CONFIGS[3]
        tg, sr, q = make_inputs(c)
        return c, (tg, sr, c.root_lo, c.root_hi, 32.0, c.n_max, 6, c.eta2, c.l_hf), q
    c = CONFIGS[int(name[3:])]
    tg, sr, q = make_inputs(c)
    return c, (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf), q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--work", default="c4m6")
    ap.add_argument("--variants", default="TT16:;TT32:FDH_I8_TILE=32")
    ap.add_argument("--applies", type=int, default=3)
    a = ap.parse_args()
    tops = F.tensor_peak_tops(0)
    for w in a.work.split(","):
        c, args, q = workload(w)
        n = (args[6] + 1) ** 3
        for var in a.variants.split(";"):
            name, _, envs = var.partition(":")
            saved = {}
            for kv in filter(None, envs.split(",")):
                k, v = kv.split("=")
                saved[k] = os.environ.get(k)
                os.environ[k] = v
            try:
                t = time.perf_counter()
                op = F.DirectionalOperator(*args)
                if os.environ.get("FDH_CACHE_NF") == "1":
                    op.set_cache(True)  # cached near-field kernel values (fdh_set_cache)
                if os.environ.get("FDH_ACA_EPS"):
                    op.set_aca(float(os.environ["FDH_ACA_EPS"]))  # ACA-compressed coupling (lossy)
                setup = time.perf_counter() - t
                op.apply(q)  # warm-up (graph capture)
                op.set_timing(True)
                for _ in range(a.applies):
                    op.apply(q)
                st = op.stats()
                ks = int(st["m2l_i8_digits"])
                alg = st["m2l_i8_products"] * 8.0 * n * n * st["n_c"]
                ms = st["m2l_gemm_ms"]
                print(json.dumps({"work": w, "variant": name, "env": envs, "setup_s": round(setup, 2),
                                  "apply_ms": st["apply_ms_sum"] / max(1, st["applies_collected"]), "m2l_ms": ms,
                                  "alg_tops": alg / ms / 1e9, "frac": alg / ms / 1e9 / tops,
                                  "issued_tops": st["m2l_i8_ops"] / ms / 1e9, "useful": alg / st["m2l_i8_ops"],
                                  "tiles": st["m2l_tiles"], "items": st["m2l_items"], "w_resident": st["w_resident"],
                                  "phases": {k: round(v, 3) for k, v in st["phase_ms"].items()},
                                  "peak_tops": tops, "digits": f"{ks}x{st['m2l_i8_bits']}"}), flush=True)
                del op
            except Exception as e:
                print(json.dumps({"work": w, "variant": name, "error": str(e)}), flush=True)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main()
