#!/usr/bin/env python3
"""bench-cli on the B200 path: the PAPER.md section-4
experiment (Table 1) -- a uniform 8^k tensor grid in [-1,1]^3, P_T = P_S,
kappa = 0.1 * 2^k, n_max = 512, eta2 = 5, l_hf = k - 4, m = 4, zero diagonal --
or a point file, reported with Table 1's fields.

  python tools/bench_cli.py --k 6 [--kappa K] [--n-max 512] [--eta2 5] [--l-hf L]
        [--degree 4] [--no-zero-diagonal] [--seed 1] [--sample-rows 1024]
        [--points FILE] [--output FILE] [--format json|csv] [--config FILE]

Exit codes: 0 success, 2 configuration error, 1 runtime error.
Timings: t_s = setup (wall), t_ff = S2M + M2M + M2L + L2L + L2T, t_nf = near
field, t_tot = t_s + one apply (CUDA events, per-phase).  The sampled relative
error is against the dense sum on seeded rows (oracle/ dense rows, CPU).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# PAPER.md:673-677 (single core of a Xeon Gold 5218, ACA on)
PAPER_TABLE1 = {
    5: dict(t_tot=7.31, t_s=0.34, t_nf=6.94, t_ff=0.03, nf=24.41, N_SC=316, N_C=3096),
    6: dict(t_tot=76.25, t_s=1.20, t_nf=74.29, t_ff=0.76, nf=4.06, N_SC=1522, N_C=166320),
    7: dict(t_tot=702.72, t_s=3.71, t_nf=688.14, t_ff=10.87, nf=0.58, N_SC=4554, N_C=2640960),
    8: dict(t_tot=6060.16, t_s=15.24, t_nf=5907.66, t_ff=137.26, nf=0.077, N_SC=9824, N_C=33103296),
    9: dict(t_tot=50204.00, t_s=118.89, t_nf=48576.20, t_ff=1508.91, nf=0.010, N_SC=32036, N_C=344979432),
}


def parse_args(argv):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--config", help="flat key=value file with the same keys as the flags")
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--kappa", type=float)
    ap.add_argument("--n-max", type=int, default=512)
    ap.add_argument("--eta2", type=float, default=5.0)
    ap.add_argument("--l-hf", type=int)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--aca-eps", type=float)
    ap.add_argument("--no-zero-diagonal", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sample-rows", type=int, default=-1, help="default: min(1024, 4e9 / N)")
    ap.add_argument("--points", help="text file, one point 'x y z' per line (P_T = P_S)")
    ap.add_argument("--output")
    ap.add_argument("--format", choices=["json", "csv"], default="json")
    a = ap.parse_args(argv)
    if a.config:
        for line in open(a.config):
            line = line.split("#")[0].strip()
            if not line:
                continue
            key, val = (t.strip() for t in line.split("=", 1))
            key = key.replace("-", "_")
            if not hasattr(a, key):
                raise ValueError(f"unknown config key {key}")
            cur = getattr(a, key)
            setattr(a, key, type(cur)(val) if cur is not None and not isinstance(cur, bool) else
                    (val.lower() in ("1", "true", "yes") if isinstance(cur, bool) else float(val)))
    return a


def main(argv=None) -> int:
    try:
        a = parse_args(argv)
        if a.aca_eps is not None:
            raise ValueError("--aca-eps: ACA compression is lossy and outside this build's parity contract")
        if a.points is None and a.k < 3:
            raise ValueError("--k must be >= 3 (SPEC.md:584)")
        if a.degree < 0 or a.n_max < 1 or a.eta2 <= 0:
            raise ValueError("invalid degree / n_max / eta2")
    except (ValueError, SystemExit) as e:
        if isinstance(e, SystemExit) and e.code == 0:
            return 0
        print(f"config error: {e}", file=sys.stderr)
        return 2
    try:
        import oracle
        import paper_2004_14229_b200 as F
        from paper_2004_14229_b200.configs import grid_points

        if a.points:
            P = np.loadtxt(a.points, ndmin=2)
            pts = [np.ascontiguousarray(P[:, i]) for i in range(3)]
            lo = tuple(P.min(axis=0) - 1e-9)
            hi = tuple(P.max(axis=0))
        else:
            pts = grid_points(a.k)
            lo, hi = (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)
        n = len(pts[0])
        kappa = a.kappa if a.kappa is not None else 0.1 * 2 ** a.k
        lhf = a.l_hf if a.l_hf is not None else (a.k - 4 if not a.points else F.LHF_DEFAULT)
        zd = not a.no_zero_diagonal
        rng = np.random.default_rng(a.seed)
        v = (2 * rng.random(n) - 1) + 1j * (2 * rng.random(n) - 1)
        t0 = time.perf_counter()
        op = F.DirectionalOperator(pts, pts, lo, hi, kappa, a.n_max, a.degree, a.eta2, lhf, zero_diagonal=zd)
        t_s = time.perf_counter() - t0
        op.apply(v)  # warm-up
        op.set_timing(True)
        y = op.apply(v)
        st = op.stats()
        ph = st["phase_ms"]
        t_ff = (ph["s2m"] + ph["m2m"] + ph["m2l"] + ph["l2l"] + ph["l2t"]) / 1e3
        t_nf = ph["p2p"] / 1e3
        t_apply = st["apply_ms"] / 1e3
        ns_rows = a.sample_rows if a.sample_rows > 0 else int(max(16, min(1024, 4e9 / n)))
        rows = rng.choice(n, min(ns_rows, n), replace=False)
        yd = oracle.dense_rows(pts, pts, v, kappa, rows, zero_diagonal=int(zd))
        rep = {
            "k": a.k if not a.points else None, "N": n, "kappa": kappa, "n_max": a.n_max, "eta2": a.eta2,
            "l_hf": st["l_hf"], "degree": a.degree, "zero_diagonal": zd,
            "t_tot": t_s + t_apply, "t_s": t_s, "t_apply": t_apply, "t_nf": t_nf, "t_ff": t_ff,
            "nf_percent": st["nf_percent"], "N_SC": st["n_sc"], "N_C": st["n_c"], "N_LE": st["n_le"],
            "M_D": st["m_d"], "bytes_stored": st["bytes_stored"],
            "sampled_rel_error": oracle.rel_l2(y[rows], yd), "sample_rows": int(len(rows)),
            "hardware": "1x NVIDIA B200 (fdhelm-b200, M2L: " + ("int8 tcgen05 digit products" if st["m2l_impl"] == 1 else "FP64 DMMA") + ")", "no_aca": True,
        }
        if not a.points and a.k in PAPER_TABLE1:
            p = PAPER_TABLE1[a.k]
            rep["paper_single_core"] = p
            rep["speedup_vs_paper_apply"] = (p["t_nf"] + p["t_ff"]) / t_apply
        if a.format == "json":
            out = json.dumps(rep, indent=1)
        else:
            buf = io.StringIO()
            flat = {k: v for k, v in rep.items() if not isinstance(v, dict)}
            w = csv.DictWriter(buf, fieldnames=list(flat))
            w.writeheader()
            w.writerow(flat)
            out = buf.getvalue()
        if a.output:
            open(a.output, "w").write(out)
        print(out)
        return 0
    except Exception as e:  # runtime error
        print(f"runtime error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
