"""Multiple right-hand sides: throughput of
fdh_create_multi / fdh_apply_device with R vectors per apply on a BASELINE config,
R = 1, 2, 4, 8, 16.  One JSON line per R: device time per batch (CUDA events on
the operator's stream, L2 flushed between batches outside the events), time per
vector, (N_T + N_S) * R / s, per-phase times, and the e2e host path
(fdh_apply_multi with the H2D / D2H copies inside).

    python tools/bench_multi.py [--config 2] [--rhs 1,2,4,8,16] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import ClockSampler  # noqa: E402
from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402


def main():
    import torch

    import paper_2004_14229_b200 as F

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--rhs", default="1,2,4,8,16")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    tg, sr, _ = make_inputs(c)
    rng = np.random.default_rng(1000 * args.config + 3)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    base = None
    for R in [int(v) for v in args.rhs.split(",")]:
        X = rng.uniform(-1, 1, (R, c.ns)) + 1j * rng.uniform(-1, 1, (R, c.ns))
        t0 = time.perf_counter()
        op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap,
                                   c.zero_diagonal, nrhs=R)
        setup_s = time.perf_counter() - t0
        stream = torch.cuda.ExternalStream(op.stream(), device=dev)
        x = torch.from_numpy(X.view(np.float64).reshape(-1)).to(dev)
        y = torch.empty(2 * R * c.nt, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            op.apply_device(x.data_ptr(), y.data_ptr(), op.stream())
        torch.cuda.synchronize()
        op.set_timing(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(0) as clk:
            for i in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                    evs[i][0].record(stream)
                op.apply_device(x.data_ptr(), y.data_ptr(), op.stream())
                evs[i][1].record(stream)
            torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        st = op.stats()
        op.set_timing(False)
        # e2e: host buffers, copies inside (fdh_apply_multi)
        Y = np.empty((R, c.nt), dtype=np.complex128)
        op.apply_multi(X, out=Y)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            op.apply_multi(X, out=Y)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        per_vec = ms / R
        if base is None:
            base = per_vec
        line = {
            "metric": "directional-FMM matvec, R right-hand sides per apply: (N_T+N_S)*R/s", "nrhs": R,
            "config": args.config, "ms_per_batch": ms, "ms_per_vector": per_vec,
            "value": R * (c.nt + c.ns) / (ms / 1e3), "unit": "points/s",
            "speedup_per_vector_vs_R1": base / per_vec,
            "phases_ms": st["phase_ms"], "m2l_gemm_ms": st["m2l_gemm_ms"],
            "m2l_impl": st["m2l_impl"], "m2l_tiles": st["m2l_tiles"], "m2l_items": st["m2l_items"],
            "m2l_i8_ops": st["m2l_i8_ops"], "gpu_launches": st["gpu_launches"], "setup_s": setup_s,
            "e2e": {"ms_per_batch": e2e_ms, "value": R * (c.nt + c.ns) / (e2e_ms / 1e3), "unit": "points/s",
                    "h2d_bytes_per_step": 16 * R * c.ns, "d2h_bytes_per_step": 16 * R * c.nt,
                    "path": "fdh_apply_multi (C-ABI) with host buffers, wall clock"},
            "clocks": clk.summary(), "l2": "flushed between batches (256 MB write, outside the events)",
        }
        print(json.dumps(line), flush=True)
        del op


if __name__ == "__main__":
    main()
