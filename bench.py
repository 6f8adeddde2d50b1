#!/usr/bin/env python3
"""Benchmark of the directional Helmholtz matvec (BASELINE.json metric:
"directional-FMM matvec time & (N_T+N_S)/s at 1/2/4/8 B200; % FP64 roofline").

A step = one apply y = A x of the configured workload (default: BASELINE config
2, N_T = N_S = 100,000, kappa = 16, m = 4, the config the metric is quoted on
that fits one GPU).  Setup (trees, partition, coupling matrices) is outside the
timed region, as t_s in PAPER.md Table 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Under torchrun (N > 1) every rank owns a cost-balanced Morton range of target
leaves (fdh_create_shard) and the step ends with an NCCL all-reduce of y.
`--impl reference` times the CPU restatement of the reference algorithm
(oracle/, OpenMP, all host cores) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2004_14229_b200.configs import CONFIGS, make_inputs  # noqa: E402

METRIC = "directional-FMM matvec (N_T+N_S)/s"
UNIT = "points/s"
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "m2l_traffic.json")


def workload_desc(c):
    return (f"BASELINE config {c.cfg}: N_T={c.nt}, N_S={c.ns}, kappa={c.kappa:g}, degree m={c.m} "
            f"({(c.m + 1) ** 3} nodes/box), n_max={c.n_max}, eta2={c.eta2:g}, default directions, "
            f"root {c.root_lo}-{c.root_hi}{', Gaussian-mixture sources' if c.mixture_sources else ''}")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_oracle(c, tg, sr):
    import oracle

    return oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap,
                         c.zero_diagonal)


def cpu_oracle_sample(c, tg, sr, q, target_s=12.0, o=None, seed=7, single_core=True):
    """The CPU restatement (oracle/) on a bounded sample: full upward pass plus
    M2L/L2L/L2T/P2P for a seeded sample of target leaves; the full-apply time is
    extrapolated linearly in the number of target leaves."""
    import oracle

    cores = oracle.lib().orc_set_threads(0)
    if o is None:
        o = build_oracle(c, tg, sr)
    nl = o.leaf_count(0)
    rng = np.random.default_rng(seed)
    t = time.perf_counter()
    o.apply_sampled(q, np.zeros(0, dtype=np.int64))
    t0 = time.perf_counter() - t
    k = min(nl, 16)
    t = time.perf_counter()
    o.apply_sampled(q, rng.choice(nl, k, replace=False))
    tk = time.perf_counter() - t
    per_leaf = max((tk - t0) / k, 1e-9)
    k2 = int(min(nl, max(k, (target_s - t0) / per_leaf)))
    t = time.perf_counter()
    o.apply_sampled(q, rng.choice(nl, k2, replace=False))
    tk2 = time.perf_counter() - t
    t_full = t0 + (tk2 - t0) * nl / k2
    # the same restatement on ONE core (nproc cores and 1 core), a
    # smaller leaf sample (~1/4 of the budget), extrapolated the same way
    if not single_core:
        return {"value": (c.nt + c.ns) / t_full, "unit": UNIT, "cores": int(cores), "kind": "port",
                "sample": (f"oracle/ (CPU restatement, OpenMP {cores} threads): full S2M+M2M, then M2L/L2L/L2T/P2P "
                           f"for {k2} of {nl} seeded target leaves in {tk2:.2f} s; full apply extrapolated to "
                           f"{t_full:.2f} s (linear in target leaves; upward pass {t0:.2f} s)"),
                "seconds_measured": tk2, "apply_s_extrapolated": t_full}
    L = oracle.lib()
    L.orc_set_threads(1)
    try:
        t = time.perf_counter()
        o.apply_sampled(q, np.zeros(0, dtype=np.int64))
        s0 = time.perf_counter() - t
        k1 = int(min(nl, max(2, (target_s / 4 - s0) / max(per_leaf * cores, 1e-9))))
        t = time.perf_counter()
        o.apply_sampled(q, rng.choice(nl, k1, replace=False))
        sk = time.perf_counter() - t
    finally:
        L.orc_set_threads(int(cores))
    t1 = s0 + (sk - s0) * nl / k1
    single = {"value": (c.nt + c.ns) / t1, "unit": UNIT, "cores": 1, "apply_s_extrapolated": t1,
              "sample": f"same restatement, 1 thread: {k1} of {nl} target leaves in {sk:.2f} s (upward pass {s0:.2f} s)"}
    return {
        "value": (c.nt + c.ns) / t_full,
        "unit": UNIT,
        "cores": int(cores),
        "kind": "port",
        "sample": (f"oracle/ (CPU restatement, OpenMP {cores} threads): full S2M+M2M, then M2L/L2L/L2T/P2P for "
                   f"{k2} of {nl} seeded target leaves in {tk2:.2f} s; full apply extrapolated to {t_full:.2f} s "
                   f"(linear in target leaves; upward pass {t0:.2f} s)"),
        "seconds_measured": tk2,
        "apply_s_extrapolated": t_full,
        "single_core": single,
    }


def roofline_block(st, c, m2l_flops, achieved, peak, gemm_ms, ms_per_step, traffic):
    """Roofline of the M2L kernel: the int8 tcgen05 digit GEMM (k_m2l_i8) against
    the measured int8 tensor peak, or the FP64 DMMA GEMM against the FP64 peak."""
    share = gemm_ms / ms_per_step if ms_per_step else None
    fp64 = {"achieved_tflops": achieved, "fp64_peak_tflops": peak,
            "ratio": (achieved / peak) if (achieved and peak) else None,
            "note": "algorithmic FP64 flop (8 n^2 per admissible block) per second of the M2L kernel, against the "
                    "measured FP64 DMMA peak"}
    if st["m2l_impl"] == 1:
        import paper_2004_14229_b200 as F
        tops = F.tensor_peak_tops(0)
        # algorithmic int8 work: the 28 digit-pair products (i + j <= 6 of 7 digits) of every
        # real MAC of the complex product (4 n^2 per block, 2 ops per MAC)
        alg = 28.0 * m2l_flops
        ach = alg / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        iss = st["m2l_i8_ops"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        return {"bound": "tensor", "kernel": "k_m2l_i8 (tcgen05.mma kind::i8, exact 7-digit fixed-point products, "
                                            "TMEM int32 level accumulators)",
                "achieved": ach, "peak": tops, "unit": "TOPS", "frac": (ach / tops) if (ach and tops) else None,
                "traffic": traffic,
                "peak_source": "measured live: fdh_tensor_peak_tops(0) int8 tcgen05 microbenchmark, M=128 N=256 "
                               "(MEASURED_PEAKS.json has no int8 entry; its bf16 burst 1625.8 TF/s x 2 = 3252 for "
                               "comparison)",
                "algorithmic": f"28 digit products x 8 n^2 ops per admissible block x N_C={st['n_c']} = {alg:.4g} "
                               f"int8 ops per launch",
                "issued_ops": st["m2l_i8_ops"], "issued_frac": (iss / tops) if (iss and tops) else None,
                "issued_note": "int8 ops the kernel issues: every target column of a tile for every key of the tile "
                               "(absent columns are zero), rows padded to 128, K to 2 x 16k",
                "fp64_equivalent": fp64, "gemm_ms": gemm_ms, "share_of_step": share}
    return {"bound": "tensor", "kernel": "k_m2l_gemm (FP64 DMMA mma.sync.m8n8k4)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
            "peak_source": "measured live: fdh_fp64_peak_tflops(0) DMMA microbenchmark (no FP64 entry in "
                           "MEASURED_PEAKS.json)",
            "algorithmic": f"8 n^2 flop per admissible block x N_C={st['n_c']} = {m2l_flops:.4g} flop per "
                           f"launch (SURVEY.md 8(d); the count holds for a 3M complex product)",
            "issued_flop": st["m2l_flops_executed"],
            "issued_frac": (st["m2l_flops_executed"] / (gemm_ms * 1e-3) / 1e12 / peak
                            if (gemm_ms > 0 and peak) else None),
            "issued_note": "flop the kernel issues on DMMA: Gauss 3-multiplication product (6 n^2) for "
                           "8-target n-tiles, 8 n^2 real GEMM for <= 4, incl. padding columns",
            "gemm_ms": gemm_ms, "share_of_step": share}


def hbm_passes(st, ph):
    """S2M / M2M / L2L / L2T against the measured HBM copy bandwidth (MEASURED_PEAKS.json
    hbm_gbs): algorithmic bytes of SURVEY.md 8(d) (fdh_stats.hbm_bytes) / phase time."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "fallback: nominal B200 HBM3e (MEASURED_PEAKS.json absent)"
    out = {"peak_gbs": peak, "peak_source": src,
           "note": "< 1 % of the step; per (box, direction) work items of 15-60 points are latency / FP64-bound "
                   "(sincos, Lagrange cardinals per point), not bandwidth-bound, at these sizes"}
    for k in ("s2m", "m2m", "l2l", "l2t"):
        b, ms = st["hbm_bytes"][k], ph.get(k, 0.0)
        gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[k] = {"bytes": b, "ms": ms, "achieved_gbs": gbs, "frac": gbs / peak if gbs else None}
    return out


def run_reference(args, c, rank, world):
    """--impl reference: the reference algorithm on the host cores (oracle port)."""
    if rank != 0:
        return
    tg, sr, q = make_inputs(c)
    steps = []
    cb = None
    o = build_oracle(c, tg, sr)
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(c, tg, sr, q, target_s=args.ref_seconds, o=o, seed=7 + i, single_core=False)
        if i >= args.warmup:
            steps.append(r["apply_s_extrapolated"])
            cb = r
    t = float(np.mean(steps))
    value = (c.nt + c.ns) / t
    cb = dict(cb)
    cb["value"] = value
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": {"workload": workload_desc(c), "cfg": c.cfg, "parallelism": "cpu-openmp"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_ours(args, c, rank, world, local_rank):
    import torch

    import paper_2004_14229_b200 as F

    dist = None
    if world > 1:
        import torch.distributed as dist

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    tg, sr, q = make_inputs(c)
    t_setup = time.perf_counter()
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap,
                               c.zero_diagonal, rank=rank, world=world)
    setup_s = time.perf_counter() - t_setup
    st0 = op.stats()
    stream = torch.cuda.ExternalStream(op.stream(), device=dev)
    x = torch.from_numpy(q.view(np.float64)).to(dev)
    y = torch.empty(2 * c.nt, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    torch.cuda.synchronize()  # x / y are produced on torch's stream, consumed on the operator's

    def step():
        op.apply_device(x.data_ptr(), y.data_ptr(), op.stream())
        if world > 1:
            with torch.cuda.stream(stream):
                dist.all_reduce(y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    op.set_timing(True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    st = op.stats()
    op.set_timing(False)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = args.steps * (c.nt + c.ns) / (total_ms / 1e3)

    # ---- e2e: host buffers (pinned), copies inside the timed region.  N = 1: the
    # C-ABI host call fdh_apply; N > 1: H2D + fdh_apply_device + NCCL all-reduce
    # of the rank partials + D2H, all on the operator's stream.
    xh_t = torch.from_numpy(q.copy()).pin_memory()
    yh_t = torch.empty(c.nt, dtype=torch.complex128).pin_memory()
    xh, yh = xh_t.numpy(), yh_t.numpy()

    def e2e_step():
        if world == 1:
            op.apply(xh, out=yh)
        else:
            with torch.cuda.stream(stream):
                x.copy_(xh_t.view(torch.float64), non_blocking=True)
            op.apply_device(x.data_ptr(), y.data_ptr(), op.stream())
            with torch.cuda.stream(stream):
                dist.all_reduce(y)
                yh_t.view(torch.float64).copy_(y, non_blocking=True)
            stream.synchronize()

    e2e_step()  # warm the host path (pinned buffers, copy engines)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_s.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e_e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e_s.elapsed_time(e_e)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        dist.barrier()
    e2e_value = args.steps * (c.nt + c.ns) / (e2e_ms / 1e3)

    if rank != 0:
        return
    # ---- roofline of the dominant kernel (the M2L GEMM)
    peak = F.fp64_peak_tflops(0)
    n = (c.m + 1) ** 3
    m2l_flops = 8.0 * n * n * st["n_c"]  # algorithmic
    gemm_ms = st["m2l_gemm_ms"]
    achieved = m2l_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    traffic = None
    if os.path.exists(PROFILE_TRAFFIC):
        try:
            tr = json.load(open(PROFILE_TRAFFIC))
            traffic = tr.get(f"cfg{c.cfg}{'_i8' if st['m2l_impl'] == 1 else ''}")
        except Exception:
            traffic = None
    ph = st["phase_ms"]
    p2p_ms = ph.get("p2p", 0.0)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("complex128 (f64; M2L as exact int8 x int8 -> int32 digit products of 49-bit fixed-point operands "
                  "on tcgen05)" if st["m2l_impl"] == 1 else "complex128 (f64)"),
        "data": "synthetic (seeded uniform / Gaussian-mixture points, U(-1,1) complex charges; SURVEY.md 8(d))",
        "config": {"workload": workload_desc(c), "cfg": c.cfg, "parallelism": f"target-leaf shards x{world}",
                   "l2": "flushed between timed steps (256 MB write, outside the step events)",
                   "setup_s": setup_s},
        "roofline": roofline_block(st, c, m2l_flops, achieved, peak, gemm_ms, ms_per_step, traffic),
        "phases_ms": ph,
        "p2p": {"pairs": st["m_d"], "ms": p2p_ms,
                "tflops_24flop_per_pair": 24.0 * st["m_d"] / (p2p_ms * 1e-3) / 1e12 if p2p_ms > 0 else None,
                "frac_of_fp64_peak": (24.0 * st["m_d"] / (p2p_ms * 1e-3) / 1e12 / peak
                                      if (p2p_ms > 0 and peak) else None),
                "note": "24 flop per pair (SURVEY.md 8(d), rsqrt and sincos counted as 1 each); the kernel issues "
                        "~33 FP64 instructions per pair (SASS), FP64 pipe 64 % active (profiles/r01_ncu_p2p_unroll4.json)"},
        "hbm_passes": hbm_passes(st, ph),
        "counters": {k: st[k] for k in ("n_c", "n_sc", "m_d", "n_le", "n_lminus", "l_hf", "slots_t", "slots_s",
                                        "depth_t", "depth_s")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * c.ns, "d2h_bytes_per_step": 16 * c.nt,
                "ms_per_step": e2e_ms / args.steps,
                "path": ("fdh_apply (C-ABI) with pinned host buffers" if world == 1 else
                         "pinned H2D + fdh_apply_device + NCCL all-reduce of y + D2H")},
        "gpu_launches": int(st["gpu_launches"]) * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = {k: v for k, v in cpu_oracle_sample(c, tg, sr, q, args.cpu_seconds).items()
                                   if k in ("value", "unit", "cores", "kind", "sample", "single_core")}
        except Exception as e:  # the baseline is reported, never required
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {e}"}
    print(json.dumps(out), flush=True)
    del st0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    c = CONFIGS[args.config]
    if args.impl == "reference":
        if rank == 0:
            # every step is a bounded sample; keep the whole run within a few minutes
            args.ref_seconds = max(1.0, min(args.ref_seconds, 150.0 / max(1, args.steps + args.warmup)))
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=False)
        run_reference(args, c, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    run_ours(args, c, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
