#!/usr/bin/env python3
"""Benchmark of the directional Helmholtz matvec (BASELINE.json metric:
"directional-FMM matvec time & (N_T+N_S)/s at 1/2/4/8 B200; % FP64 roofline").

A step = one apply y = A x of the configured workload.  Default: BASELINE
config 4 (N_T = N_S = 4,000,000, kappa = 64, m = 6) -- the scaling config the
metric is quoted on ("at 1/2/4/8 B200"), the largest that runs on one GPU.
Setup (trees, partition, coupling scales) is outside the timed region, as t_s in
PAPER.md Table 1, and reported as run.setup_s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Timed region (every step, N = 1): the C-ABI host call fdh_apply with pinned host
buffers (H2D of x, the apply as one CUDA-graph replay, D2H of y) -- `e2e` -- and,
inside it, the device time of the apply kernels from the library's CUDA events
around the graph launch -- `value` (inputs already in HBM).  The per-phase times
and the M2L kernel time come from event-record nodes inside the same replays.
N > 1 (torchrun, or `--gpus N` which re-launches itself under torchrun): every
rank owns a cost-balanced Morton range of target leaves (fdh_create_shard) and
the step is H2D + fdh_apply_device + NCCL all-reduce of y + D2H on the
operator's stream; times are the max over ranks.
`--impl reference` times the CPU restatement of the reference algorithm
(oracle/, OpenMP, all host cores) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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


def config_block(c):
    """`config` of the JSON line: the workload and the L2 statement -- the same dict in both
    arms (the driver compares them); run-specific facts (parallelism, launch mode, setup
    seconds) are in `run`."""
    return {"workload": workload_desc(c), "cfg": c.cfg,
            "l2": "the apply's working set (coupling matrices / digits, moments: GBs) is far larger than the 126 MB "
                  "L2 and any CPU cache; the GPU arm also flushes L2 (256 MB write) between timed steps, outside "
                  "the step events"}


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML in-process
    (pynvml; no subprocess, so the sampler does not perturb short steps), else the
    nvidia-smi query of the profiling recipe."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period=0.2):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml as N

        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append([str(sm), str(mx), hex(r)] + ["Active" if r & b else "Not Active" for b in bits])
            self._stop.wait(self.period)

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            self.samples = []
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(self.period)

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


# ---------------------------------------------------------------- CPU reference
class CpuReference:
    """The CPU restatement of the reference algorithm (oracle/, TEST INFRASTRUCTURE,
    OpenMP over all host threads) on bounded samples of the workload.

    The sampled-structure oracle (orc_create_sampled) builds both trees in full and
    refines the partition below the sampled target leaves' ancestors; each sample
    is a set of COMPLETE sibling groups (all leaf children of random parent boxes)
    so the parent level's M2L is paid once per 8 leaves, as in a full run.  Per
    sample the oracle reports its upward-pass, coupling-generation (once per key
    the sample uses), M2L and downward/near-field seconds; the full apply is
    extrapolated as upward + coupling x N_SC / keys used + (M2L + downward) x
    target leaves / sampled leaves (label: extrapolated)."""

    def __init__(self, c, tg, sr, nsamples, groups_per_sample=1, seed=7):
        import oracle

        self.oracle = oracle
        self.c = c
        self.cores = int(oracle.lib().orc_set_threads(0))
        args = (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap, c.zero_diagonal)
        t = time.perf_counter()
        probe = oracle.Oracle(*args, sample_leaves=[0])
        tt = probe.tree(0)
        self.n_sc = None
        del probe
        lv = tt[tt[:, 6] == 1]
        self.nl = len(lv)
        # parent of each leaf = its coordinate >> 1 at level - 1
        par = np.stack([lv[:, 0] - 1, lv[:, 1] >> 1, lv[:, 2] >> 1, lv[:, 3] >> 1], axis=1)
        _, gid = np.unique(par, axis=0, return_inverse=True)
        gid = gid.reshape(-1)
        ngroups = int(gid.max()) + 1
        rng = np.random.default_rng(seed)
        pick = rng.choice(ngroups, min(ngroups, nsamples * groups_per_sample), replace=False)
        self.samples = []
        for i in range(nsamples):
            gsel = pick[i * groups_per_sample:(i + 1) * groups_per_sample]
            self.samples.append(np.nonzero(np.isin(gid, gsel))[0].astype(np.int64))
        allv = np.unique(np.concatenate(self.samples))
        self.op = oracle.Oracle(*args, sample_leaves=allv)
        self.setup_s = time.perf_counter() - t
        self.q = None

    def run(self, q, i, n_sc):
        t = time.perf_counter()
        self.op.apply_sampled(q, self.samples[i])
        wall = time.perf_counter() - t
        tm = self.op.last_timing()
        k = max(tm["keys_generated"], 1.0)
        full = (tm["upward"] + tm["coupling"] * n_sc / k + (tm["m2l"] + tm["down_nf"]) * self.nl / len(self.samples[i]))
        return {"wall_s": wall, "apply_s_extrapolated": full, "timing": tm, "leaves": int(len(self.samples[i]))}

    def describe(self, r, n):
        tm = r["timing"]
        return (f"oracle/ (CPU restatement of PAPER Alg. 4, OpenMP {self.cores} threads), sampled-structure mode: "
                f"{n} sample(s) of complete sibling groups of target leaves (last: {r['leaves']} of {self.nl} leaves, "
                f"{r['wall_s']:.1f} s: upward {tm['upward']:.2f} s, coupling generation {tm['coupling']:.2f} s for "
                f"{int(tm['keys_generated'])} keys, M2L {tm['m2l']:.2f} s, L2L/L2T/near field {tm['down_nf']:.2f} s); "
                f"full apply extrapolated to {r['apply_s_extrapolated']:.1f} s = upward + coupling x N_SC / keys + "
                f"(M2L + downward) x leaves ratio")


def run_reference(args, c, rank, world):
    """--impl reference: the reference algorithm on the host cores (oracle port)."""
    if rank != 0:
        return
    tg, sr, q = make_inputs(c)
    n_sc = int(json.load(open(os.path.join(ROOT, "tests", "golden", f"structure_cfg{c.cfg}.json")))["counts"]["n_sc"])
    ref = CpuReference(c, tg, sr, args.steps, groups_per_sample=args.ref_groups)
    for _ in range(args.warmup):  # warm-up: the upward pass only (no target leaves)
        ref.op.apply_sampled(q, np.zeros(0, dtype=np.int64))
    steps, walls = [], []
    r = None
    for i in range(args.steps):
        r = ref.run(q, i, n_sc)
        steps.append(r["apply_s_extrapolated"])
        walls.append(r["wall_s"])
    t = float(np.mean(steps))
    value = (c.nt + c.ns) / t
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128 (f64)", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "config": config_block(c),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.cores, "kind": "port",
                         "sample": ref.describe(r, args.steps) + f"; mean over {args.steps} samples (extrapolated)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": ref.setup_s,
        # ms_per_step is the full apply EXTRAPOLATED from the step's bounded sample; the wall
        # time a step actually took on the host is this:
        "extrapolated": True, "sample_wall_ms_per_step": 1e3 * float(np.mean(walls)),
    }
    print(json.dumps(out), flush=True)


def cpu_baseline(c, tg, sr, q, seconds):
    """cpu_baseline leg of our arm (rank 0, N = 1): one or two sibling-group samples."""
    n_sc = int(json.load(open(os.path.join(ROOT, "tests", "golden", f"structure_cfg{c.cfg}.json")))["counts"]["n_sc"])
    ref = CpuReference(c, tg, sr, 2, groups_per_sample=1, seed=11)
    r1 = ref.run(q, 0, n_sc)
    rs = [r1]
    if r1["wall_s"] < 0.5 * seconds:
        rs.append(ref.run(q, 1, n_sc))
    t = float(np.mean([r["apply_s_extrapolated"] for r in rs]))
    return {"value": (c.nt + c.ns) / t, "unit": UNIT, "cores": ref.cores, "kind": "port",
            "sample": ref.describe(rs[-1], len(rs)) + f"; mean of {len(rs)} (extrapolated)"}


# ---------------------------------------------------------------- roofline
def roofline_block(st, c, m2l_flops, peak, gemm_ms, ms_per_step, traffic):
    """Roofline of the M2L kernel: the int8 tcgen05 digit GEMM (k_m2l_i8) against
    the measured int8 tensor peak, or the FP64 DMMA GEMM against the FP64 peak."""
    share = gemm_ms / ms_per_step if ms_per_step else None
    achieved = m2l_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    fp64 = {"achieved_tflops": achieved, "fp64_peak_tflops": peak,
            "ratio": (achieved / peak) if (achieved and peak) else None,
            "note": "algorithmic FP64 flop (8 n^2 per admissible block) per second of the M2L kernel, against the "
                    "measured FP64 DMMA peak"}
    if st["m2l_impl"] == 1:
        import paper_2004_14229_b200 as F
        tops_burst = F.tensor_peak_tops(0)
        # a kernel timed inside a long step runs at the sustained (power-limited) clocks: its
        # roofline is the sustained peak (the same MMA loop held for ~3 s); short steps: burst
        sustained = gemm_ms >= 1000.0
        tops_sust = F.tensor_peak_tops(1) if sustained else None
        tops = tops_sust if sustained and tops_sust else tops_burst
        # algorithmic int8 work: the KS (KS + 1) / 2 digit-pair products (i + j <= KS - 1) of every
        # real MAC of the complex product (4 n^2 per block, 2 ops per MAC); KS x bits from the library
        ks, bits = int(st["m2l_i8_digits"]), int(st["m2l_i8_bits"])
        npair = int(st["m2l_i8_products"])
        alg = float(npair) * m2l_flops
        ach = alg / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        iss = st["m2l_i8_ops"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        return {"bound": "tensor", "kernel": f"k_m2l_i8 (tcgen05.mma kind::i8, exact {ks} x {bits}-bit digit fixed-point "
                                            f"products, TMEM int32 level accumulators)",
                "achieved": ach, "peak": tops, "unit": "TOPS", "frac": (ach / tops) if (ach and tops) else None,
                "traffic": traffic,
                "peak_source": ("measured live: int8 tcgen05 microbenchmark (M=128 N=256 K=32 MMAs back to back on all "
                                "SMs; MEASURED_PEAKS.json has no int8 entry), " +
                                ("SUSTAINED: held for ~3 s, rate over the last 0.6 s (the M2L kernel runs for seconds at "
                                 "the power-limited clocks)" if sustained and tops_sust else
                                 "BURST: best of three ~1 ms runs (the M2L kernel is short)")),
                "peak_burst": tops_burst, "peak_sustained": tops_sust,
                "frac_of_burst_peak": (ach / tops_burst) if (ach and tops_burst) else None,
                "algorithmic": f"{npair} digit products x 8 n^2 ops per admissible block x N_C={st['n_c']} = {alg:.4g} "
                               f"int8 ops per apply",
                "issued_ops": st["m2l_i8_ops"], "issued_frac": (iss / tops) if (iss and tops) else None,
                "issued_note": "int8 ops the kernel issues: every target column of a tile for every key of the tile "
                               "(absent columns are zero), rows padded to 128, K to 2 x 16k",
                "fp64_equivalent": fp64, "gemm_ms": gemm_ms, "share_of_step": share,
                "timing": "CUDA event-record nodes inside the timed graph replays, on the operator's stream"}
    return {"bound": "tensor", "kernel": "k_m2l_gemm (FP64 DMMA mma.sync.m8n8k4)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
            "peak_source": "measured live: fdh_fp64_peak_tflops(0) DMMA microbenchmark (no FP64 entry in "
                           "MEASURED_PEAKS.json)",
            "algorithmic": f"8 n^2 flop per admissible block x N_C={st['n_c']} = {m2l_flops:.4g} flop per "
                           f"apply (SURVEY.md 8(d); the count holds for a 3M complex product)",
            "issued_flop": st["m2l_flops_executed"], "gemm_ms": gemm_ms, "share_of_step": share}


def hbm_passes(st, ph):
    """S2M / M2M / L2L / L2T against the measured HBM copy bandwidth (MEASURED_PEAKS.json
    hbm_gbs): algorithmic bytes of SURVEY.md 8(d) (fdh_stats.hbm_bytes) / phase time."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "fallback: nominal B200 HBM3e (MEASURED_PEAKS.json absent)"
    out = {"peak_gbs": peak, "peak_source": src}
    for k in ("s2m", "m2m", "l2l", "l2t"):
        b, ms = st["hbm_bytes"][k], ph.get(k, 0.0)
        gbs = b / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[k] = {"bytes": b, "ms": ms, "achieved_gbs": gbs, "frac": gbs / peak if gbs else None}
    return out


# ---------------------------------------------------------------- our arm
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
    stream = torch.cuda.ExternalStream(op.stream(), device=dev)
    xh_t = torch.from_numpy(q.view(np.float64).copy()).pin_memory()
    yh_t = torch.empty(2 * c.nt, dtype=torch.float64).pin_memory()
    xh, yh = xh_t.numpy().view(np.complex128), yh_t.numpy().view(np.complex128)
    x = torch.empty(2 * c.ns, dtype=torch.float64, device=dev)
    y = torch.empty(2 * c.nt, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    torch.cuda.synchronize()
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def step():
        """one e2e step; returns the device ms of the apply alone (N > 1: events
        around fdh_apply_device on the operator's stream)"""
        if world == 1:
            op.apply(xh, out=yh)  # C-ABI host call: H2D, graph replay, D2H, sync
            return None
        with torch.cuda.stream(stream):
            x.copy_(xh_t, non_blocking=True)
            ev_a[0].record(stream)
        op.apply_device(x.data_ptr(), y.data_ptr(), op.stream())
        with torch.cuda.stream(stream):
            ev_a[1].record(stream)
            dist.all_reduce(y)
            yh_t.copy_(y, non_blocking=True)
        stream.synchronize()
        return ev_a[0].elapsed_time(ev_a[1])

    op.set_timing(True)  # phase events as event-record nodes inside the graph (captured in the warm-up)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    op.sync()  # deferred device errors of the warm-up (fdh_sync)
    if world > 1:
        dist.barrier()
    op.set_timing(True)  # reset the averages: only the timed applies below count (same graph, no re-capture)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dev_ms = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank, period=0.1 if args.config <= 2 else 0.5) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (outside the step events)
                evs[i][0].record(stream)
            d = step()
            evs[i][1].record(stream)
            if d is not None:
                dev_ms.append(d)
        torch.cuda.synchronize()
    op.sync()
    st = op.stats()
    e2e_ms = sum(a.elapsed_time(b) for a, b in evs)
    if world == 1:
        assert st["applies_collected"] == args.steps, st["applies_collected"]
        apply_ms = st["apply_ms_sum"]
    else:
        apply_ms = sum(dev_ms)
    if world > 1:
        t = torch.tensor([apply_ms, e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        apply_ms, e2e_ms = float(t[0].item()), float(t[1].item())
        dist.barrier()
    ms_per_step = apply_ms / args.steps
    value = args.steps * (c.nt + c.ns) / (apply_ms / 1e3)
    e2e_value = args.steps * (c.nt + c.ns) / (e2e_ms / 1e3)
    if rank != 0:
        return
    # ---- roofline of the dominant kernel (the M2L GEMM)
    peak = F.fp64_peak_tflops(0)
    n = (c.m + 1) ** 3
    m2l_flops = 8.0 * n * n * st["n_c"]  # algorithmic
    gemm_ms = st["m2l_gemm_ms"]
    traffic = None
    if os.path.exists(PROFILE_TRAFFIC):
        try:
            traffic = json.load(open(PROFILE_TRAFFIC)).get(f"cfg{c.cfg}{'_i8' if st['m2l_impl'] == 1 else ''}")
        except Exception:
            traffic = None
    ph = st["phase_ms"]
    p2p_ms = ph.get("p2p", 0.0)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": (f"complex128 (f64; M2L as exact int8 x int8 -> int32 digit products of "
                  f"{st['m2l_i8_digits'] * st['m2l_i8_bits']}-bit fixed-point operands on tcgen05)" if st["m2l_impl"] == 1 else "complex128 (f64)"),
        "data": "synthetic (seeded uniform / Gaussian-mixture points, U(-1,1) complex charges; SURVEY.md 8(d))",
        "config": config_block(c),
        "run": {"parallelism": f"target-leaf shards x{world}",
                "launch_mode": f"CUDA graph replays ({st['graph_replays']} in total incl. warm-up), phase timing "
                               f"by event-record nodes inside the graph",
                "setup_s": setup_s},
        "roofline": roofline_block(st, c, m2l_flops, peak, gemm_ms, ms_per_step, traffic),
        "phases_ms": ph,
        "p2p": {"pairs": st["m_d"], "ms": p2p_ms,
                "tflops_24flop_per_pair": 24.0 * st["m_d"] / (p2p_ms * 1e-3) / 1e12 if p2p_ms > 0 else None,
                "frac_of_fp64_peak": (24.0 * st["m_d"] / (p2p_ms * 1e-3) / 1e12 / peak
                                      if (p2p_ms > 0 and peak) else None),
                "note": "24 flop per pair (SURVEY.md 8(d), rsqrt and sincos counted as 1 each)"},
        "hbm_passes": hbm_passes(st, ph),
        "counters": {k: st[k] for k in ("n_c", "n_sc", "m_d", "n_le", "n_lminus", "l_hf", "slots_t", "slots_s",
                                        "depth_t", "depth_s")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * c.ns, "d2h_bytes_per_step": 16 * c.nt,
                "ms_per_step": e2e_ms / args.steps,
                "path": ("fdh_apply (C-ABI host call) with pinned host buffers, the same applies as `value`"
                         if world == 1 else "pinned H2D + fdh_apply_device + NCCL all-reduce of y + D2H")},
        "gpu_launches": int(st["gpu_launches"]) * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(c, tg, sr, q, args.cpu_seconds)
        except Exception as e:  # the baseline is reported, never required
            out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port", "sample": f"failed: {e}"}
    print(json.dumps(out), flush=True)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-groups", type=int, default=1, help="sibling groups of target leaves per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd, env=env).returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    c = CONFIGS[args.config]
    if args.impl == "reference":
        if rank == 0:
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=False)
        run_reference(args, c, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if torch.cuda.device_count() < world:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "error": f"--gpus {world} needs {world} visible GPUs, "
                                                              f"found {torch.cuda.device_count()}"}), flush=True)
            sys.exit(1)
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    run_ours(args, c, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
