"""Multi-GPU scaling predicted on ONE B200: every rank r of
W (fdh_create_shard: a cost-balanced Morton range of target leaves, the ancestor
closure's M2L/L2L, its leaves' L2T and near field; the upward pass replicated)
is built and applied in its own process, one after the other, on the same GPU.
Per rank: setup seconds, host peak RSS (VmHWM), the apply's device time and its
phases, the cost model's share.  Per W: the predicted parallel efficiency

    eff(W) = T_1 / (W * max_r T_r)     (T = device time of one apply)

-- what W GPUs running the ranks concurrently would achieve if the y all-reduce
(16 B x N_T, ~0.1 ms on NVLink 5) is free -- and the cost model's max/mean next
to the measured max/mean.

    python tools/shard_scaling.py --config 4 --worlds 2,4,8 [--out gpurun_out/shard_cfg4.json]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def vm_hwm_gb():
    with open("/proc/self/status") as f:
        for line in f:
            if line.startswith("VmHWM:"):
                return int(line.split()[1]) / 1024 / 1024
    return None


def one(cfg, rank, world, applies):
    import numpy as np
    import torch

    import paper_2004_14229_b200 as F
    from paper_2004_14229_b200.configs import CONFIGS, make_inputs

    c = CONFIGS[cfg]
    tg, sr, q = make_inputs(c)
    t = time.perf_counter()
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, c.depth_cap,
                               c.zero_diagonal, rank=rank, world=world)
    setup_s = time.perf_counter() - t
    x = torch.from_numpy(q.view(np.float64).copy()).cuda()
    y = torch.empty(2 * c.nt, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(applies - 1):  # warm-up (graph capture)
        op.apply_device(x.data_ptr(), y.data_ptr())
    op.sync()
    op.set_timing(True)
    op.apply_device(x.data_ptr(), y.data_ptr())
    op.sync()
    st = op.stats()
    own = op.owned_leaves()
    res = {"config": cfg, "rank": rank, "world": world, "setup_s": setup_s, "vm_hwm_gb": vm_hwm_gb(),
           "apply_ms": st["apply_ms"], "phases_ms": st["phase_ms"], "m2l_gemm_ms": st["m2l_gemm_ms"],
           "shard_cost": st["shard_cost"], "total_cost": st["total_cost"], "owned_leaves": int(len(own)),
           "owned_points": int((own[:, 5] - own[:, 4]).sum()) if len(own) else 0, "m2l_items": st["m2l_items"],
           "m2l_tiles": st["m2l_tiles"], "bytes_stored": st["bytes_stored"], "structure_ms": st["structure_ms"],
           "upward_ms": st["phase_ms"]["s2m"] + st["phase_ms"]["m2m"]}
    print("RESULT " + json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--applies", type=int, default=0, help="applies per rank (last one timed); 0 = auto")
    ap.add_argument("--out", default=None)
    ap.add_argument("--one", nargs=2, type=int, default=None, metavar=("RANK", "WORLD"))
    args = ap.parse_args()
    applies = args.applies or (1 if args.config == 4 else 2)
    if args.one:
        one(args.config, args.one[0], args.one[1], applies)
        return
    out = args.out or os.path.join(os.environ.get("GRAFT_REPO_ROOT", ROOT), "gpurun_out",
                                   f"shard_cfg{args.config}.json")
    res = {"config": args.config, "method": __doc__.strip().splitlines()[0], "runs": {}}

    def run(rank, world):
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--config", str(args.config), "--applies",
                            str(applies), "--one", str(rank), str(world)], capture_output=True, text=True)
        for line in p.stdout.splitlines():
            if line.startswith("RESULT "):
                return json.loads(line[7:])
        return {"rank": rank, "world": world, "error": (p.stderr or p.stdout)[-2000:]}

    base = run(0, 1)
    res["runs"]["1"] = [base]
    t1 = base.get("apply_ms")
    for w in [int(v) for v in args.worlds.split(",")]:
        rr = [run(r, w) for r in range(w)]
        res["runs"][str(w)] = rr
        ok = [r for r in rr if "apply_ms" in r]
        if len(ok) == w and t1:
            tm = [r["apply_ms"] for r in ok]
            cm = [r["shard_cost"] for r in ok]
            res[f"W{w}"] = {
                "predicted_efficiency": t1 / (w * max(tm)),
                "apply_ms_max": max(tm), "apply_ms_mean": sum(tm) / w,
                "measured_max_over_mean": max(tm) / (sum(tm) / w),
                "cost_model_max_over_mean": max(cm) / (sum(cm) / w),
                "upward_ms_per_rank": [r["upward_ms"] for r in ok],
                "setup_s_max": max(r["setup_s"] for r in ok),
                "vm_hwm_gb_max": max(r["vm_hwm_gb"] for r in ok),
            }
        json.dump(res, open(out, "w"), indent=1)
        print(json.dumps({k: v for k, v in res.items() if k != "runs"}), flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
