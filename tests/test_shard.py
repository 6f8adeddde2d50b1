"""Multi-GPU sharding on CPU: world_size-2 gloo process group,
each rank builds its shard plan (fdh_plan_only); the shards must partition the
target leaves exactly, balance the estimated cost, and keep the M2L / L2L work
restricted to the ancestor closure of their leaves."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2004_14229_b200 as F
    from paper_2004_14229_b200.configs import CONFIGS, make_inputs

    c = CONFIGS[cfg]
    nt, ns = (60000, 30000) if cfg == 5 else (c.nt, c.ns)
    tg, sr, _ = make_inputs(c, nt=nt, ns=ns)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf,
                               rank=rank, world=world, plan_only=True)
    own = op.owned_leaves()
    st = op.stats()
    # gather owned leaves and costs over the group (gloo)
    n = torch.tensor([len(own)], dtype=torch.int64)
    ns_ = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ns_, n)
    mx = int(max(t.item() for t in ns_))
    buf = torch.full((mx, 6), -1, dtype=torch.int64)
    buf[: len(own)] = torch.from_numpy(own)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    cost = torch.tensor([st["shard_cost"], st["total_cost"], float(st["m2l_flops_executed"])], dtype=torch.float64)
    costs = [torch.zeros_like(cost) for _ in range(world)]
    dist.all_gather(costs, cost)
    if rank == 0:
        full = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf,
                                     plan_only=True)
        allown = np.concatenate([b.numpy()[: int(k.item())] for b, k in zip(bufs, ns_)])
        np.save(os.path.join(out_dir, "union.npy"), allown)
        np.save(os.path.join(out_dir, "full.npy"), full.owned_leaves())
        np.save(os.path.join(out_dir, "costs.npy"), torch.stack(costs).numpy())
        np.save(os.path.join(out_dir, "full_m2l.npy"), np.array([float(full.stats()["m2l_flops_executed"])]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [2, 5])
def test_two_rank_shards_partition_targets(cfg, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), cfg, str(tmp_path)), nprocs=world, join=True)
    union = np.load(tmp_path / "union.npy")
    full = np.load(tmp_path / "full.npy")
    u = union[np.lexsort(union.T[::-1])]
    assert np.array_equal(u, full)  # every target leaf owned exactly once
    costs = np.load(tmp_path / "costs.npy")
    shard, total = costs[:, 0], costs[0, 1]
    assert abs(shard.sum() - total) <= 1e-9 * total
    assert shard.max() / shard.mean() < 1.05  # cost-weighted Morton split
    # each shard executes only its part of M2L (plus shared coarse ancestors)
    full_m2l = np.load(tmp_path / "full_m2l.npy")[0]
    assert costs[:, 2].max() < 0.75 * full_m2l
    assert costs[:, 2].sum() >= full_m2l * 0.99
