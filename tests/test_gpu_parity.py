"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Tolerance: relative l2 <= 1e-12 on y (BASELINE.json
north_star); structure is bit-exact (tests/test_plan.py)."""
import numpy as np
import pytest

import oracle
import paper_2004_14229_b200 as F
from paper_2004_14229_b200.configs import CONFIGS, grid_points, make_inputs

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu(gpu_required):
    F.build()


def run_pair(tg, sr, q, lo, hi, kappa, n_max=64, m=4, eta2=1.0, l_hf=-2, zero_diagonal=0, depth_cap=30):
    op = F.DirectionalOperator(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal)
    o = oracle.Oracle(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal)
    return op.apply(q), o.apply(q), op, o


def test_cfg1_full_parity():
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c)
    y, yo, op, _ = run_pair(tg, sr, q, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    err = oracle.rel_l2(y, yo)
    print("cfg1 rel l2 vs oracle", err, op.stats()["apply_ms"], "ms")
    assert err <= TOL
    assert np.array_equal(op.apply(q), y)  # bitwise determinism


@pytest.mark.parametrize("m", [0, 1, 2, 3, 4, 5, 6])
def test_degrees(m):
    rng = np.random.default_rng(100 + m)
    tg = [rng.random(6000) for _ in range(3)]
    sr = [rng.random(5000) for _ in range(3)]
    q = rng.uniform(-1, 1, 5000) + 1j * rng.uniform(-1, 1, 5000)
    y, yo, _, _ = run_pair(tg, sr, q, (0, 0, 0), (1, 1, 1), 12.0, 32, m, 1.0, -2)
    assert oracle.rel_l2(y, yo) <= TOL


@pytest.mark.parametrize("lhf", [-1, 1, 2, 3])
def test_direction_levels(lhf):
    """Directional transfers with c and c' both nonzero (l_hf forced above the
    leaf level), and the non-directional case (l_hf = -1)."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=30000, ns=25000)
    y, yo, op, _ = run_pair(tg, sr, q, c.root_lo, c.root_hi, 24.0, 32, 3, 1.0, lhf)
    assert op.stats()["n_c"] > 0
    assert oracle.rel_l2(y, yo) <= TOL


def test_cfg5_shape_nonuniform():
    c = CONFIGS[5]
    tg, sr, q = make_inputs(c, nt=40000, ns=20000)
    y, yo, op, _ = run_pair(tg, sr, q, c.root_lo, c.root_hi, c.kappa, c.n_max, 4, c.eta2, c.l_hf)
    assert oracle.rel_l2(y, yo) <= TOL


@pytest.mark.parametrize("kappa,eta2", [(1e6, 1.0), (5e5, 1e-9), (57.0, 1e-9), (1.0, 1e-9)])
def test_pure_nearfield_and_dense(kappa, eta2):
    # near-field phase kappa * d_max (d_max ~ sqrt 3) selects the P2P variant:
    # > 1.5e6 library sincos, < 1.5e6 exact r + fast sincos, <= 100 FMA r + table sincos
    rng = np.random.default_rng(11)
    pt = [rng.random(900) for _ in range(3)]
    ps = [rng.random(700) for _ in range(3)]
    q = rng.standard_normal(700) + 1j * rng.standard_normal(700)
    op = F.DirectionalOperator(pt, ps, (0, 0, 0), (1, 1, 1), kappa, n_max=16, m=2, eta2=eta2)
    assert op.stats()["n_c"] == 0
    yd = oracle.dense_rows(pt, ps, q, kappa, np.arange(900))
    assert oracle.rel_l2(op.apply(q), yd) <= 1e-13


def test_zero_diagonal_grid():
    g = grid_points(4)
    rng = np.random.default_rng(5)
    q = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    y, yo, _, _ = run_pair(g, g, q, (-1, -1, -1), (1, 1, 1), 1.6, 64, 4, 5.0, 0, zero_diagonal=1)
    assert oracle.rel_l2(y, yo) <= TOL


def test_linearity():
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m)
    q2 = np.random.default_rng(1).standard_normal(c.ns) + 0j
    a = 0.3 - 1.7j
    assert oracle.rel_l2(op.apply(a * q + q2), a * op.apply(q) + op.apply(q2)) <= 1e-12


def test_singular_kernel_reported():
    rng = np.random.default_rng(2)
    pts = [rng.random(500) for _ in range(3)]
    op = F.DirectionalOperator(pts, pts, (0, 0, 0), (1, 1, 1), 2.0, n_max=32, m=2)
    with pytest.raises(F.FdhError) as e:
        op.apply(np.ones(500, dtype=np.complex128))
    assert e.value.code == F.ERR_DOMAIN  # geometry.hpp:82 domain_error
    opz = F.DirectionalOperator(pts, pts, (0, 0, 0), (1, 1, 1), 2.0, n_max=32, m=2, zero_diagonal=True)
    opz.apply(np.ones(500, dtype=np.complex128))
    # device path: the error is deferred to fdh_sync (include/fdhelm_c.h)
    import torch

    x = torch.ones(1000, dtype=torch.float64, device="cuda")
    y = torch.empty(1000, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    op.apply_device(x.data_ptr(), y.data_ptr())
    op.apply_device(x.data_ptr(), y.data_ptr())
    with pytest.raises(F.FdhError) as e:
        op.sync()
    assert e.value.code == F.ERR_DOMAIN
    op.sync()  # cleared
    opz.apply_device(x.data_ptr(), y.data_ptr())
    opz.sync()


def test_dimension_mismatch():
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c, nt=2000, ns=2000)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa)
    with pytest.raises(F.FdhError) as e:
        op.apply(q[:10])
    assert e.value.code == F.ERR_DIM


def test_cfg2_sampled_oracle():
    """BASELINE config 2 at full size: sampled-target oracle."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    y = op.apply(q)
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    nl = o.leaf_count(0)
    leaves = np.unique(np.concatenate([[0, nl - 1], np.random.default_rng(2).choice(nl, 40, replace=False)]))
    rows, ys = o.apply_sampled(q, leaves)
    err = oracle.rel_l2(y[rows], ys)
    print("cfg2 sampled rel l2", err, "rows", len(rows))
    assert err <= TOL


def test_cpp_host_demo():
    """The C++ host API (include/fdhelm_b200.hpp) end to end: examples/matvec_demo."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "matvec_demo")
    out = subprocess.run([exe, "20000", "8", "4"], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0


@pytest.mark.parametrize("world", [2, 3])
def test_shards_sum_to_full_apply(world):
    """fdh_create_shard semantics on one GPU: the ranks' outputs (their targets,
    zeros elsewhere) sum to the single-operator result (what the NCCL all-reduce
    in bench.py computes across GPUs)."""
    c = CONFIGS[5]
    tg, sr, q = make_inputs(c, nt=60000, ns=30000)
    full = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, 4, c.eta2, c.l_hf).apply(q)
    acc = np.zeros_like(full)
    rows = []
    for r in range(world):
        op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, 4, c.eta2, c.l_hf,
                                   rank=r, world=world)
        y = op.apply(q)
        own = op.owned_leaves()
        rows.append(int((own[:, 5] - own[:, 4]).sum()))
        acc += y
    assert sum(rows) == 60000  # every target row owned by exactly one rank
    assert oracle.rel_l2(acc, full) <= 1e-14


def test_onthefly_coupling_segments(monkeypatch):
    """Coupling matrices generated per apply in key-chunk segments (the mode used
    when they do not fit in HBM, e.g. config 4): identical to the resident mode."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=60000, ns=50000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    monkeypatch.setenv("FDH_M2L_IMPL", "dmma")  # the mode is an FP64-path feature (config 4, m = 6)
    y_res = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_W_ONTHEFLY", "1")
    op = F.DirectionalOperator(*args)
    st = op.stats()
    assert st["w_resident"] == 0 and st["w_segments"] >= 1
    y = op.apply(q)
    assert np.array_equal(y, y_res)  # same matrices, same summation order


@pytest.mark.parametrize("m", [1, 2, 4, 5, 6])
def test_m2l_int8_tensor_vs_fp64_dmma(m, monkeypatch):
    """The int8 tcgen05 M2L (k_m2l_i8: exact products of 48-bit fixed-point
    operands) against the FP64 DMMA M2L and the oracle on the same inputs."""
    c = CONFIGS[2]
    nt, ns = (30000, 25000) if m <= 4 else (15000, 12000)  # the oracle's cost grows with (m+1)^6
    tg, sr, q = make_inputs(c, nt=nt, ns=ns)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    op8 = F.DirectionalOperator(*args)
    assert op8.stats()["m2l_impl"] == 1
    y8 = op8.apply(q)
    assert op8.stats()["m2l_i8_ops"] > 0
    monkeypatch.setenv("FDH_M2L_IMPL", "dmma")
    opd = F.DirectionalOperator(*args)
    assert opd.stats()["m2l_impl"] == 0
    yd = opd.apply(q)
    yo = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf).apply(q)
    e8, ed, e8d = oracle.rel_l2(y8, yo), oracle.rel_l2(yd, yo), oracle.rel_l2(y8, yd)
    print(f"m={m}: int8 vs oracle {e8:.2e}, dmma vs oracle {ed:.2e}, int8 vs dmma {e8d:.2e}")
    # measured with the 6 x 8-bit + level-6 digits: int8 vs dmma <= 3e-14 at every m
    assert e8 <= TOL and ed <= TOL and e8d <= 1e-13
    assert np.array_equal(op8.apply(q), y8)  # deterministic: exact integer sums, fixed FP64 chain order


def test_m2l_int8_item_split(monkeypatch):
    """Items capped at 8 keys (many chained items per tile, the int32 overflow
    guard F of k_m2l_i8) give the same y up to FP64 rounding of the chain."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=40000, ns=40000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    monkeypatch.setenv("FDH_M2L_HYBRID", "0")  # chained target-tile items only
    monkeypatch.setenv("FDH_M2L_PAIR", "0")
    op = F.DirectionalOperator(*args)
    y = op.apply(q)
    monkeypatch.setenv("FDH_M2L_FKEYS", "8")
    op2 = F.DirectionalOperator(*args)
    assert op2.stats()["m2l_items"] > 2 * op.stats()["m2l_items"]
    assert oracle.rel_l2(op2.apply(q), y) <= 1e-14


def test_m6_int8_two_mblock_groups():
    """n = 343 nodes per box (m = 6): 352 rows run as two M-block groups ({0, 1}
    and {2}, separate ticket chains); the int8 path is used and matches the oracle."""
    rng = np.random.default_rng(7)
    tg = [rng.random(3000) for _ in range(3)]
    sr = [rng.random(3000) for _ in range(3)]
    y, yo, op, _ = run_pair(tg, sr, rng.uniform(-1, 1, 3000) + 1j * rng.uniform(-1, 1, 3000), (0, 0, 0), (1, 1, 1),
                            12.0, 32, 6, 1.0, -2)
    assert op.stats()["m2l_impl"] == 1 and op.stats()["n_c"] > 0
    assert oracle.rel_l2(y, yo) <= TOL


@pytest.mark.parametrize("m", [4, 6])
def test_onthefly_coupling_segments_int8(m, monkeypatch):
    """int8 coupling digits generated per apply in key-chunk segments (config 4:
    229 GB of digits do not fit) against digits generated once at setup: bitwise."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=40000 if m <= 4 else 20000, ns=30000 if m <= 4 else 15000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    op_res = F.DirectionalOperator(*args)
    assert op_res.stats()["m2l_impl"] == 1 and op_res.stats()["w_resident"] == 1
    y_res = op_res.apply(q)
    monkeypatch.setenv("FDH_W_ONTHEFLY", "1")
    monkeypatch.setenv("FDH_W_SLOT_MB", "64")  # several segments at this size
    op = F.DirectionalOperator(*args)
    st = op.stats()
    assert st["m2l_impl"] == 1 and st["w_resident"] == 0 and st["w_segments"] >= 2
    y = op.apply(q)
    assert np.array_equal(y, y_res)  # same digits and scales, same summation order


def test_cuda_graph_replay_matches_direct(monkeypatch):
    """The apply runs as a replay of a captured CUDA graph (one graph launch per
    apply); the direct launches (FDH_CUDA_GRAPH=0) give the same bits."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=30000, ns=25000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    op = F.DirectionalOperator(*args)
    y1 = op.apply(q)
    y2 = op.apply(2 * q)
    assert op.stats()["graph_replays"] >= 2
    monkeypatch.setenv("FDH_CUDA_GRAPH", "0")
    opd = F.DirectionalOperator(*args)
    assert np.array_equal(opd.apply(q), y1) and np.array_equal(opd.apply(2 * q), y2)
    assert opd.stats()["graph_replays"] == 0


def test_overlapped_near_field_same_bits(monkeypatch):
    """FDH_OVERLAP_NEARFIELD=1: the near field as a persistent grid on the second
    stream, launched before the M2L -- same y bits as the sequential order."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=30000, ns=25000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    y = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_OVERLAP_NEARFIELD", "1")
    assert np.array_equal(F.DirectionalOperator(*args).apply(q), y)


@pytest.mark.parametrize("impl", ["i8", "dmma"])
def test_m2l_progress_with_concurrent_kernel(impl, monkeypatch):
    """The M2L item chains progress whatever the CTA dispatch order: a CTA claims
    its item from an atomic counter only once it runs, so every item an epilogue
    waits for is held by a running CTA.  A long GEMM on another stream competes
    for the SMs; y is bitwise the same as alone."""
    import torch

    if impl == "dmma":
        monkeypatch.setenv("FDH_M2L_IMPL", "dmma")
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=40000, ns=30000)
    op = F.DirectionalOperator(tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    y_ref = op.apply(q)
    x = torch.from_numpy(q.view(np.float64).copy()).cuda()
    y = torch.empty(2 * 40000, dtype=torch.float64, device="cuda")
    a = torch.randn(4096, 4096, device="cuda")
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s2):
        for _ in range(30):
            a = torch.tanh(a @ a)
    op.apply_device(x.data_ptr(), y.data_ptr())
    with torch.cuda.stream(s2):
        for _ in range(30):
            a = torch.tanh(a @ a)
    torch.cuda.synchronize()
    op.sync()
    assert np.array_equal(y.cpu().numpy().view(np.complex128), y_ref)


@pytest.mark.parametrize("m", [5, 6])
def test_m2l_int8_tile32_mblock_passes(m, monkeypatch):
    """m = 5, 6 (2-3 M-blocks): 32 target columns (N up to 448 per W digit, one
    128-row M-block per pass, W digits stored per block) against 16 columns (one
    pass over M-blocks {0, 1} [+ {2}]) and the oracle; the planner picks one of
    the two per operator (FDH_I8_TILE forces it)."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=15000, ns=12000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    monkeypatch.setenv("FDH_I8_TILE", "16")
    y16 = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_I8_TILE", "32")
    op = F.DirectionalOperator(*args)
    assert op.stats()["m2l_impl"] == 1
    y32 = op.apply(q)
    yo = oracle.Oracle(*args).apply(q)
    assert oracle.rel_l2(y32, yo) <= TOL and oracle.rel_l2(y32, y16) <= 1e-13
    monkeypatch.setenv("FDH_W_ONTHEFLY", "1")
    monkeypatch.setenv("FDH_W_SLOT_MB", "64")
    op2 = F.DirectionalOperator(*args)
    assert op2.stats()["w_segments"] >= 2
    assert np.array_equal(op2.apply(q), y32)


def test_multi_gpu_group_operator(monkeypatch):
    """fdh_create(n_gpus): the in-library multi-GPU operator (one shard per device,
    NCCL broadcast of x / reduce of y).  On this one-GPU box: the group path with
    n_gpus = 1 (FDH_GROUP=1: NCCL communicator of one device) equals the plain
    operator bitwise, and n_gpus beyond the device count is refused."""
    import torch

    c = CONFIGS[5]
    tg, sr, q = make_inputs(c, nt=40000, ns=20000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, 4, c.eta2, c.l_hf)
    y = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_GROUP", "1")
    g = F.DirectionalOperator(*args, n_gpus=1)
    assert np.array_equal(g.apply(q), y)
    x = torch.from_numpy(q.view(np.float64).copy()).cuda()
    yd = torch.empty(2 * 40000, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    g.apply_device(x.data_ptr(), yd.data_ptr())
    g.sync()
    assert np.array_equal(yd.cpu().numpy().view(np.complex128), y)
    assert len(g.owned_leaves()) > 0 and g.stats()["n_c"] > 0
    n = torch.cuda.device_count()
    with pytest.raises(F.FdhError) as e:
        F.DirectionalOperator(*args, n_gpus=n + 1)
    assert e.value.code == F.ERR_UNSUPPORTED
    if n >= 2:
        g2 = F.DirectionalOperator(*args, n_gpus=2)
        assert oracle.rel_l2(g2.apply(q), y) <= 1e-14


@pytest.mark.parametrize("m", [7, 8])
def test_high_degrees(m):
    """Interpolation degree m >= 7 (the reference builders accept any m >= 0,
    interpolation.cpp:9-20): the int8 M2L with one 128-row M-block per pass and
    32 target columns (n = 512 / 729 nodes per box) against the oracle."""
    rng = np.random.default_rng(200 + m)
    tg = [rng.random(4000) for _ in range(3)]
    sr = [rng.random(3500) for _ in range(3)]
    q = rng.uniform(-1, 1, 3500) + 1j * rng.uniform(-1, 1, 3500)
    y, yo, op, _ = run_pair(tg, sr, q, (0, 0, 0), (1, 1, 1), 12.0, 32, m, 1.0, -2)
    st = op.stats()
    assert st["m2l_impl"] == 1 and st["n_c"] > 0
    err = oracle.rel_l2(y, yo)
    print(f"m={m}: rel l2 vs oracle {err:.2e}")
    assert err <= TOL


@pytest.mark.parametrize("m", [4, 5, 6])
def test_aca_compressed_m2l(m):
    """ACA-compressed coupling on the B200 (fdh_set_aca, lossy):
    at eps = 1e-8 the apply agrees with the exact one and with the oracle's ACA
    and dense matvecs to 1e-6; eps = 0 restores the exact M2L."""
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c, nt=6000 if m == 6 else 10000, ns=5000 if m == 6 else 10000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32 if m > 4 else c.n_max, m, c.eta2, c.l_hf)
    op = F.DirectionalOperator(*args)
    y = op.apply(q)
    op.set_aca(1e-8)
    st = op.stats()
    ya = op.apply(q)
    o = oracle.Oracle(*args)
    yo = o.apply(q)
    o.set_aca(1e-8)
    yoa = o.apply(q)
    e1, e2, e3 = oracle.rel_l2(ya, y), oracle.rel_l2(ya, yo), oracle.rel_l2(ya, yoa)
    print(f"m={m}: ACA mean rank {st['aca_mean_rank']:.1f} (dense keys {st['aca_dense_keys']}), vs exact {e1:.2e}, "
          f"vs oracle {e2:.2e}, vs oracle ACA {e3:.2e}")
    assert st["aca_eps"] == 1e-8 and st["aca_bytes"] > 0
    assert e1 <= 1e-6 and e2 <= 1e-6 and e3 <= 1e-6
    op.set_aca(0.0)
    assert np.array_equal(op.apply(q), y)


def test_cached_near_field():
    """FDH_CACHE_NEARFIELD (fdh_set_cache): the near-field kernel values
    cached once, streamed by later applies -- the same y as recomputing them (to the
    sincos / rsqrt rounding) and the oracle; zero diagonal, several right-hand sides,
    and freeing the cache restore the computing kernel bitwise."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=30000, ns=25000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    op = F.DirectionalOperator(*args)
    y = op.apply(q)
    op.set_cache(True)
    st = op.stats()
    assert st["nf_cache_bytes"] >= 16 * st["m_d"]
    yc = op.apply(q)
    assert oracle.rel_l2(yc, y) <= 1e-13
    assert oracle.rel_l2(yc, oracle.Oracle(*args).apply(q)) <= TOL
    op.set_cache(False)
    assert np.array_equal(op.apply(q), y)
    rng = np.random.default_rng(4)
    pts = [rng.random(8000) for _ in range(3)]
    X = rng.standard_normal((3, 8000)) + 1j * rng.standard_normal((3, 8000))
    opz = F.DirectionalOperator(pts, pts, (0, 0, 0), (1, 1, 1), 10.0, 32, 4, 1.0, -2, 30, True, nrhs=4)
    Y = opz.apply_multi(X)
    opz.set_cache(True)
    assert oracle.rel_l2(opz.apply_multi(X), Y) <= 1e-13
    ops = F.DirectionalOperator(pts, pts, (0, 0, 0), (1, 1, 1), 10.0, 32, 4)
    with pytest.raises(F.FdhError) as e:
        ops.set_cache(True)  # coincident points without the zero diagonal: singular
    assert e.value.code == F.ERR_DOMAIN


@pytest.mark.parametrize("m", [4, 5, 6])
def test_m2l_pair_mode(m, monkeypatch):
    """int8 M2L in pair mode (key-major over (target, source) pairs, chosen by the
    planner for clustered sources): against the target-tile mode and the oracle;
    many output segments (FDH_PAIR_OUT_MB) and per-apply W digits in segments give
    the same bits."""
    c = CONFIGS[5]
    tg, sr, q = make_inputs(c, nt=30000 if m < 6 else 12000, ns=15000 if m < 6 else 8000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    monkeypatch.setenv("FDH_M2L_PAIR", "0")
    yt = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_M2L_PAIR", "1")
    op = F.DirectionalOperator(*args)
    st = op.stats()
    assert st["m2l_pair_mode"] == 1 and st["n_c"] > 0
    y = op.apply(q)
    yo = oracle.Oracle(*args).apply(q)
    e1, e2 = oracle.rel_l2(y, yo), oracle.rel_l2(y, yt)
    print(f"m={m}: pair mode vs oracle {e1:.2e}, vs tile mode {e2:.2e}")
    assert e1 <= TOL and e2 <= 1e-13
    assert np.array_equal(op.apply(q), y)  # deterministic
    monkeypatch.setenv("FDH_PAIR_OUT_MB", "8")
    monkeypatch.setenv("FDH_W_ONTHEFLY", "1")
    monkeypatch.setenv("FDH_W_SLOT_MB", "64")
    op2 = F.DirectionalOperator(*args)
    assert op2.stats()["w_segments"] >= 3
    assert np.array_equal(op2.apply(q), y)


@pytest.mark.parametrize("m", [4, 6])
def test_m2l_hybrid_mode(m, monkeypatch):
    """int8 M2L hybrid: (tile, key) rows with every column present stay in the
    target tiles, the pairs of the partial ones run key-major (pair part) -- the
    same y as the plain target tiles (to FP64 summation order) and the oracle; W
    digits generated per apply and a small pair buffer give the same bits."""
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=30000 if m == 4 else 12000, ns=25000 if m == 4 else 10000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    monkeypatch.setenv("FDH_M2L_HYBRID", "0")
    yt = F.DirectionalOperator(*args).apply(q)
    monkeypatch.setenv("FDH_M2L_HYBRID", "1")
    op = F.DirectionalOperator(*args)
    assert op.stats()["m2l_pair_mode"] == 1
    y = op.apply(q)
    yo = oracle.Oracle(*args).apply(q)
    e1, e2 = oracle.rel_l2(y, yo), oracle.rel_l2(y, yt)
    print(f"m={m}: hybrid vs oracle {e1:.2e}, vs target tiles {e2:.2e}")
    assert e1 <= TOL and e2 <= 1e-13
    monkeypatch.setenv("FDH_PAIR_OUT_MB", "4")
    monkeypatch.setenv("FDH_W_ONTHEFLY", "1")
    monkeypatch.setenv("FDH_W_SLOT_MB", "64")
    op2 = F.DirectionalOperator(*args)
    assert op2.stats()["w_segments"] >= 3
    assert np.array_equal(op2.apply(q), y)


@pytest.mark.parametrize("m", [4, 6])
def test_int8_m2l_wide_dynamic_range(m):
    """The int8 M2L rounds moments against one scale per level: charges spanning twelve
    orders of magnitude, clustered sources (box populations from 1 to hundreds) and a
    zero block of charges must still give y within 1e-12 (relative l2) of the oracle --
    the absolute rounding error is relative to the level's largest moment, as the
    l2 norm of y is."""
    rng = np.random.default_rng(900 + m)
    nt, ns = 9000, 8000
    tg = [rng.random(nt) for _ in range(3)]
    ctr = rng.random((6, 3))
    sr = [np.clip(ctr[rng.integers(0, 6, ns), a] + 0.04 * rng.standard_normal(ns), 1e-9, 1.0) for a in range(3)]
    mag = 10.0 ** rng.uniform(-6, 6, ns)
    q = mag * np.exp(2j * np.pi * rng.random(ns))
    q[: ns // 10] = 0.0
    y, yo, op, _ = run_pair(tg, sr, q, (0, 0, 0), (1, 1, 1), 14.0, 32, m, 1.0, -2)
    assert op.stats()["m2l_impl"] == 1 and op.stats()["n_c"] > 0
    err = oracle.rel_l2(y, yo)
    print(f"m={m}: wide dynamic range, rel l2 vs oracle {err:.2e}")
    assert err <= TOL
    # all-zero charges: zero moments (scale exponent of 0) -> exactly zero far field
    y0 = op.apply(np.zeros(ns, dtype=np.complex128))
    assert np.all(y0 == 0)
