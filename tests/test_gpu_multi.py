"""Multiple right-hand sides (SPEC.md:527 `apply(X[N_S x r])`):
fdh_create_multi / fdh_apply_multi against one single-vector apply per column and
against the CPU oracle.  M2L tile columns become (target slot, rhs) pairs and the
near field forms each kernel value once for up to 8 vectors, so the summation
order inside the M2L differs from the single-vector plan.  On the int8 M2L every
vector of a batch has its own per-level moment scale (the same digits as its
single-vector apply), so a batch never changes a vector's rounding (SPEC.md:527,
"batching must not change results"): columns agree with the single applies to
FP64 summation order (bound 1e-13) even when the vectors' norms differ by 1e12,
and with the oracle to the parity bound 1e-12 (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
import paper_2004_14229_b200 as F
from paper_2004_14229_b200.configs import CONFIGS, make_inputs

pytestmark = pytest.mark.gpu
TOL = 1e-12
I8 = 1e-13  # int8 M2L, same digits, different (tile, item) summation order


@pytest.fixture(scope="module", autouse=True)
def _gpu(gpu_required):
    F.build()


def _charges(k, ns, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (k, ns)) + 1j * rng.uniform(-1, 1, (k, ns))


@pytest.mark.parametrize("m,nrhs", [(4, 2), (4, 8), (4, 16), (5, 4), (6, 2)])
def test_multi_rhs_vs_single(m, nrhs):
    c = CONFIGS[2]
    nt, ns = (15000, 12000) if m <= 4 else (12000, 10000)  # the oracle's cost grows with (m+1)^6
    tg, sr, _ = make_inputs(c, nt=nt, ns=ns)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    X = _charges(nrhs + 1, ns, 7 + m)  # the last device batch is padded with zero vectors
    opm = F.DirectionalOperator(*args, nrhs=nrhs)
    st = opm.stats()
    assert st["nrhs"] == nrhs and st["n_c"] > 0
    Y = opm.apply_multi(X)
    op1 = F.DirectionalOperator(*args)
    for r in range(X.shape[0]):
        assert oracle.rel_l2(Y[r], op1.apply(X[r])) <= I8, r
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, 32, m, c.eta2, c.l_hf)
    for r in (0, nrhs):
        assert oracle.rel_l2(Y[r], o.apply(X[r])) <= TOL
    assert np.array_equal(opm.apply_multi(X), Y)  # deterministic


def test_multi_rhs_fp64_dmma(monkeypatch):
    monkeypatch.setenv("FDH_M2L_IMPL", "dmma")
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=30000, ns=25000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    X = _charges(4, 25000, 3)
    opm = F.DirectionalOperator(*args, nrhs=4)
    assert opm.stats()["m2l_impl"] == 0
    Y = opm.apply_multi(X)
    op1 = F.DirectionalOperator(*args)
    for r in range(4):
        assert oracle.rel_l2(Y[r], op1.apply(X[r])) <= 1e-13


def test_multi_rhs_zero_diagonal_and_linearity():
    """Targets == sources with the zero diagonal (batched near field skips j == k
    for every rhs); column r of A [x, 2x + i y] is linear in the inputs."""
    rng = np.random.default_rng(11)
    pts = [rng.random(20000) for _ in range(3)]
    x, yv = _charges(2, 20000, 5)
    op = F.DirectionalOperator(pts, pts, (0, 0, 0), (1, 1, 1), 10.0, 32, 4, 1.0, -2, 30, True, nrhs=4)
    Y = op.apply_multi(np.stack([x, yv, 2 * x + 1j * yv]))
    o = oracle.Oracle(pts, pts, (0, 0, 0), (1, 1, 1), 10.0, 32, 4, 1.0, -2, 30, True)
    assert oracle.rel_l2(Y[0], o.apply(x)) <= TOL
    assert oracle.rel_l2(Y[2], 2 * Y[0] + 1j * Y[1]) <= TOL


def test_multi_rhs_single_apply_and_errors():
    c = CONFIGS[2]
    tg, sr, q = make_inputs(c, nt=20000, ns=20000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    op = F.DirectionalOperator(*args, nrhs=4)
    y1 = F.DirectionalOperator(*args).apply(q)
    assert oracle.rel_l2(op.apply(q), y1) <= I8  # fdh_apply = one vector + zero padding
    with pytest.raises(F.FdhError):
        F.DirectionalOperator(*args, nrhs=3)  # not a power of two
    with pytest.raises(F.FdhError):
        op.apply_multi(np.zeros((2, 7), dtype=np.complex128))  # dimension mismatch


def test_multi_rhs_shards_sum_to_full():
    """Target shards (fdh_create_multi with rank / world) of a multi-vector
    operator: the rank outputs sum to the full multi-vector apply."""
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=20000, ns=15000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    X = _charges(4, 15000, 21)
    full = F.DirectionalOperator(*args, nrhs=4).apply_multi(X)
    acc = np.zeros_like(full)
    for rank in range(2):
        acc += F.DirectionalOperator(*args, rank=rank, world=2, nrhs=4).apply_multi(X)
    assert oracle.rel_l2(acc, full) <= I8


@pytest.mark.parametrize("nrhs,scales", [(2, [1.0, 1e-9]), (8, [1e6, 1.0, 1e-6, 3e3, 1e-3, 2e-5, 7e4, 1e-6])])
def test_multi_rhs_disparate_norms(nrhs, scales):
    """Adversarial batches: a vector 1e-9 x the other's norm, and eight
    vectors whose norms span 1e+-6.  Each column matches its own single-vector
    apply (same digit rounding: per-(rhs, level) moment scales) and the oracle."""
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=15000, ns=12000)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    X = _charges(nrhs, 12000, 40 + nrhs) * np.asarray(scales)[:, None]
    opm = F.DirectionalOperator(*args, nrhs=nrhs)
    assert opm.stats()["m2l_impl"] == 1
    Y = opm.apply_multi(X)
    op1 = F.DirectionalOperator(*args)
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, 32, 4, c.eta2, c.l_hf)
    for r in range(nrhs):
        e1, eo = oracle.rel_l2(Y[r], op1.apply(X[r])), oracle.rel_l2(Y[r], o.apply(X[r]))
        print(f"rhs {r} (scale {scales[r]:g}): vs single {e1:.2e}, vs oracle {eo:.2e}")
        assert e1 <= I8 and eo <= TOL, (r, e1, eo)
