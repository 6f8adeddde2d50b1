"""CPU oracle pinned against the reference's own code (oracle/_ref), the SPEC
examples and PAPER Table 1.  (tiers 1-2.)"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2004_14229_b200.configs import CONFIGS, grid_points, make_inputs

REF = oracle.ref()
needs_ref = pytest.mark.skipif(REF is None, reason="reference build (oracle/_ref) unavailable")
P = oracle._p


def f64(*a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- geometry
def test_kernel_spec_examples():
    # kappa=2pi, r=1 -> 1/(4pi); kappa=pi -> -1/(4pi)
    out = np.zeros(2)
    oracle.lib().orc_kernel(P(f64(1, 0, 0)), 2 * math.pi, P(out))
    assert abs(out[0] - 1 / (4 * math.pi)) < 1e-15 and abs(out[1]) < 1e-15
    oracle.lib().orc_kernel(P(f64(1, 0, 0)), math.pi, P(out))
    assert abs(out[0] + 1 / (4 * math.pi)) < 1e-15
    assert oracle.lib().orc_kernel(P(f64(0, 0, 0)), 1.0, P(out)) == 2  # domain_error at r=0


@needs_ref
def test_kernel_matches_reference_bitwise():
    rng = np.random.default_rng(7)
    a, b = np.zeros(2), np.zeros(2)
    for _ in range(200):
        d = rng.standard_normal(3)
        kap = float(rng.uniform(0.1, 100))
        oracle.lib().orc_kernel(P(f64(*d)), kap, P(a))
        REF.ref_kernel(P(f64(*d)), kap, P(b))
        assert np.array_equal(a, b)


# ---------------------------------------------------------- interpolation
@needs_ref
@pytest.mark.parametrize("m", [0, 1, 4, 5, 6])
def test_chebyshev_and_transfer_bitwise(m):
    a, b = np.zeros(m + 1), np.zeros(m + 1)
    for lo, hi in [(-1.0, 1.0), (0.0, 1.0), (0.25, 0.3125), (-3.0, 7.5)]:
        oracle.lib().orc_chebyshev_nodes(lo, hi, m, P(a))
        REF.ref_chebyshev_nodes(lo, hi, m, P(b))
        assert np.array_equal(a, b)
    n = (m + 1) ** 3
    Ea, Eb = np.zeros(8 * n * n), np.zeros(8 * n * n)
    oracle.lib().orc_transfer_reference(m, P(Ea))
    REF.ref_transfer_reference(m, P(Eb))
    assert np.array_equal(Ea, Eb)
    # SPEC.md:371 partition of unity
    assert np.abs(Ea.reshape(8, n, n).sum(axis=2) - 1).max() < 1e-13


def test_chebyshev_spec_m1():
    out = np.zeros(2)
    oracle.lib().orc_chebyshev_nodes(-1.0, 1.0, 1, P(out))
    assert abs(out[0] - math.sqrt(2) / 2) < 1e-15 and abs(out[1] + math.sqrt(2) / 2) < 1e-15


@needs_ref
@pytest.mark.parametrize("m", [2, 4, 6])
def test_interp_matrix_bitwise(m):
    rng = np.random.default_rng(m)
    lo, hi = f64(0.25, 0.5, 0.0), f64(0.375, 0.625, 0.125)
    pts = [np.ascontiguousarray(lo[a] + (hi[a] - lo[a]) * rng.random(17)) for a in range(3)]
    n = (m + 1) ** 3
    for c in (f64(0, 0, 0), f64(1, 0, 0), oracle.dir_vector(0, 2, 37)):
        A, B = np.zeros(2 * 17 * n), np.zeros(2 * 17 * n)
        oracle.lib().orc_interp_matrix(P(pts[0]), P(pts[1]), P(pts[2]), 17, P(lo), P(hi), P(c), 12.5, m, P(A))
        REF.ref_interp_matrix(P(pts[0]), P(pts[1]), P(pts[2]), 17, P(lo), P(hi), P(c), 12.5, m, P(B))
        assert np.array_equal(A, B)


# ------------------------------------------------------------ cluster tree
def _tree_cases():
    c1 = CONFIGS[1]
    tg, sr, _ = make_inputs(c1)
    c5 = CONFIGS[5]
    t5, s5, _ = make_inputs(c5, nt=30000, ns=30000)
    rng = np.random.default_rng(3)
    # points snapped onto grid lines and the lower boundary (App. C hazards)
    snap = rng.integers(0, 65, size=(20000, 3)) / 64.0
    snap[snap == 0] = 0.0
    snap = [np.ascontiguousarray(snap[:, a]) for a in range(3)]
    g = grid_points(4)
    return [
        ("cfg1_targets", tg, (0, 0, 0), (1, 1, 1), 64),
        ("cfg5_mixture", s5, (0, 0, 0), (2, 1, 1), 64),
        ("snapped", snap, (0, 0, 0), (1, 1, 1), 16),
        ("grid_k4", g, (-1, -1, -1), (1, 1, 1), 7),
        ("tiny", [f64(0.5), f64(0.5), f64(0.5)], (0, 0, 0), (1, 1, 1), 1),
    ]


@needs_ref
@pytest.mark.parametrize("case", _tree_cases(), ids=lambda c: c[0])
def test_tree_bitwise_vs_reference(case):
    name, pts, lo, hi, nmax = case
    o = oracle.Oracle(pts, pts, lo, hi, 1.0, n_max=nmax, m=1, structure_only=True)
    x, y, z = (np.ascontiguousarray(a, dtype=np.float64) for a in pts)
    h = REF.ref_tree_create(P(x), P(y), P(z), len(x), P(f64(*lo)), P(f64(*hi)), nmax, 30)
    assert h
    try:
        n = REF.ref_tree_export(h, None)
        rows = np.zeros((n, 7), dtype=np.int64)
        REF.ref_tree_export(h, oracle._pi(rows))
        perm = np.zeros(len(x), dtype=np.int64)
        REF.ref_tree_perm(h, oracle._pi(perm))
    finally:
        REF.ref_tree_destroy(h)
    assert np.array_equal(o.tree(0), rows)
    assert np.array_equal(o.perm(0), perm)


def test_tree_spec_examples():
    g = grid_points(5)
    o = oracle.Oracle(g, g, (-1, -1, -1), (1, 1, 1), 3.2, n_max=512, m=4, eta2=5.0, l_hf=1, structure_only=True)
    t = o.tree(0)
    leaves = t[t[:, 6] == 1]
    assert len(leaves) == 64 and np.all(leaves[:, 5] - leaves[:, 4] == 512)
    one = [f64(0.3), f64(0.3), f64(0.3)]
    o1 = oracle.Oracle(one, one, (0, 0, 0), (1, 1, 1), 1.0, n_max=1, m=1, structure_only=True)
    assert o1.tree(0).shape[0] == 1


def test_tree_errors():
    p = [f64(0.5, 1.5), f64(0.5, 0.5), f64(0.5, 0.5)]
    with pytest.raises(oracle.OracleError) as e:
        oracle.Oracle(p, p, (0, 0, 0), (1, 1, 1), 1.0, structure_only=True)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError):
        oracle.Oracle(p, p, (0, 0, 0), (2, 1, 1), -1.0, structure_only=True)


# --------------------------------------------------------------- directions
def test_direction_counts_and_nesting():
    for lhf in (1, 2, 3, 5):
        for l in range(lhf + 1):
            nd = 6 * 4 ** (lhf - l)
            V = np.array([oracle.dir_vector(l, lhf, j) for j in range(nd)])
            assert np.allclose(np.linalg.norm(V, axis=1), 1.0, atol=1e-15)
            if l < lhf:  # nesting: dir_(l+1)(c_j) = j >> 2
                for j in range(nd):
                    assert oracle.dir_map_vector(l + 1, lhf, V[j]) == j >> 2
            for j in range(nd):  # dir_map(l, c_j) = j
                assert oracle.dir_map_vector(l, lhf, V[j]) == j
    # SPEC.md:193 normalize(1, 1/2, 1/2) in D^(1) for l_hf = 2
    V = np.array([oracle.dir_vector(1, 2, j) for j in range(24)])
    w = np.array([1, 0.5, 0.5]) / np.linalg.norm([1, 0.5, 0.5])
    assert np.min(np.linalg.norm(V - w, axis=1)) < 1e-15
    # SPEC.md:201 (1,1,1)/sqrt3 -> (1,0,0), index 1; zero above l_hf
    assert oracle.dir_map_vector(2, 2, np.ones(3) / math.sqrt(3)) == 1
    assert oracle.dir_map_vector(5, 2, np.ones(3)) == 0
    assert oracle.dir_index(2, 2, (-3, 0, 0)) == 0 and oracle.dir_index(2, 2, (0, 0, 4)) == 5


# ---------------------------------------------------------------- block tree
@pytest.mark.parametrize("k,nc,nsc,nf", [(5, 3096, 316, 24.41), (6, 166320, 1522, 4.06)])
def test_table1_counters(k, nc, nsc, nf):
    """PAPER.md:673-674 / SPEC.md:278-279, 429-430 (Table 1)."""
    g = grid_points(k)
    o = oracle.Oracle(g, g, (-1, -1, -1), (1, 1, 1), 0.1 * 2 ** k, n_max=512, m=4, eta2=5.0, l_hf=k - 4,
                      zero_diagonal=1, structure_only=True)
    s = o.stats()
    assert s["N_C"] == nc and s["N_SC"] == nsc
    assert round(100.0 * s["M_D"] / (8 ** k) ** 2, 2) == nf
    lm = o.lminus()
    assert np.all(lm[:, 0] == k - 4 + 1)  # SPEC.md:293 all inadmissible blocks at l_hf + 1


def test_block_partition_identity_cfg1():
    c = CONFIGS[1]
    tg, sr, _ = make_inputs(c)
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf, structure_only=True)
    s = o.stats()
    assert s["N_C"] == 166344 and s["N_SC"] == 2986 and s["l_hf"] == 2
    T, S = o.tree(0), o.tree(1)
    cntT = {tuple(r[:4]): r[5] - r[4] for r in T}
    cntS = {tuple(r[:4]): r[5] - r[4] for r in S}
    tot = sum(cntT[tuple(b[:4])] * cntS[(b[0], b[4], b[5], b[6])] for b in o.lplus())
    tot += sum(cntT[tuple(b[:4])] * cntS[tuple(b[4:8])] for b in o.lminus())
    assert tot == c.nt * c.ns  # SPEC.md:291 partition identity


# -------------------------------------------------------------------- engine
def test_engine_cfg1_vs_dense_and_linearity():
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c)
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    y = o.apply(q)
    rows = np.random.default_rng(0).choice(c.nt, 256, replace=False)
    err = oracle.rel_l2(y[rows], oracle.dense_rows(tg, sr, q, c.kappa, rows))
    assert err < 1e-4  # survey: ~4e-6
    q2 = np.random.default_rng(1).standard_normal(c.ns) + 0j
    a = 0.3 - 1.7j
    y2 = o.apply(q2)
    y3 = o.apply(a * q + q2)
    assert oracle.rel_l2(y3, a * y + y2) < 1e-12
    assert np.array_equal(o.apply(q), y)  # SPEC.md:516 determinism
    lv = np.arange(0, o.leaf_count(0), 5)
    r, ys = o.apply_sampled(q, lv)
    assert np.array_equal(ys, y[r])


def test_engine_pure_nearfield_equals_dense():
    # L+ empty (huge kappa): fast == dense to 1e-13
    rng = np.random.default_rng(11)
    pt = [rng.random(900) for _ in range(3)]
    ps = [rng.random(700) for _ in range(3)]
    q = rng.standard_normal(700) + 1j * rng.standard_normal(700)
    o = oracle.Oracle(pt, ps, (0, 0, 0), (1, 1, 1), 1e6, n_max=16, m=2)
    assert o.stats()["N_C"] == 0
    y = o.apply(q)
    yd = oracle.dense_rows(pt, ps, q, 1e6, np.arange(900))
    assert oracle.rel_l2(y, yd) < 1e-13


def test_zero_diagonal():
    g = grid_points(3)
    rng = np.random.default_rng(5)
    q = rng.standard_normal(512) + 1j * rng.standard_normal(512)
    o = oracle.Oracle(g, g, (-1, -1, -1), (1, 1, 1), 0.8, n_max=8, m=3, eta2=5.0, l_hf=-1, zero_diagonal=1)
    y = o.apply(q)
    assert o.stats()["M_D_zero"] == 512
    yd = oracle.dense_rows(g, g, q, 0.8, np.arange(512), zero_diagonal=1)
    assert oracle.rel_l2(y, yd) < 1e-2


@pytest.mark.parametrize("cfg,m", [(1, 4), (2, 3)])
def test_sampled_structure_oracle_matches_full(cfg, m):
    """orc_create_sampled (partition only below the sampled leaves' ancestors,
    coupling generated per block; used for config 4, whose full L+ and coupling
    set do not fit in host memory) gives bitwise the rows of the full oracle."""
    c = CONFIGS[cfg]
    nt, ns = (None, None) if cfg == 1 else (30000, 25000)
    tg, sr, q = make_inputs(c) if cfg == 1 else make_inputs(c, nt=nt, ns=ns)
    args = (tg, sr, c.root_lo, c.root_hi, c.kappa, 32 if cfg == 2 else c.n_max, m, c.eta2, c.l_hf)
    full = oracle.Oracle(*args)
    nl = full.leaf_count(0)
    leaves = np.unique(np.concatenate([[0, nl - 1], np.random.default_rng(cfg).choice(nl, 4, replace=False)]))
    rows, yf = full.apply_sampled(q, leaves)
    samp = oracle.Oracle(*args, sample_leaves=leaves)
    rows2, ys = samp.apply_sampled(q, leaves)
    assert np.array_equal(rows, rows2)
    assert np.array_equal(yf, ys)


# ------------------------------------------------------ ACA
def test_aca_spec_examples():
    rng = np.random.default_rng(3)
    u = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    v = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    A = np.outer(u, v)
    U, W = oracle.aca_compress(A, 1e-10)
    assert U.shape[1] == 1 and np.linalg.norm(A - U @ W) <= 1e-14 * np.linalg.norm(A)  # rank 1 recovered
    assert oracle.aca_compress(np.eye(30, dtype=np.complex128), 1e-12) is None  # incompressible: dense
    # a k = 5 (PAPER section 4 grid) coupling matrix at eps = 1e-6 -> residual <= 1e-5
    A = oracle.coupling_matrix(4, 3.2, (2 / 32, 2 / 32, 2 / 32), (2, 1, 0), oracle.dir_vector(1, 1, 0))
    U, W = oracle.aca_compress(A, 1e-6)
    assert U.shape[1] < 125 / 2 and np.linalg.norm(A - U @ W) <= 1e-5 * np.linalg.norm(A)


def test_aca_matvec_agrees_with_dense():
    """with ACA at eps = 1e-8 the matvec agrees with the dense one to 1e-6."""
    c = CONFIGS[1]
    tg, sr, q = make_inputs(c)
    o = oracle.Oracle(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    y = o.apply(q)
    o.set_aca(1e-8)
    r = o.aca_ranks()
    assert (r > 0).sum() > 0 and r.max() < 125 // 2 + 1
    ya = o.apply(q)
    err = oracle.rel_l2(ya, y)
    assert 0 < err <= 1e-6, err
    o.set_aca(0.0)
    assert np.array_equal(o.apply(q), y)
