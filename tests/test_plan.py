"""Product planner (host setup of libfdhelm_b200.so, built with fdh_plan_only --
no GPU needed) against the CPU oracle: bit-exact trees, permutations, L+/L-
lists, direction indices and direction sets (tier 3)."""
import numpy as np
import pytest

import oracle
import paper_2004_14229_b200 as F
from paper_2004_14229_b200.configs import CONFIGS, grid_points, make_inputs


def both(tg, sr, lo, hi, kappa, n_max=64, m=4, eta2=1.0, l_hf=-2, zero_diagonal=0):
    op = F.DirectionalOperator(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, zero_diagonal=zero_diagonal,
                               plan_only=True)
    o = oracle.Oracle(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, zero_diagonal=zero_diagonal,
                      structure_only=True)
    return op, o


def assert_same(op, o):
    for w in (0, 1):
        assert np.array_equal(op.tree(w), o.tree(w))
        assert np.array_equal(op.perm(w), o.perm(w))
        assert np.array_equal(op.dirsets(w), o.dirsets(w))
    assert np.array_equal(op.lplus(), o.lplus())
    assert np.array_equal(op.lminus(), o.lminus())
    s, t = op.stats(), o.stats()
    assert (s["n_c"], s["n_sc"], s["m_d"], s["n_le"], s["n_lminus"], s["l_hf"]) == (
        t["N_C"], t["N_SC"], t["M_D"], t["N_LE"], t["N_Lminus"], t["l_hf"])
    assert (s["slots_t"], s["slots_s"], s["nodes_t"], s["nodes_s"]) == (
        t["slots_T"], t["slots_S"], t["nodes_T"], t["nodes_S"])


def test_symbols_exported():
    L = F.lib()
    for s in F.SYMBOLS:
        assert hasattr(L, s), s
    assert "sm_100a" in F.version()


@pytest.mark.parametrize("cfg", [1, 2])
def test_planner_matches_oracle_baseline_configs(cfg):
    c = CONFIGS[cfg]
    tg, sr, _ = make_inputs(c)
    op, o = both(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    assert_same(op, o)


def test_planner_cfg5_shape_subsample():
    c = CONFIGS[5]
    tg, sr, _ = make_inputs(c, nt=60000, ns=30000)
    op, o = both(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    assert_same(op, o)
    assert op.stats()["depth_s"] > op.stats()["depth_t"]  # clustered sources refine deeper


@pytest.mark.parametrize("k", [5, 6])
def test_planner_table1(k):
    g = grid_points(k)
    op, o = both(g, g, (-1, -1, -1), (1, 1, 1), 0.1 * 2 ** k, 512, 4, 5.0, k - 4, zero_diagonal=1)
    s = op.stats()
    assert s["n_c"] == {5: 3096, 6: 166320}[k] and s["n_sc"] == {5: 316, 6: 1522}[k]
    assert_same(op, o)


@pytest.mark.parametrize("lhf", [-1, 0, 1, 2, 3, 4])
def test_planner_forced_lhf(lhf):
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=20000, ns=15000)
    op, o = both(tg, sr, c.root_lo, c.root_hi, 24.0, 32, 3, 1.0, lhf)
    assert_same(op, o)


def test_planner_snapped_and_boundary_points():
    rng = np.random.default_rng(3)
    a = rng.integers(0, 33, size=(9000, 3)) / 32.0
    b = rng.integers(0, 33, size=(7000, 3)) / 32.0
    # avoid exact target == source coincidences only matter for apply, not structure
    tg = [np.ascontiguousarray(a[:, i]) for i in range(3)]
    sr = [np.ascontiguousarray(b[:, i]) for i in range(3)]
    op, o = both(tg, sr, (0, 0, 0), (1, 1, 1), 10.0, 8, 2, 1.5, -2)
    assert_same(op, o)


def test_planner_nonuniform_depth_cap():
    rng = np.random.default_rng(9)
    a = np.concatenate([rng.random((4000, 3)), np.full((100, 3), 0.3)])  # 100 coincident points
    tg = [np.ascontiguousarray(a[:, i]) for i in range(3)]
    sr = [np.ascontiguousarray(rng.random(3000)) for _ in range(3)]
    op = F.DirectionalOperator(tg, sr, (0, 0, 0), (1, 1, 1), 5.0, 16, 2, 1.0, -2, depth_cap=6, plan_only=True)
    o = oracle.Oracle(tg, sr, (0, 0, 0), (1, 1, 1), 5.0, 16, 2, 1.0, -2, depth_cap=6, structure_only=True)
    assert_same(op, o)
    t = op.tree(0)
    assert t[:, 0].max() == 6 and ((t[:, 5] - t[:, 4])[t[:, 6] == 1] > 16).any()  # oversized leaf at the cap


def test_planner_errors():
    p = [np.array([0.5, 1.5]), np.array([0.5, 0.5]), np.array([0.5, 0.5])]
    with pytest.raises(F.FdhError) as e:
        F.DirectionalOperator(p, p, (0, 0, 0), (1, 1, 1), 1.0, plan_only=True)
    assert e.value.code == F.ERR_ARG
    q = [np.array([0.5]), np.array([0.5]), np.array([0.5])]
    for kw in ({"kappa": -1.0}, {"kappa": float("inf")}, {"n_max": 0}):
        args = dict(kappa=1.0)
        args.update(kw)
        with pytest.raises(F.FdhError) as e:
            F.DirectionalOperator(q, q, (0, 0, 0), (1, 1, 1), plan_only=True, **args)
        assert e.value.code == F.ERR_ARG
    with pytest.raises(F.FdhError):
        F.DirectionalOperator([np.zeros(0)] * 3, q, (0, 0, 0), (1, 1, 1), 1.0, plan_only=True)


def test_apply_refused_without_device_state():
    q = [np.array([0.5]), np.array([0.5]), np.array([0.25])]
    op = F.DirectionalOperator(q, q, (0, 0, 0), (1, 1, 1), 1.0, plan_only=True)
    with pytest.raises(F.FdhError) as e:
        op.apply(np.ones(1, dtype=np.complex128))
    assert e.value.code == F.ERR_UNSUPPORTED
