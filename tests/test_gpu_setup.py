"""GPU setup (k_setup.cu: trees, block partition, key directions, D/D^ slots)
against the host planner, which is bit-exact with the oracle and the reference's
own ClusterTree (tests/test_plan.py, tests/test_oracle.py): every export must be
identical, bit for bit."""
import os

import numpy as np
import pytest

import paper_2004_14229_b200 as F
from paper_2004_14229_b200.configs import CONFIGS, grid_points, make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu(gpu_required):
    F.build()


def compare(tg, sr, lo, hi, kappa, n_max=64, m=4, eta2=1.0, l_hf=-2, depth_cap=30, zero_diagonal=0):
    g = F.DirectionalOperator(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal)
    os.environ["FDH_PLAN_I8"] = "1"  # the host plan of the same M2L kernel as the device operator
    try:
        h = F.DirectionalOperator(tg, sr, lo, hi, kappa, n_max, m, eta2, l_hf, depth_cap, zero_diagonal,
                                  plan_only=True)
    finally:
        del os.environ["FDH_PLAN_I8"]
    assert g.stats()["gpu_structure"] == 1 and h.stats()["gpu_structure"] == 0
    for w in (0, 1):
        assert np.array_equal(g.tree(w), h.tree(w)), f"tree {w}"
        assert np.array_equal(g.perm(w), h.perm(w)), f"perm {w}"
        assert np.array_equal(g.dirsets(w), h.dirsets(w)), f"dirsets {w}"
    assert np.array_equal(g.lplus(), h.lplus())
    assert np.array_equal(g.lminus(), h.lminus())
    sg, sh = g.stats(), h.stats()
    for k in ("n_c", "n_sc", "m_d", "n_le", "n_lminus", "l_hf", "slots_t", "slots_s", "m2l_tiles", "m2l_items",
              "m2l_impl", "m2l_flops_executed", "m2l_i8_ops"):
        assert sg[k] == sh[k], k
    return g


@pytest.mark.parametrize("cfg", [1, 2])
def test_gpu_structure_baseline(cfg):
    c = CONFIGS[cfg]
    tg, sr, _ = make_inputs(c)
    g = compare(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)
    print(f"cfg{cfg} structure {g.stats()['structure_ms']:.1f} ms on GPU")


def test_gpu_structure_cfg5_shape():
    c = CONFIGS[5]
    tg, sr, _ = make_inputs(c, nt=200000, ns=100000)
    compare(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, 4, c.eta2, c.l_hf)


@pytest.mark.parametrize("lhf", [-1, 1, 3])
def test_gpu_structure_forced_lhf(lhf):
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=30000, ns=20000)
    compare(tg, sr, c.root_lo, c.root_hi, 24.0, 32, 3, 1.0, lhf)


def test_gpu_structure_grid_and_cap():
    g = grid_points(5)
    compare(g, g, (-1, -1, -1), (1, 1, 1), 3.2, 512, 4, 5.0, 1, zero_diagonal=1)
    rng = np.random.default_rng(9)
    a = np.concatenate([rng.random((4000, 3)), np.full((100, 3), 0.3)])
    tg = [np.ascontiguousarray(a[:, i]) for i in range(3)]
    sr = [np.ascontiguousarray(rng.random(3000)) for _ in range(3)]
    compare(tg, sr, (0, 0, 0), (1, 1, 1), 5.0, 16, 2, 1.0, -2, depth_cap=6)
    s = rng.integers(0, 33, size=(9000, 3)) / 32.0
    pts = [np.ascontiguousarray(s[:, i]) for i in range(3)]
    compare(pts, pts, (0, 0, 0), (1, 1, 1), 10.0, 8, 2, 1.5, -2, zero_diagonal=1)


def test_gpu_structure_single_point_and_errors():
    one = [np.array([0.5]), np.array([0.5]), np.array([0.25])]
    compare(one, one, (0, 0, 0), (1, 1, 1), 1.0, 1, 1, zero_diagonal=1)
    bad = [np.array([0.5, 1.5]), np.array([0.5, 0.5]), np.array([0.5, 0.5])]
    with pytest.raises(F.FdhError) as e:
        F.DirectionalOperator(bad, bad, (0, 0, 0), (1, 1, 1), 1.0)
    assert e.value.code == F.ERR_ARG


def test_gpu_structure_chunked_pairs(monkeypatch):
    """the chunked two-pass partition (used for the 3e9-pair levels of config 4)"""
    monkeypatch.setenv("FDH_SETUP_PAIR_CHUNK", "5000")
    c = CONFIGS[2]
    tg, sr, _ = make_inputs(c, nt=40000, ns=30000)
    compare(tg, sr, c.root_lo, c.root_hi, c.kappa, c.n_max, c.m, c.eta2, c.l_hf)


@pytest.mark.parametrize("name", ["uniform", "snapped", "grid_k3"])
def test_gpu_tree_golden(name):
    """Trees built on the B200 (k_setup.cu) against the reference's own trees
    (tests/golden, written from oracle/_ref by tools/make_golden.py)."""
    import os

    G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_r01.npz"))
    p = G[f"tree_{name}_pts"]
    lo, hi = G[f"tree_{name}_root"]
    pts = [np.ascontiguousarray(p[:, a]) for a in range(3)]
    op = F.DirectionalOperator(pts, pts, lo, hi, 1.0, n_max=int(G[f"tree_{name}_nmax"]), m=1)
    assert op.stats()["gpu_structure"] == 1
    assert np.array_equal(op.tree(0), G[f"tree_{name}_rows"])
    assert np.array_equal(op.perm(0), G[f"tree_{name}_perm"])
