"""The CPU oracle against golden vectors of the reference's own C++ (kernel,
Chebyshev nodes, transfer matrices, interpolation matrices, cluster trees),
written by tools/make_golden.py from oracle/_ref (cluster_tree.cpp and
interpolation.cpp compiled unmodified from /root/reference).  Bitwise; runs
without /root/reference, so the oracle stays pinned on any machine."""
import os

import numpy as np
import pytest

import oracle

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_r01.npz"))
P = oracle._p


def test_kernel_golden():
    d, kap, want = G["kernel_d"], G["kernel_kappa"], G["kernel_val"]
    got = np.zeros(2)
    for i in range(len(kap)):
        oracle.lib().orc_kernel(P(np.ascontiguousarray(d[i])), float(kap[i]), P(got))
        assert np.array_equal(got, want[i])


@pytest.mark.parametrize("m", [0, 1, 4, 5, 6])
def test_chebyshev_golden(m):
    got = np.zeros(m + 1)
    for j, (lo, hi) in enumerate(G["cheb_intervals"]):
        oracle.lib().orc_chebyshev_nodes(float(lo), float(hi), m, P(got))
        assert np.array_equal(got, G[f"cheb_m{m}"][j])


@pytest.mark.parametrize("m", [1, 2, 3])
def test_transfer_golden(m):
    n = (m + 1) ** 3
    got = np.zeros(8 * n * n)
    oracle.lib().orc_transfer_reference(m, P(got))
    assert np.array_equal(got, G[f"transfer_m{m}"])


@pytest.mark.parametrize("m", [2, 3])
def test_interp_matrix_golden(m):
    n = (m + 1) ** 3
    pts, dirs = G["interp_pts"], G["interp_dirs"]
    lo, hi = (np.ascontiguousarray(G[k]) for k in ("interp_lo", "interp_hi"))
    px, py, pz = (np.ascontiguousarray(pts[a]) for a in range(3))
    for j in range(3):
        got = np.zeros(2 * 17 * n)
        oracle.lib().orc_interp_matrix(P(px), P(py), P(pz), 17, P(lo), P(hi), P(np.ascontiguousarray(dirs[j])), 12.5,
                                       m, P(got))
        assert np.array_equal(got, G[f"interp_m{m}"][j])


@pytest.mark.parametrize("name", ["uniform", "snapped", "grid_k3"])
def test_tree_golden(name):
    p = G[f"tree_{name}_pts"]
    lo, hi = G[f"tree_{name}_root"]
    pts = [np.ascontiguousarray(p[:, a]) for a in range(3)]
    o = oracle.Oracle(pts, pts, lo, hi, 1.0, n_max=int(G[f"tree_{name}_nmax"]), m=1, structure_only=True)
    assert np.array_equal(o.tree(0), G[f"tree_{name}_rows"])
    assert np.array_equal(o.perm(0), G[f"tree_{name}_perm"])


@pytest.mark.parametrize("name", ["uniform", "snapped", "grid_k3"])
def test_product_planner_tree_golden(name):
    """The product's host planner (fdh_plan_only) against the reference's trees."""
    import paper_2004_14229_b200 as F

    p = G[f"tree_{name}_pts"]
    lo, hi = G[f"tree_{name}_root"]
    pts = [np.ascontiguousarray(p[:, a]) for a in range(3)]
    op = F.DirectionalOperator(pts, pts, lo, hi, 1.0, n_max=int(G[f"tree_{name}_nmax"]), m=1, plan_only=True)
    assert np.array_equal(op.tree(0), G[f"tree_{name}_rows"])
    assert np.array_equal(op.perm(0), G[f"tree_{name}_perm"])
