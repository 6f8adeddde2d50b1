"""Golden vectors from the reference's own C++ (oracle/_ref: cluster_tree.cpp and
interpolation.cpp compiled unmodified from /root/reference), written to
tests/golden/reference_r01.npz so that the oracle stays pinned where
/root/reference is absent (tests/test_golden.py).  Run here (the container that
has /root/reference):  python tools/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2004_14229_b200.configs import grid_points  # noqa: E402

R = oracle.ref()
if R is None:
    sys.exit("oracle/_ref (the reference build) is unavailable: run where /root/reference exists")
P, PI = oracle._p, oracle._pi
f64 = lambda *a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
out = {}
rng = np.random.default_rng(2004_14229)

# geometry.hpp:80-86 kernel_diff
d = rng.standard_normal((64, 3))
kap = rng.uniform(0.1, 100.0, 64)
kv = np.zeros((64, 2))
for i in range(64):
    R.ref_kernel(P(np.ascontiguousarray(d[i])), float(kap[i]), P(kv[i]))
out.update(kernel_d=d, kernel_kappa=kap, kernel_val=kv)

# interpolation.cpp:9-20 chebyshev_nodes, 89-119 build_transfer_reference
ivals = np.array([(-1.0, 1.0), (0.0, 1.0), (0.25, 0.3125), (-3.0, 7.5)])
out["cheb_intervals"] = ivals
for m in (0, 1, 4, 5, 6):
    nodes = np.zeros((len(ivals), m + 1))
    for j, (lo, hi) in enumerate(ivals):
        R.ref_chebyshev_nodes(float(lo), float(hi), m, P(nodes[j]))
    out[f"cheb_m{m}"] = nodes
for m in (1, 2, 3):
    n = (m + 1) ** 3
    E = np.zeros(8 * n * n)
    R.ref_transfer_reference(m, P(E))
    out[f"transfer_m{m}"] = E

# interpolation.cpp:56-87 build_interp_matrix (rows L_k(x_j) exp(i kappa <x_j, c>))
lo, hi = f64(0.25, 0.5, 0.0), f64(0.375, 0.625, 0.125)
pts = np.stack([lo[a] + (hi[a] - lo[a]) * rng.random(17) for a in range(3)])
dirs = np.stack([f64(0, 0, 0), f64(1, 0, 0), oracle.dir_vector(0, 2, 37)])
out.update(interp_lo=lo, interp_hi=hi, interp_pts=pts, interp_dirs=dirs)
for m in (2, 3):
    n = (m + 1) ** 3
    A = np.zeros((3, 2 * 17 * n))
    px, py, pz = (np.ascontiguousarray(pts[a]) for a in range(3))
    for j in range(3):
        R.ref_interp_matrix(P(px), P(py), P(pz), 17, P(lo), P(hi), P(np.ascontiguousarray(dirs[j])), 12.5, m, P(A[j]))
    out[f"interp_m{m}"] = A

# cluster_tree.cpp:12-151 ClusterTree: canonical rows (level, i, j, k, begin, end, leaf) + permutation
snap = rng.integers(0, 65, size=(3000, 3)) / 64.0
cases = {
    "uniform": (1.0 - rng.random((3000, 3)), (0, 0, 0), (1, 1, 1), 32),
    "snapped": (snap, (0, 0, 0), (1, 1, 1), 16),
    "grid_k3": (np.stack(grid_points(3), axis=1), (-1, -1, -1), (1, 1, 1), 7),
}
for name, (p, clo, chi, nmax) in cases.items():
    x, y, z = (np.ascontiguousarray(p[:, a], dtype=np.float64) for a in range(3))
    h = R.ref_tree_create(P(x), P(y), P(z), len(x), P(f64(*clo)), P(f64(*chi)), nmax, 30)
    assert h, R.ref_last_error()
    n = R.ref_tree_export(h, None)
    rows = np.zeros((n, 7), dtype=np.int64)
    R.ref_tree_export(h, PI(rows))
    perm = np.zeros(len(x), dtype=np.int64)
    R.ref_tree_perm(h, PI(perm))
    R.ref_tree_destroy(h)
    out.update({f"tree_{name}_pts": p.astype(np.float64), f"tree_{name}_root": np.array([clo, chi], dtype=np.float64),
                f"tree_{name}_nmax": np.array(nmax), f"tree_{name}_rows": rows, f"tree_{name}_perm": perm})

dst = os.path.join(ROOT, "tests", "golden", "reference_r01.npz")
os.makedirs(os.path.dirname(dst), exist_ok=True)
np.savez_compressed(dst, **out)
print(dst, os.path.getsize(dst), "bytes,", len(out), "arrays")
