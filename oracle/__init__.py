"""ctypes bindings of the CPU oracle (liboracle.so) and the reference build
(_ref/libfdhelm_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REFLIB = os.path.join(HERE, "_ref", "libfdhelm_ref.so")

NSTATS = 13
STAT_NAMES = ["N_C", "N_SC", "M_D", "N_LE", "N_Lminus", "depth_T", "depth_S", "l_hf",
              "slots_T", "slots_S", "nodes_T", "nodes_S", "M_D_zero"]

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    if force or not os.path.exists(LIB) or (os.path.isdir("/root/reference/proj") and not os.path.exists(REFLIB)):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)


def _p(a):
    return a.ctypes.data_as(_d)


def _pi(a):
    return a.ctypes.data_as(_i64)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_create.argtypes = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_int64, _d, _d, C.c_double, C.c_int,
                                 C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.orc_create_structure.argtypes = L.orc_create.argtypes
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_apply.argtypes = [C.c_void_p, _d, _d]
        L.orc_apply_sampled.argtypes = [C.c_void_p, _d, _i64, C.c_int64, _d]
        L.orc_leaf_count.argtypes = [C.c_void_p, C.c_int]
        L.orc_leaf_count.restype = C.c_int64
        L.orc_leaf_points.argtypes = [C.c_void_p, C.c_int, C.c_int64, _i64, C.c_int64]
        L.orc_leaf_points.restype = C.c_int64
        L.orc_stats.argtypes = [C.c_void_p, _i64]
        L.orc_last_timing.argtypes = [C.c_void_p, _d]
        L.orc_set_aca.argtypes = [C.c_void_p, C.c_double]
        L.orc_aca_ranks.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.orc_aca_ranks.restype = C.c_int64
        L.orc_aca_compress.argtypes = [_d, C.c_int, C.c_double, C.c_int, _d, _d]
        for f in ("orc_export_tree", "orc_export_perm", "orc_export_dirsets"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, _i64]
            getattr(L, f).restype = C.c_int64
        for f in ("orc_export_lplus", "orc_export_lminus"):
            getattr(L, f).argtypes = [C.c_void_p, _i64]
            getattr(L, f).restype = C.c_int64
        L.orc_chebyshev_nodes.argtypes = [C.c_double, C.c_double, C.c_int, _d]
        L.orc_lagrange_eval.argtypes = [_d, C.c_int, C.c_int, C.c_double]
        L.orc_lagrange_eval.restype = C.c_double
        L.orc_transfer_reference.argtypes = [C.c_int, _d]
        L.orc_interp_matrix.argtypes = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_double, C.c_int, _d]
        L.orc_dir_index.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, _d]
        L.orc_dir_vector.argtypes = [C.c_int, C.c_int, C.c_int, _d]
        L.orc_dir_map_vector.argtypes = [C.c_int, C.c_int, _d]
        L.orc_coupling_matrix.argtypes = [C.c_int, C.c_double, _d, C.c_int64, C.c_int64, C.c_int64, _d, _d]
        L.orc_dense_rows.argtypes = [_d, _d, _d, _i64, C.c_int64, _d, _d, _d, C.c_int64, _d, C.c_double, C.c_int, _d]
        L.orc_kernel.argtypes = [_d, C.c_double, _d]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_structure_digest.argtypes = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_int64, _d, _d, C.c_double,
                                           C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                           _i64]
        L.orc_create_sampled.argtypes = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_int64, _d, _d, C.c_double, C.c_int,
                                         C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, _i64, C.c_int64,
                                         C.POINTER(C.c_void_p)]
        _lib = L
    return _lib


def ref():
    """The reference's own C++ (cluster tree + interpolation), or None if not built."""
    global _ref
    if _ref is None:
        build()
        if not os.path.exists(REFLIB):
            return None
        R = C.CDLL(REFLIB)
        R.ref_last_error.restype = C.c_char_p
        R.ref_tree_create.argtypes = [_d, _d, _d, C.c_int64, _d, _d, C.c_int, C.c_int]
        R.ref_tree_create.restype = C.c_void_p
        R.ref_tree_destroy.argtypes = [C.c_void_p]
        R.ref_tree_depth.argtypes = [C.c_void_p]
        R.ref_tree_oversized.argtypes = [C.c_void_p]
        R.ref_tree_level_diameter.argtypes = [C.c_void_p, C.c_int]
        R.ref_tree_level_diameter.restype = C.c_double
        R.ref_tree_export.argtypes = [C.c_void_p, _i64]
        R.ref_tree_export.restype = C.c_int64
        R.ref_tree_perm.argtypes = [C.c_void_p, _i64]
        R.ref_tree_perm.restype = C.c_int64
        R.ref_tree_box.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, _d, _d]
        R.ref_chebyshev_nodes.argtypes = [C.c_double, C.c_double, C.c_int, _d]
        R.ref_lagrange_eval.argtypes = [_d, C.c_int, C.c_int, C.c_double]
        R.ref_lagrange_eval.restype = C.c_double
        R.ref_transfer_reference.argtypes = [C.c_int, _d]
        R.ref_interp_matrix.argtypes = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_double, C.c_int, _d]
        R.ref_directional_diag.argtypes = [_d, _d, _d, _d, C.c_double, C.c_int, _d]
        R.ref_kernel.argtypes = [_d, C.c_double, _d]
        R.ref_kernel_directional.argtypes = [_d, _d, C.c_double, _d]
        R.ref_box_distance.argtypes = [_d, _d, _d, _d]
        R.ref_box_distance.restype = C.c_double
        R.ref_box_diameter.argtypes = [_d, _d]
        R.ref_box_diameter.restype = C.c_double
        _ref = R
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """CPU oracle operator (Alg. 1-4 restated)."""

    def __init__(self, targets, sources, root_lo, root_hi, kappa, n_max=64, m=4, eta2=1.0, l_hf=-2,
                 depth_cap=30, zero_diagonal=0, structure_only=False, sample_leaves=None):
        """sample_leaves: canonical target-leaf indices -> sampled-structure operator
        (orc_create_sampled: partition below those leaves' ancestors only, coupling
        generated per block); only apply_sampled on the same leaves is defined."""
        L = lib()
        self._keep = [_f64(a) for a in (*targets, *sources)]
        tx, ty, tz, sx, sy, sz = self._keep
        lo, hi = _f64(root_lo), _f64(root_hi)
        h = C.c_void_p()
        args = (_p(tx), _p(ty), _p(tz), len(tx), _p(sx), _p(sy), _p(sz), len(sx), _p(lo), _p(hi), float(kappa),
                int(n_max), int(m), float(eta2), int(l_hf), int(depth_cap), int(zero_diagonal))
        if sample_leaves is not None:
            self._lv = np.ascontiguousarray(sample_leaves, dtype=np.int64)
            _chk(L.orc_create_sampled(*args, _pi(self._lv), len(self._lv), C.byref(h)))
        else:
            fn = L.orc_create_structure if structure_only else L.orc_create
            _chk(fn(*args, C.byref(h)))
        self.h = h
        self.nt, self.ns = len(tx), len(sx)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.zeros(self.nt, dtype=np.complex128)
        _chk(lib().orc_apply(self.h, x.view(np.float64).ctypes.data_as(_d), y.view(np.float64).ctypes.data_as(_d)))
        return y

    def apply_sampled(self, x, leaves):
        """Returns (rows, y_rows) for the points of the sampled target leaves."""
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.full(self.nt, np.nan + 0j, dtype=np.complex128)
        lv = np.ascontiguousarray(leaves, dtype=np.int64)
        _chk(lib().orc_apply_sampled(self.h, x.view(np.float64).ctypes.data_as(_d), _pi(lv), len(lv),
                                     y.view(np.float64).ctypes.data_as(_d)))
        rows = np.concatenate([self.leaf_points(0, int(i)) for i in lv]) if len(lv) else np.zeros(0, np.int64)
        return rows, y[rows]

    def set_aca(self, eps):
        """ACA-compressed coupling with tolerance eps (0 = dense)."""
        _chk(lib().orc_set_aca(self.h, float(eps)))

    def aca_ranks(self):
        n = lib().orc_aca_ranks(self.h, None)
        out = np.zeros(n, dtype=np.int32)
        lib().orc_aca_ranks(self.h, out.ctypes.data_as(C.POINTER(C.c_int32)))
        return out

    def last_timing(self):
        """Seconds of the last apply: upward, coupling generation, M2L products,
        downward + near field, and the number of coupling matrices generated."""
        out = np.zeros(5)
        lib().orc_last_timing(self.h, _p(out))
        return dict(zip(("upward", "coupling", "m2l", "down_nf", "keys_generated"), out.tolist()))

    def leaf_count(self, which=0):
        return lib().orc_leaf_count(self.h, which)

    def leaf_points(self, which, leaf):
        cnt = lib().orc_leaf_points(self.h, which, leaf, None, 0)
        out = np.zeros(cnt, dtype=np.int64)
        lib().orc_leaf_points(self.h, which, leaf, _pi(out), cnt)
        return out

    def stats(self):
        out = np.zeros(NSTATS, dtype=np.int64)
        lib().orc_stats(self.h, _pi(out))
        return dict(zip(STAT_NAMES, out.tolist()))

    def _export(self, fn, cols, *args):
        n = fn(self.h, *args, None)
        out = np.zeros((n, cols), dtype=np.int64)
        if n:
            fn(self.h, *args, _pi(out))
        return out

    def tree(self, which):
        return self._export(lib().orc_export_tree, 7, which)

    def perm(self, which):
        n = lib().orc_export_perm(self.h, which, None)
        out = np.zeros(n, dtype=np.int64)
        lib().orc_export_perm(self.h, which, _pi(out))
        return out

    def lplus(self):
        return self._export(lib().orc_export_lplus, 8)

    def lminus(self):
        return self._export(lib().orc_export_lminus, 8)

    def dirsets(self, which):
        return self._export(lib().orc_export_dirsets, 6, which)


def dense_rows(targets, sources, x, kappa, rows, zero_diagonal=0):
    L = lib()
    tx, ty, tz = (_f64(a) for a in targets)
    sx, sy, sz = (_f64(a) for a in sources)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    x = np.ascontiguousarray(x, dtype=np.complex128)
    out = np.zeros(len(rows), dtype=np.complex128)
    _chk(L.orc_dense_rows(_p(tx), _p(ty), _p(tz), _pi(rows), len(rows), _p(sx), _p(sy), _p(sz), len(sx),
                          x.view(np.float64).ctypes.data_as(_d), float(kappa), int(zero_diagonal),
                          out.view(np.float64).ctypes.data_as(_d)))
    return out


def dir_vector(level, l_hf, idx):
    out = np.zeros(3)
    _chk(lib().orc_dir_vector(level, l_hf, idx, _p(out)))
    return out


def dir_map_vector(level, l_hf, v):
    v = _f64(v)
    return lib().orc_dir_map_vector(level, l_hf, _p(v))


def dir_index(level, l_hf, d, rho=(1.0, 1.0, 1.0)):
    r = _f64(rho)
    return lib().orc_dir_index(level, l_hf, int(d[0]), int(d[1]), int(d[2]), _p(r))


def coupling_matrix(m, kappa, side, d, c):
    n = (m + 1) ** 3
    out = np.zeros((n, n), dtype=np.complex128)
    s, cc = _f64(side), _f64(c)
    _chk(lib().orc_coupling_matrix(m, float(kappa), _p(s), int(d[0]), int(d[1]), int(d[2]), _p(cc),
                                   out.view(np.float64).ctypes.data_as(_d)))
    return out


DIGEST_NAMES = ["tree_T", "tree_S", "lplus", "lminus", "dirsets_T", "dirsets_S"]
DIGEST_COUNTS = ["n_c", "n_sc", "n_lminus", "m_d", "nodes_t", "nodes_s", "slots_t", "slots_s", "depth_t", "depth_s",
                 "l_hf"]


def structure_digest(targets, sources, root_lo, root_hi, kappa, n_max=64, eta2=1.0, l_hf=-2, depth_cap=30):
    """Streaming digest of the full structure (orc_structure_digest): 6 uint64 digests
    (DIGEST_NAMES) and the counters (DIGEST_COUNTS), without storing L+."""
    tx, ty, tz = (_f64(a) for a in targets)
    sx, sy, sz = (_f64(a) for a in sources)
    lo, hi = _f64(root_lo), _f64(root_hi)
    out = np.zeros(6, dtype=np.uint64)
    cnt = np.zeros(11, dtype=np.int64)
    _chk(lib().orc_structure_digest(_p(tx), _p(ty), _p(tz), len(tx), _p(sx), _p(sy), _p(sz), len(sx), _p(lo), _p(hi),
                                    float(kappa), int(n_max), 0, float(eta2), int(l_hf), int(depth_cap),
                                    out.ctypes.data_as(C.POINTER(C.c_uint64)), _pi(cnt)))
    return [int(v) for v in out], dict(zip(DIGEST_COUNTS, cnt.tolist()))


def _mix64(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def rows_digest(rows):
    """sum over rows (int64 [n, c]) of the splitmix64 row hash, mod 2^64 -- the
    row digest of orc_structure_digest / fdh_structure_digest, in numpy."""
    rows = np.ascontiguousarray(rows, dtype=np.int64).view(np.uint64)
    with np.errstate(over="ignore"):
        h = np.full(rows.shape[0], 0x12345678, dtype=np.uint64)
        for c in range(rows.shape[1]):
            h = _mix64(h ^ rows[:, c])
        return int(h.sum(dtype=np.uint64))


def export_digest(o):
    """The 6 digests from a full oracle's canonical exports (cross-check of the
    streaming digest)."""
    out = []
    for w in (0, 1):
        perm = o.perm(w)
        pr = np.stack([np.arange(len(perm), dtype=np.int64), perm], axis=1)
        out.append((rows_digest(o.tree(w)) + rows_digest(pr)) % (1 << 64))
    out.append(rows_digest(o.lplus()))
    out.append(rows_digest(o.lminus()))
    out += [rows_digest(o.dirsets(0)), rows_digest(o.dirsets(1))]
    return out


def aca_compress(A, eps, max_rank=None):
    """SPEC.md aca_compress on one complex matrix: returns (U, W) with A ~ U @ W,
    or None when the matrix stays dense (2 k n >= n^2)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    n = A.shape[0]
    U = np.zeros(n * n, dtype=np.complex128)
    W = np.zeros(n * n, dtype=np.complex128)
    k = lib().orc_aca_compress(A.view(np.float64).ctypes.data_as(_d), n, float(eps), int(max_rank or n),
                               U.view(np.float64).ctypes.data_as(_d), W.view(np.float64).ctypes.data_as(_d))
    if k == 0:
        return None
    return U[:n * k].reshape(k, n).T.copy(), W[:n * k].reshape(k, n).copy()


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
