"""fdhelm-b200: B200-native directional multi-level Helmholtz matvec.

Python mirror (ctypes) of the C-ABI in include/fdhelm_c.h, with the reference's
operator vocabulary (setup -> Operator, matvec(op, v) -> g, stats):

    op = DirectionalOperator(targets, sources, root_lo, root_hi, kappa,
                             n_max=64, m=4, eta2=1.0, l_hf=LHF_DEFAULT)
    y = op.apply(x)          # complex128, original point order
    op.stats()               # RunStats counters

The compute path is the CUDA library libfdhelm_b200.so (sm_100a).  There is no
CPU fallback: constructing an operator without the library or without a CUDA
device raises FdhError.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDHELM_LIB") or os.path.join(HERE, "libfdhelm_b200.so")  # override: A/B builds
LHF_DEFAULT = -2

ERR_ARG, ERR_DOMAIN, ERR_DIM, ERR_UNSUPPORTED, ERR_CUDA, ERR_MEMORY = 1, 2, 3, 4, 5, 6
CACHE_NEARFIELD = 1
PHASES = ["h2d", "s2m", "m2m", "m2l", "l2l", "l2t", "p2p", "d2h"]
SYMBOLS = ["fdh_create", "fdh_create_shard", "fdh_create_multi", "fdh_plan_only", "fdh_apply", "fdh_apply_multi",
           "fdh_apply_device", "fdh_sync", "fdh_set_aca", "fdh_set_cache", "fdh_stream",
           "fdh_set_timing", "fdh_get_stats", "fdh_export_tree", "fdh_export_perm", "fdh_export_lplus",
           "fdh_export_lminus", "fdh_export_dirsets", "fdh_export_owned_leaves", "fdh_structure_digest", "fdh_destroy", "fdh_last_error", "fdh_version",
           "fdh_fp64_peak_tflops", "fdh_tensor_peak_tops"]


class FdhStats(C.Structure):
    _fields_ = [("n_le", C.c_int64), ("n_c", C.c_int64), ("n_sc", C.c_int64), ("m_d", C.c_int64),
                ("n_lminus", C.c_int64), ("nf_percent", C.c_double), ("bytes_stored", C.c_int64),
                ("depth_t", C.c_int32), ("depth_s", C.c_int32), ("l_hf", C.c_int32), ("n_pad", C.c_int32),
                ("slots_t", C.c_int64), ("slots_s", C.c_int64), ("nodes_t", C.c_int64), ("nodes_s", C.c_int64),
                ("phase_ms", C.c_double * 8), ("apply_ms", C.c_double), ("setup_ms", C.c_double),
                ("gpu_launches", C.c_int64), ("m2l_flops_executed", C.c_int64), ("m2l_gemm_ms", C.c_double),
                ("timed_applies", C.c_int64), ("m2l_tiles", C.c_int64), ("m2l_items", C.c_int64),
                ("m2l_chunk", C.c_int64), ("shard_cost", C.c_double), ("total_cost", C.c_double),
                ("structure_ms", C.c_double), ("gpu_structure", C.c_int64), ("w_resident", C.c_int64),
                ("w_segments", C.c_int64), ("m2l_impl", C.c_int64), ("m2l_i8_ops", C.c_int64),
                ("nrhs", C.c_int64), ("hbm_bytes", C.c_int64 * 4), ("graph_replays", C.c_int64),
                ("apply_ms_sum", C.c_double), ("applies_collected", C.c_int64), ("aca_eps", C.c_double),
                ("aca_mean_rank", C.c_double), ("aca_bytes", C.c_int64), ("aca_dense_keys", C.c_int64),
                ("nf_cache_bytes", C.c_int64), ("m2l_pair_mode", C.c_int64),
                ("m2l_i8_digits", C.c_int64), ("m2l_i8_bits", C.c_int64),
                ("m2l_i8_products", C.c_int64)]


class FdhError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"fdhelm error {code}: {msg}")
        self.code = code


_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_lib = None


def build(force: bool = False) -> str:
    """Compile libfdhelm_b200.so in-tree (nvcc, sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s", "-j8"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FdhError(ERR_CUDA, f"CUDA extension missing: {LIB_PATH} (run build())")
        L = C.CDLL(LIB_PATH)
        create_args = [_d, _d, _d, C.c_int64, _d, _d, _d, C.c_int64, _d, _d, C.c_double, C.c_int, C.c_int,
                       C.c_double, C.c_int, C.c_int, C.c_int]
        L.fdh_create.argtypes = create_args + [C.c_int, C.POINTER(C.c_void_p)]
        L.fdh_create_shard.argtypes = create_args + [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.fdh_create_multi.argtypes = create_args + [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.fdh_plan_only.argtypes = create_args + [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.fdh_apply.argtypes = [C.c_void_p, _d, _d]
        L.fdh_apply_multi.argtypes = [C.c_void_p, _d, C.c_int64, _d]
        L.fdh_apply_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.fdh_sync.argtypes = [C.c_void_p]
        L.fdh_set_aca.argtypes = [C.c_void_p, C.c_double]
        L.fdh_set_cache.argtypes = [C.c_void_p, C.c_int]
        L.fdh_stream.argtypes = [C.c_void_p]
        L.fdh_stream.restype = C.c_void_p
        L.fdh_set_timing.argtypes = [C.c_void_p, C.c_int]
        L.fdh_get_stats.argtypes = [C.c_void_p, C.POINTER(FdhStats)]
        for f in ("fdh_export_tree", "fdh_export_perm", "fdh_export_dirsets"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, _i64]
            getattr(L, f).restype = C.c_int64
        for f in ("fdh_export_lplus", "fdh_export_lminus", "fdh_export_owned_leaves"):
            getattr(L, f).argtypes = [C.c_void_p, _i64]
            getattr(L, f).restype = C.c_int64
        L.fdh_destroy.argtypes = [C.c_void_p]
        L.fdh_last_error.restype = C.c_char_p
        L.fdh_version.restype = C.c_char_p
        L.fdh_structure_digest.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.fdh_fp64_peak_tflops.argtypes = [C.c_int]
        L.fdh_fp64_peak_tflops.restype = C.c_double
        L.fdh_tensor_peak_tops.argtypes = [C.c_int]
        L.fdh_tensor_peak_tops.restype = C.c_double
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise FdhError(rc, lib().fdh_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class DirectionalOperator:
    """y = A x for A[j,k] = exp(i kappa |x_j - y_k|) / (4 pi |x_j - y_k|).

    Mirrors SPEC.md L4 `setup(T_T, T_S, BlockTree, DirectionTable, kappa, m)`:
    both cluster trees (ClusterTree(points, root, n_max, depth_cap),
    cluster_tree.hpp:47) share the root box; kappa > 0 (WaveNumber,
    geometry.hpp:38-43); eta2 is the admissibility constant of (A1)/(A3);
    l_hf = LHF_DEFAULT selects the default direction sets.
    """

    def __init__(self, targets, sources, root_lo, root_hi, kappa, n_max=64, m=4, eta2=1.0, l_hf=LHF_DEFAULT,
                 depth_cap=30, zero_diagonal=False, rank=0, world=1, plan_only=False, nrhs=1, n_gpus=1):
        L = lib()
        self._keep = [_f64(a) for a in (*targets, *sources)]
        tx, ty, tz, sx, sy, sz = self._keep
        if not (len(tx) == len(ty) == len(tz)) or not (len(sx) == len(sy) == len(sz)):
            raise FdhError(ERR_DIM, "coordinate arrays of one point set differ in length")
        lo, hi = _f64(root_lo), _f64(root_hi)
        p = lambda a: a.ctypes.data_as(_d)  # noqa: E731
        h = C.c_void_p()
        args = (p(tx), p(ty), p(tz), len(tx), p(sx), p(sy), p(sz), len(sx), p(lo), p(hi), float(kappa), int(n_max),
                int(m), float(eta2), int(l_hf), int(depth_cap), int(bool(zero_diagonal)))
        if plan_only:
            _chk(L.fdh_plan_only(*args, int(rank), int(world), C.byref(h)))
        elif nrhs != 1:
            _chk(L.fdh_create_multi(*args, int(rank), int(world), int(nrhs), C.byref(h)))
        elif world > 1:
            _chk(L.fdh_create_shard(*args, int(rank), int(world), C.byref(h)))
        else:
            # n_gpus > 1: one process drives n_gpus devices (shard g on device g, NCCL
            # reduce of y onto device 0 inside the library)
            _chk(L.fdh_create(*args, int(n_gpus), C.byref(h)))
        self.h = h
        self.nt, self.ns = len(tx), len(sx)

    def close(self):
        if getattr(self, "h", None):
            lib().fdh_destroy(self.h)
            self.h = None

    __del__ = close

    # ---- matvec
    def apply(self, x, out=None):
        """Host path: x complex128[N_S] (original order) -> y complex128[N_T]."""
        x = np.ascontiguousarray(x, dtype=np.complex128)
        if x.shape != (self.ns,):
            raise FdhError(ERR_DIM, f"x has shape {x.shape}, expected ({self.ns},)")
        y = out if out is not None else np.empty(self.nt, dtype=np.complex128)
        _chk(lib().fdh_apply(self.h, x.view(np.float64).ctypes.data_as(_d), y.view(np.float64).ctypes.data_as(_d)))
        return y

    matvec = apply

    def apply_multi(self, X, out=None):
        """k right-hand sides: X complex128[k, N_S] (one rhs per row) -> Y[k, N_T]
        (SPEC.md:527 `apply(X[N_S x r])`, stored rhs-major)."""
        X = np.ascontiguousarray(X, dtype=np.complex128)
        if X.ndim != 2 or X.shape[1] != self.ns:
            raise FdhError(ERR_DIM, f"X has shape {X.shape}, expected (k, {self.ns})")
        Y = out if out is not None else np.empty((X.shape[0], self.nt), dtype=np.complex128)
        _chk(lib().fdh_apply_multi(self.h, X.view(np.float64).ctypes.data_as(_d), X.shape[0],
                                   Y.view(np.float64).ctypes.data_as(_d)))
        return Y

    def apply_device(self, x_ptr: int, y_ptr: int, stream: int = 0):
        """Device path: raw device pointers (e.g. torch tensor.data_ptr())."""
        _chk(lib().fdh_apply_device(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(stream or None)))

    def set_aca(self, eps):
        """ACA-compressed coupling (lossy, opt-in): eps > 0 factorises
        the coupling matrices on the device, eps = 0 returns to the exact M2L."""
        _chk(lib().fdh_set_aca(self.h, float(eps)))

    def set_cache(self, nearfield=True):
        """Cache the near-field kernel values for repeated applies (fdh_set_cache,
        SPEC.md:519); False frees the cache."""
        _chk(lib().fdh_set_cache(self.h, CACHE_NEARFIELD if nearfield else 0))

    def sync(self):
        """Wait for the device-path applies; raises their deferred device error
        (singular kernel -> ERR_DOMAIN) if any (fdh_sync)."""
        _chk(lib().fdh_sync(self.h))

    def stream(self) -> int:
        return lib().fdh_stream(self.h) or 0

    def set_timing(self, on=True):
        _chk(lib().fdh_set_timing(self.h, int(on)))

    def stats(self) -> dict:
        s = FdhStats()
        _chk(lib().fdh_get_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in FdhStats._fields_ if f not in ("phase_ms", "hbm_bytes")}
        d["hbm_bytes"] = dict(zip(("s2m", "m2m", "l2l", "l2t"), list(s.hbm_bytes)))
        d["phase_ms"] = dict(zip(PHASES, list(s.phase_ms)))
        return d

    # ---- canonical introspection (identical layout to the oracle's exports)
    def _export(self, fn, cols, *a):
        n = fn(self.h, *a, None)
        out = np.zeros((n, cols), dtype=np.int64)
        if n:
            fn(self.h, *a, out.ctypes.data_as(_i64))
        return out

    def tree(self, which):
        return self._export(lib().fdh_export_tree, 7, which)

    def perm(self, which):
        n = lib().fdh_export_perm(self.h, which, None)
        out = np.zeros(n, dtype=np.int64)
        lib().fdh_export_perm(self.h, which, out.ctypes.data_as(_i64))
        return out

    def lplus(self):
        return self._export(lib().fdh_export_lplus, 8)

    def lminus(self):
        return self._export(lib().fdh_export_lminus, 8)

    def dirsets(self, which):
        return self._export(lib().fdh_export_dirsets, 6, which)

    def owned_leaves(self):
        return self._export(lib().fdh_export_owned_leaves, 6)

    def structure_digest(self):
        out = (C.c_uint64 * 6)()
        _chk(lib().fdh_structure_digest(self.h, out))
        return list(out)


def version() -> str:
    return lib().fdh_version().decode()


def fp64_peak_tflops(kind: int = 0) -> float:
    """Measured FP64 peak on the current device (0: DMMA m8n8k4, 1: DFMA)."""
    return float(lib().fdh_fp64_peak_tflops(kind))


def tensor_peak_tops(kind: int = 0) -> float:
    """Measured int8 tcgen05 dense peak (TOPS) of the current device."""
    return float(lib().fdh_tensor_peak_tops(kind))
