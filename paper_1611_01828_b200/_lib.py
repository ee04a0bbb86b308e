"""ctypes binding of libhsde.so (include/hsde.h).

The shared library is built in-tree (``make -C paper_1611_01828_b200/csrc``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library or
a CUDA device is missing, every product entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import EigenFailure, FactorizationFailure, TauZero

LIB_PATH = Path(__file__).resolve().parent / "libhsde.so"

HSDE_OK, HSDE_ERR_CUDA, HSDE_ERR_EIGEN, HSDE_ERR_FACTOR, HSDE_ERR_ARG, HSDE_ERR_TAUZERO = range(6)
HSDE_FLAG_EXACT_UY = 1
HSDE_FLAG_NO_FACTOR = 2
HSDE_FLAG_COLD_EIG = 4
HSDE_FLAG_NO_SPLIT = 8
HSDE_FLAG_JACOBI = 16
HSDE_STATS_LEN = 14
HSDE_CHECK_LEN = 8
HSDE_CERT_LEN = 7
HSDE_PROFILE_SLOTS = 16

EXPORTED = (
    "hsde_create", "hsde_destroy", "hsde_last_error", "hsde_info", "hsde_set_state",
    "hsde_get_state", "hsde_reset_state", "hsde_iterate", "hsde_check", "hsde_certificate",
    "hsde_affine_project", "hsde_solve_inner", "hsde_project_cone", "hsde_residuals",
    "hsde_get_minv_zeta", "hsde_time_iterations", "hsde_profile_iterations",
    "hsde_profile_name", "hsde_sync", "hsde_set_alpha", "hsde_stats", "hsde_create_sharded",
    "hsde_nccl_unique_id", "hsde_shard_total", "hsde_set_state_shard", "hsde_get_state_shard",
    "hsde_debug_jacobi", "hsde_pattern_decompose", "hsde_pattern_sizes", "hsde_pattern_cliques",
    "hsde_pattern_fill", "hsde_pattern_destroy", "hsde_sdpa_parse", "hsde_sdpa_error",
    "hsde_sdpa_sizes", "hsde_sdpa_data", "hsde_sdpa_destroy", "hsde_pattern_index", "hsde_report_vectors",
    "hsde_cover_build", "hsde_cover_fill", "hsde_cover_destroy",
)
HSDE_NCCL_ID_BYTES = 128

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class ProblemDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("m", C.c_int32), ("n_c", C.c_int32), ("p", C.c_int32),
        ("n_d", C.c_int64), ("nnz", C.c_int64),
        ("a_row_ptr", _i64p), ("a_col", _i32p), ("a_val", _dp),
        ("c", _dp), ("b", _dp),
        ("clique_offsets", _i64p), ("clique_sizes", _i32p), ("slot_cov", _i32p),
        ("cover_counts", _dp), ("owned", C.POINTER(C.c_uint8)), ("n_sep", C.c_int32),
        ("n_sep_local", C.c_int32), ("sep_local", _i32p), ("sep_pos", _i32p),
        ("follower", C.c_int32),
    ]


class Comm(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("nccl_id", C.c_uint8 * 128)]


class Settings(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("tol", C.c_double), ("infeas_tau_tol", C.c_double),
        ("infeas_kappa_tol", C.c_double), ("check_interval", C.c_int32),
        ("normalize", C.c_int32), ("device", C.c_int32), ("flags", C.c_int32),
    ]


class Info(C.Structure):
    _fields_ = [
        ("total", C.c_int64), ("n_c", C.c_int32), ("m", C.c_int32), ("p", C.c_int32),
        ("n_d", C.c_int64), ("nnz", C.c_int64), ("sigma_c", C.c_double),
        ("sigma_b", C.c_double), ("zeta_scale", C.c_double), ("schur_diagonal", C.c_int32),
        ("max_clique", C.c_int32), ("n_shards", C.c_int32), ("mode", C.c_int32),
        ("half_passes", C.c_int32), ("reserved", C.c_int32),
    ]


_LIB = None


def load() -> C.CDLL:
    """Load libhsde.so (fail loudly: there is no fallback path)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C paper_1611_01828_b200/csrc` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    sig = {
        "hsde_create": (C.c_int, [C.POINTER(ProblemDesc), C.POINTER(Settings), C.POINTER(vp)]),
        "hsde_destroy": (None, [vp]),
        "hsde_last_error": (C.c_char_p, [vp]),
        "hsde_info": (C.c_int, [vp, C.POINTER(Info)]),
        "hsde_set_state": (C.c_int, [vp, _dp, _dp]),
        "hsde_get_state": (C.c_int, [vp, _dp, _dp]),
        "hsde_reset_state": (C.c_int, [vp]),
        "hsde_iterate": (C.c_int, [vp, C.c_int32]),
        "hsde_check": (C.c_int, [vp, _dp]),
        "hsde_certificate": (C.c_int, [vp, _dp]),
        "hsde_affine_project": (C.c_int, [vp, _dp, _dp]),
        "hsde_solve_inner": (C.c_int, [vp, _dp, _dp]),
        "hsde_project_cone": (C.c_int, [vp, _dp, _dp]),
        "hsde_residuals": (C.c_int, [vp, _dp, _dp]),
        "hsde_get_minv_zeta": (C.c_int, [vp, _dp]),
        "hsde_time_iterations": (C.c_int, [vp, C.c_int32, C.POINTER(C.c_float)]),
        "hsde_profile_iterations": (C.c_int, [vp, C.c_int32, C.POINTER(C.c_float), _i32p]),
        "hsde_profile_name": (C.c_char_p, [C.c_int32]),
        "hsde_sync": (C.c_int, [vp]),
        "hsde_set_alpha": (C.c_int, [vp, C.c_double]),
        "hsde_stats": (C.c_int, [vp, _dp]),
        "hsde_create_sharded": (C.c_int, [C.POINTER(ProblemDesc), C.c_int32, C.POINTER(Settings),
                                          C.POINTER(Comm), C.POINTER(vp)]),
        "hsde_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "hsde_shard_total": (C.c_int, [vp, C.c_int32, C.POINTER(C.c_int64)]),
        "hsde_set_state_shard": (C.c_int, [vp, C.c_int32, _dp, _dp]),
        "hsde_get_state_shard": (C.c_int, [vp, C.c_int32, _dp, _dp]),
        "hsde_debug_jacobi": (C.c_int, [vp, C.c_int32, _dp]),
        "hsde_pattern_decompose": (C.c_int, [C.c_int32, C.c_int64, _i32p, _i32p, C.c_int32,
                                             C.POINTER(vp)]),
        "hsde_pattern_sizes": (C.c_int, [vp, _i64p, _i64p, _i64p, _i32p]),
        "hsde_pattern_cliques": (C.c_int, [vp, _i64p, _i32p]),
        "hsde_pattern_fill": (C.c_int, [vp, _i32p, _i32p]),
        "hsde_pattern_destroy": (None, [vp]),
        "hsde_sdpa_parse": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(vp)]),
        "hsde_sdpa_error": (C.c_char_p, [_i64p, _i32p]),
        "hsde_sdpa_sizes": (C.c_int, [vp, _i32p, _i32p, _i64p]),
        "hsde_sdpa_data": (C.c_int, [vp, _i32p, _dp, _i32p, _i32p, _i32p, _i32p, _dp]),
        "hsde_sdpa_destroy": (None, [vp]),
        "hsde_report_vectors": (C.c_int, [vp, C.c_double, _dp, _dp, _dp]),
        "hsde_cover_build": (C.c_int, [C.c_int64, _dp, _i64p, C.c_int64, _i32p, _i64p, C.c_int64,
                                       C.POINTER(vp), _i64p]),
        "hsde_cover_fill": (C.c_int, [vp, _dp, _i64p, C.c_int64, _i32p, _i64p, C.c_int64, _i64p, _dp,
                                      _i32p, _i32p]),
        "hsde_cover_destroy": (None, [vp]),
        "hsde_pattern_index": (C.c_int, [_i64p, C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p, C.c_int32,
                                         _i64p, _i64p, _i64p, _i64p, C.POINTER(C.c_uint8)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def raise_for(rc: int, msg: str):
    if rc == HSDE_OK:
        return
    if rc == HSDE_ERR_EIGEN:
        raise EigenFailure(msg)
    if rc == HSDE_ERR_FACTOR:
        raise FactorizationFailure(msg)
    if rc == HSDE_ERR_TAUZERO:
        raise TauZero(msg)
    if rc == HSDE_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"libhsde CUDA error: {msg}")


class Handle:
    """Owns one device-resident problem + ADMM state (one hsde_t)."""

    def __init__(self, cp, *, alpha=1.6, tol=1e-4, infeas_tau_tol=1e-9, infeas_kappa_tol=1e-6,
                 check_interval=20, normalize=True, device=0, flags=0, shards=None, comm=None):
        """One problem on one device (`cp`), or sharded (`shards`, list of
        paper_1611_01828_b200.shard.Shard): all shards emulated on this device
        (comm None) or this rank's single shard with an NCCL communicator
        (comm = (world, rank, nccl_id bytes))."""
        lib = load()
        self._lib = lib
        self.cp = cp
        keep = []
        parts = shards if shards is not None else [None]
        descs = (ProblemDesc * len(parts))()
        for i, sh in enumerate(parts):
            self._fill_desc(descs[i], cp if sh is None else sh.problem, sh, keep)
        st = Settings(alpha=alpha, tol=tol, infeas_tau_tol=infeas_tau_tol,
                      infeas_kappa_tol=infeas_kappa_tol, check_interval=check_interval,
                      normalize=1 if normalize else 0, device=device, flags=flags)
        cm = None
        if comm is not None:
            cm = Comm(world=int(comm[0]), rank=int(comm[1]))
            C.memmove(cm.nccl_id, bytes(comm[2]), HSDE_NCCL_ID_BYTES)
        h = C.c_void_p()
        rc = lib.hsde_create_sharded(descs, len(parts), C.byref(st),
                                     C.byref(cm) if cm is not None else None, C.byref(h))
        if rc != HSDE_OK:
            raise_for(rc, lib.hsde_last_error(None).decode())
        self._h = h
        del keep  # the library copied everything
        inf = Info()
        lib.hsde_info(h, C.byref(inf))
        self.n_shards = int(inf.n_shards)
        self.mode = int(inf.mode)
        self.totals = []
        for g in range(self.n_shards):
            t = C.c_int64()
            lib.hsde_shard_total(h, g, C.byref(t))
            self.totals.append(int(t.value))
        self.total = self.totals[0]
        self.sigma_c = float(inf.sigma_c)
        self.sigma_b = float(inf.sigma_b)
        self.zeta_scale = float(inf.zeta_scale)
        self.schur_diagonal = bool(inf.schur_diagonal)
        self.max_clique = int(inf.max_clique)
        self.half_passes = bool(inf.half_passes)
        self.alpha = alpha

    @staticmethod
    def _fill_desc(desc, cp, sh, keep):
        A = cp.A
        arrs = {
            "rp": np.ascontiguousarray(A.indptr, dtype=np.int64),
            "col": np.ascontiguousarray(A.indices, dtype=np.int32),
            "val": np.ascontiguousarray(A.data, dtype=np.float64),
            "c": np.ascontiguousarray(cp.c, dtype=np.float64),
            "b": np.ascontiguousarray(cp.b, dtype=np.float64),
            "off": np.ascontiguousarray(cp.offsets, dtype=np.int64),
            "sz": np.ascontiguousarray(cp.sizes, dtype=np.int32),
            "sc": np.ascontiguousarray(cp.slot_cov, dtype=np.int32),
        }
        keep.append(arrs)
        desc.n, desc.m, desc.n_c, desc.p = cp.n, cp.m, cp.N_c, cp.p
        desc.n_d, desc.nnz = cp.n_d, int(A.nnz)
        desc.a_row_ptr = _ptr(arrs["rp"], C.c_int64)
        desc.a_col = _ptr(arrs["col"], C.c_int32)
        desc.a_val = _ptr(arrs["val"], C.c_double)
        desc.c = _ptr(arrs["c"], C.c_double)
        desc.b = _ptr(arrs["b"], C.c_double)
        desc.clique_offsets = _ptr(arrs["off"], C.c_int64)
        desc.clique_sizes = _ptr(arrs["sz"], C.c_int32)
        desc.slot_cov = _ptr(arrs["sc"], C.c_int32)
        if sh is not None:
            arrs["D"] = np.ascontiguousarray(sh.D, dtype=np.float64)
            arrs["own"] = np.ascontiguousarray(sh.owned, dtype=np.uint8)
            arrs["sl"] = np.ascontiguousarray(sh.sep_local, dtype=np.int32)
            arrs["sp"] = np.ascontiguousarray(sh.sep_pos, dtype=np.int32)
            desc.cover_counts = _ptr(arrs["D"], C.c_double)
            desc.owned = _ptr(arrs["own"], C.c_uint8)
            desc.n_sep = int(sh.n_sep)
            desc.n_sep_local = int(arrs["sl"].size)
            desc.sep_local = _ptr(arrs["sl"], C.c_int32)
            desc.sep_pos = _ptr(arrs["sp"], C.c_int32)
            desc.follower = 0 if sh.rank == 0 else 1

    # -- plumbing -------------------------------------------------------------
    def _rc(self, rc):
        if rc != HSDE_OK:
            raise_for(rc, self._lib.hsde_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.hsde_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _vec(self, a, n=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if n is not None and a.shape != (n,):
            raise ValueError(f"expected length {n}, got {a.shape}")
        return a

    # -- state -----------------------------------------------------------------
    def set_alpha(self, alpha: float):
        if alpha != self.alpha:
            self._rc(self._lib.hsde_set_alpha(self._h, float(alpha)))
            self.alpha = alpha

    def set_state(self, u, w):
        u = self._vec(u, self.total)
        w = self._vec(w, self.total)
        self._rc(self._lib.hsde_set_state(self._h, _ptr(u, C.c_double), _ptr(w, C.c_double)))

    def get_state(self, shard: int = 0):
        u = np.empty(self.totals[shard])
        w = np.empty(self.totals[shard])
        self._rc(self._lib.hsde_get_state_shard(self._h, shard, _ptr(u, C.c_double),
                                                _ptr(w, C.c_double)))
        return u, w

    def report_vectors(self, tau: float):
        """(u_x, u_y, H'((u_v / sigma_c) / tau)) for the report (single shard)."""
        x = np.empty(self.cp.N_c)
        y = np.empty(self.cp.m)
        hv = np.empty(self.cp.N_c)
        self._rc(self._lib.hsde_report_vectors(self._h, float(tau), _ptr(x, C.c_double),
                                               _ptr(y, C.c_double), _ptr(hv, C.c_double)))
        return x, y, hv

    def get_u(self, shard: int = 0):
        """u alone (the report needs no w)."""
        u = np.empty(self.totals[shard])
        self._rc(self._lib.hsde_get_state_shard(self._h, shard, _ptr(u, C.c_double), None))
        return u

    def set_state_shard(self, shard: int, u, w):
        u = self._vec(u, self.totals[shard])
        w = self._vec(w, self.totals[shard])
        self._rc(self._lib.hsde_set_state_shard(self._h, shard, _ptr(u, C.c_double),
                                                _ptr(w, C.c_double)))

    def reset_state(self):
        self._rc(self._lib.hsde_reset_state(self._h))

    def iterate(self, k: int):
        self._rc(self._lib.hsde_iterate(self._h, int(k)))

    def sync(self):
        self._rc(self._lib.hsde_sync(self._h))

    def check(self) -> np.ndarray:
        out = np.empty(HSDE_CHECK_LEN)
        self._rc(self._lib.hsde_check(self._h, _ptr(out, C.c_double)))
        return out

    def certificate(self) -> np.ndarray:
        out = np.empty(HSDE_CERT_LEN)
        self._rc(self._lib.hsde_certificate(self._h, _ptr(out, C.c_double)))
        return out

    # -- unit-level -----------------------------------------------------------------
    def affine_project(self, w):
        w = self._vec(w, self.total)
        u = np.empty(self.total)
        self._rc(self._lib.hsde_affine_project(self._h, _ptr(w, C.c_double), _ptr(u, C.c_double)))
        return u

    def solve_inner(self, w12):
        w12 = self._vec(w12, self.total - 1)
        u = np.empty(self.total - 1)
        self._rc(self._lib.hsde_solve_inner(self._h, _ptr(w12, C.c_double), _ptr(u, C.c_double)))
        return u

    def project_cone(self, v):
        v = self._vec(v, self.total)
        out = np.empty(self.total)
        self._rc(self._lib.hsde_project_cone(self._h, _ptr(v, C.c_double), _ptr(out, C.c_double)))
        return out

    def residuals(self, u):
        u = self._vec(u, self.total)
        out = np.empty(3)
        self._rc(self._lib.hsde_residuals(self._h, _ptr(u, C.c_double), _ptr(out, C.c_double)))
        return out

    def minv_zeta(self):
        out = np.empty(self.total - 1)
        self._rc(self._lib.hsde_get_minv_zeta(self._h, _ptr(out, C.c_double)))
        return out

    def stats(self) -> dict:
        out = np.empty(HSDE_STATS_LEN)
        self._rc(self._lib.hsde_stats(self._h, _ptr(out, C.c_double)))
        return {"mean_sweeps": float(out[0]), "max_sweeps": float(out[1]),
                "mean_sweeps_large": float(out[2]), "warm_start": bool(out[3]),
                "split_done": float(out[4]), "split_handoff": float(out[5]),
                "split_fp_iters": float(out[6]), "handoff_off": float(out[7]), "handoff_rn": float(out[8]),
                "handoff_stall": float(out[9]), "split_resumed": float(out[10]),
                "handoff_refresh": float(out[11]), "cold_done": float(out[12]), "cold_failed": float(out[13])}

    def debug_jacobi(self, clique: int = 0) -> np.ndarray:
        out = np.empty(64)
        self._rc(self._lib.hsde_debug_jacobi(self._h, int(clique), _ptr(out, C.c_double)))
        return out

    # -- measurement ---------------------------------------------------------------------
    def time_iterations(self, k: int) -> float:
        ms = C.c_float()
        self._rc(self._lib.hsde_time_iterations(self._h, int(k), C.byref(ms)))
        return float(ms.value)

    def profile_iterations(self, k: int):
        ms = (C.c_float * HSDE_PROFILE_SLOTS)()
        nl = C.c_int32()
        self._rc(self._lib.hsde_profile_iterations(self._h, int(k), ms, C.byref(nl)))
        out = {}
        for i in range(HSDE_PROFILE_SLOTS):
            name = self._lib.hsde_profile_name(i).decode()
            if name:
                out[name] = float(ms[i])
        return out, int(nl.value)


def nccl_unique_id() -> bytes:
    lib = load()
    buf = (C.c_uint8 * HSDE_NCCL_ID_BYTES)()
    rc = lib.hsde_nccl_unique_id(buf)
    if rc != HSDE_OK:
        raise_for(rc, lib.hsde_last_error(None).decode())
    return bytes(buf)


def exported_symbols() -> list[str]:
    """Symbols include/hsde.h declares (checked by the CPU tests)."""
    return list(EXPORTED)


def device_count() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def default_device() -> int:
    return int(os.environ.get("HSDE_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def cover_layout(n2: int, c_full: np.ndarray, gather_index: np.ndarray, a_col: np.ndarray):
    """(covered, c on covered, rank of A's column ids, rank of the gather index) of a
    reference-layout problem (library, host threads; hsde_cover_*)."""
    lib = load()
    cf = np.ascontiguousarray(c_full, dtype=np.float64)
    gi = np.ascontiguousarray(gather_index, dtype=np.int64)
    col = np.ascontiguousarray(a_col)
    if col.dtype == np.int32:
        c32, c64 = _ptr(col, C.c_int32), None
    else:
        col = np.ascontiguousarray(col, dtype=np.int64)
        c32, c64 = None, _ptr(col, C.c_int64)
    h = C.c_void_p()
    ncov = C.c_int64()
    rc = lib.hsde_cover_build(int(n2), _ptr(cf, C.c_double), _ptr(gi, C.c_int64), gi.size, c32, c64, col.size,
                              C.byref(h), C.byref(ncov))
    if rc:
        raise ValueError("hsde_cover_build: a coordinate id outside [0, n^2)")
    try:
        covered = np.empty(ncov.value, dtype=np.int64)
        c_cov = np.empty(ncov.value, dtype=np.float64)
        pos = np.empty(col.size, dtype=np.int32)
        slot_cov = np.empty(gi.size, dtype=np.int32)
        rc = lib.hsde_cover_fill(h, _ptr(cf, C.c_double), _ptr(gi, C.c_int64), gi.size, c32, c64, col.size,
                                 _ptr(covered, C.c_int64), _ptr(c_cov, C.c_double), _ptr(pos, C.c_int32),
                                 _ptr(slot_cov, C.c_int32))
        if rc:
            raise ValueError("hsde_cover_fill: bad arguments")
    finally:
        lib.hsde_cover_destroy(h)
    return covered, c_cov, pos, slot_cov


def pattern_index(covered: np.ndarray, n: int, code: np.ndarray, starts: np.ndarray):
    """(block, i, j, pos_c, hit) of the report's pattern rows (library, host; O(N))."""
    cov = np.ascontiguousarray(covered, dtype=np.int64)
    cd = np.ascontiguousarray(code, dtype=np.int64)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    outs = [np.empty(cd.size, dtype=np.int64) for _ in range(4)]
    hit = np.empty(cd.size, dtype=np.uint8)
    rc = load().hsde_pattern_index(_ptr(cov, C.c_int64), cov.size, int(n), _ptr(cd, C.c_int64), cd.size,
                                   _ptr(st, C.c_int64), st.size - 1, *[_ptr(o, C.c_int64) for o in outs],
                                   _ptr(hit, C.c_uint8))
    if rc:
        raise ValueError("hsde_pattern_index: bad arguments")
    return outs[0], outs[1], outs[2], outs[3], hit.view(bool)
