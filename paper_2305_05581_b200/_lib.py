"""ctypes binding of ``lib/libsdmrg_b200.so`` (the C ABI in include/sdmrg_b200.h).

The library is the product: every compute entry point of this package goes
through it.  Loading never falls back to a CPU path — a missing or stale
library raises ``LibraryError`` (and, when nvcc is present, is rebuilt first).
"""

import ctypes
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_dbl = ctypes.POINTER(ctypes.c_double)


class LibraryError(RuntimeError):
    pass


class SdmrgError(RuntimeError):
    """A nonzero status from the C ABI (message from sdmrg_last_error)."""

    def __init__(self, code, msg):
        super().__init__(f"[sdmrg {code}] {msg}")
        self.code = code


class WorkspaceError(SdmrgError, ValueError):
    """SDMRG_EWORKSPACE — mirrors sector_dmrg.sbmm4s.WorkspaceError."""


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("ncomp", c_int), ("nsite", c_int), ("site_qn", P_i32), ("target", P_i32),
        ("nsec_l", c_int), ("qn_l", P_i32), ("dim_l", P_i32), ("left_sign", P_dbl),
        ("nsec_r", c_int), ("qn_r", P_i32), ("dim_r", P_i32),
        ("nops_l", c_int), ("delta_l", P_i32), ("blk_off_l", P_i64), ("kind_l", P_i32),
        ("nops_r", c_int), ("delta_r", P_i32), ("blk_off_r", P_i64), ("kind_r", P_i32),
        ("nrows", c_i64), ("lop", P_i32), ("rop", P_i32), ("alpha", P_dbl), ("e_l", P_i32),
        ("site1_dst", P_i32), ("site1_val", P_dbl), ("site2_dst", P_i32), ("site2_val", P_dbl),
        ("arena_l", c_vp), ("arena_r", c_vp), ("workspace_doubles", c_i64),
        ("rank", c_int), ("world", c_int), ("keep_groups", c_int), ("dry_run", c_int),
    ]


class PlanStats(ctypes.Structure):
    _fields_ = [(name, c_i64) for name in (
        "psi_keys", "psi_size", "groups", "members", "ref_flops", "exec_flops",
        "local_members", "t_problems", "tiles", "segments", "chunks",
        "workspace_doubles", "kernels_per_apply", "algo_bytes", "products",
        "combine_outputs", "combine_terms", "build_ms_taskgen", "build_ms_emit",
        "build_ms_device", "fused_outs", "arena_bytes", "shard_balance_ppm")]

    def as_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


_SIGS = {
    "sdmrg_last_error": (ctypes.c_char_p, []),
    "sdmrg_version": (c_int, []),
    "sdmrg_launch_count": (c_i64, []),
    "sdmrg_dgemm": (c_int, [c_int, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_int, c_vp, c_int,
                            c_dbl, c_vp, c_int, c_vp]),
    "sdmrg_dgemm_strided_batched": (c_int, [c_int, c_int, c_int, c_int, c_int, c_vp, c_int, c_i64,
                                            c_vp, c_int, c_i64, c_vp, c_int, c_i64, c_int, c_vp]),
    "sdmrg_daxpy": (c_int, [c_i64, c_dbl, c_vp, c_vp, c_vp]),
    "sdmrg_sbmm4s": (c_int, [c_int, c_int, c_int, c_int, c_int, c_dbl, c_vp, c_int, c_vp, c_int,
                             c_i64, c_vp, c_int, c_i64, c_vp, c_int, c_vp, c_i64,
                             ctypes.POINTER(c_int), c_vp]),
    "sdmrg_plan_build": (c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(c_vp)]),
    "sdmrg_plan_stats_get": (c_int, [c_vp, ctypes.POINTER(PlanStats)]),
    "sdmrg_plan_layout": (c_int, [c_vp, P_i32, P_i64]),
    "sdmrg_plan_groups": (c_int, [c_vp, P_i32, P_i32, P_i64, P_i64, P_dbl]),
    "sdmrg_plan_shard": (c_int, [c_vp, P_i32]),
    "sdmrg_plan_diagonal": (c_int, [c_vp, c_vp, c_vp]),
    "sdmrg_plan_arena": (c_int, [c_vp, c_int, ctypes.POINTER(c_vp), P_i64, P_i64]),
    "sdmrg_plan_apply": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp]),
    "sdmrg_plan_destroy": (c_int, [c_vp]),
    "sdmrg_plan_invalidate": (c_int, [c_vp]),
    "sdmrg_plan_set_timing": (c_int, [c_vp, c_int]),
    "sdmrg_plan_timing": (c_int, [c_vp, P_dbl, P_i64, P_i64]),
    "sdmrg_dot": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdmrg_nrm2": (c_int, [c_i64, c_vp, c_vp, c_vp]),
    "sdmrg_gemv_t": (c_int, [c_int, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "sdmrg_gemv_n": (c_int, [c_int, c_i64, c_vp, c_i64, c_vp, c_dbl, c_vp, c_vp]),
    "sdmrg_krylov_project": (c_int, [c_int, c_vp, c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdmrg_davidson_precond": (c_int, [c_i64, c_vp, c_vp, c_dbl, c_vp, c_vp]),
    "sdmrg_scal_dev": (c_int, [c_i64, c_vp, c_vp, c_int, c_vp, c_vp]),
    "sdmrg_axpby": (c_int, [c_i64, c_dbl, c_vp, c_dbl, c_vp, c_vp]),
    "sdmrg_rotate": (c_int, [c_i64, P_i64, P_i64, P_i64, P_i64, P_i32, P_i32, P_i32, P_i32,
                             c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sdmrg_rdm_accumulate": (c_int, [c_i64, P_i64, P_i64, P_i32, P_i32, c_vp, c_vp, c_vp]),
    "sdmrg_grouped_gemm": (c_int, [c_int, c_int, c_i64, P_i64, P_i32, P_i32, P_i32, P_i32, P_i64,
                                   P_i64, P_i32, P_i64, P_i32, P_i32, P_dbl,
                                   ctypes.POINTER(c_vp), c_int, c_vp]),
}

EXPORTED = tuple(_SIGS)


def lib_path():
    return os.environ.get("SDMRG_LIB") or _build.LIB


def load(rebuild=True):
    """Load (building first if sources are newer and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if rebuild and not os.environ.get("SDMRG_LIB"):
            try:
                if _build.needs_build():
                    _build.build()
            except RuntimeError:
                if not os.path.exists(path):
                    raise
        if not os.path.exists(path):
            raise LibraryError(f"sm_100a library missing: {path} (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc):
    if rc != 0:
        msg = load().sdmrg_last_error().decode(errors="replace")
        if rc == 3:
            raise WorkspaceError(rc, msg)
        raise SdmrgError(rc, msg)
    return rc


def launch_count():
    return int(load().sdmrg_launch_count())


def ptr(t):
    """Raw device (or host) address of a torch tensor / numpy array / int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def as_p(arr, ctype):
    return arr.ctypes.data_as(ctypes.POINTER(ctype))
