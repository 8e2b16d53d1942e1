"""ctypes binding of libmdd.so (the C-ABI declared in include/mdd.h).

The shared library is built in-tree (``python -m paper_1711_03789_b200.build``)
and is the only compute path: there is no CPU fallback.  Importing this
module on a machine without the library raises immediately; creating a
context without a GPU raises ``RuntimeError`` from ``mdd_ctx_create``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDD_LIB_PATH") or os.path.join(_HERE, "libmdd.so")

MDD_OK, MDD_EINVAL, MDD_ESINGULAR, MDD_ECAP, MDD_ECUDA, MDD_ENCCL, MDD_ENOMEM, MDD_EDECOMP = range(8)


class mdd_complex(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class mdd_coeffs(C.Structure):
    _fields_ = [
        ("k", C.c_double),
        ("xi", C.c_double),
        ("eps", C.POINTER(C.c_double)),
        ("mu", C.POINTER(C.c_double)),
        ("sigma", C.POINTER(C.c_double)),
        ("eps0", C.c_double),
        ("mu0", C.c_double),
        ("sigma0", C.c_double),
        ("homogeneous", C.c_int),
    ]


class mdd_prec_desc(C.Structure):
    _fields_ = [
        ("family", C.c_int),
        ("levels", C.c_int),
        ("correction", C.c_int),
        ("lu_cap", C.c_int64),
        ("leaf_size", C.c_int),
        ("A_prec", C.c_void_p),
        ("A_corr", C.c_void_p),
        ("nsub", C.c_int32),
        ("sub_ptr", C.POINTER(C.c_int64)),
        ("sub_dofs", C.POINTER(C.c_int64)),
        ("sub_pou", C.POINTER(C.c_double)),
        ("dof_xyz", C.POINTER(C.c_int32)),
        ("space", C.c_void_p),
        ("prec_coeffs", C.POINTER(mdd_coeffs)),
        ("sub_tet_ptr", C.POINTER(C.c_int64)),
        ("sub_tets", C.POINTER(C.c_int64)),
        ("sub_bface_ptr", C.POINTER(C.c_int64)),
        ("sub_bfaces", C.POINTER(C.c_int64)),
        ("R0", C.c_void_p),
        ("coarse_space", C.c_void_p),
        ("tet_map", C.POINTER(C.c_int64)),
        ("coarse_dof_xyz", C.POINTER(C.c_int32)),
        ("nbf_global", C.c_int64),
        ("bfaces_global", C.POINTER(C.c_int64)),
        ("dof_grid", C.c_int32),
    ]


HOST_OP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(mdd_complex), C.POINTER(mdd_complex))


class mdd_gmres_cfg(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("maxit", C.c_int32),
        ("side", C.c_int32),
        ("check_drift", C.c_int32),
        ("keep_basis", C.c_int32),
        ("device_io", C.c_int32),
        ("ortho", C.c_int32),
    ]


class mdd_gmres_ops(C.Structure):
    _fields_ = [
        ("A", C.c_void_p),
        ("a_fn", HOST_OP),
        ("a_user", C.c_void_p),
        ("P", C.c_void_p),
        ("m_fn", HOST_OP),
        ("m_user", C.c_void_p),
        ("Mcsr", C.c_void_p),
        ("D", C.c_void_p),
    ]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_i64 = C.c_int64
_i32 = C.c_int32
_pd = C.POINTER(C.c_double)
_pz = C.POINTER(mdd_complex)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)

# name -> (restype, argtypes); mirrors include/mdd.h one-to-one
SIGNATURES = {
    "mdd_last_error": (C.c_char_p, []),
    "mdd_version": (C.c_int, []),
    "mdd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "mdd_ctx_create": (C.c_int, [C.c_int, _PP]),
    "mdd_ctx_destroy": (None, [_P]),
    "mdd_ctx_synchronize": (C.c_int, [_P]),
    "mdd_ctx_kernel_launches": (C.c_int64, [_P]),
    "mdd_ctx_timers": (C.c_int, [_P, _pd]),
    "mdd_ctx_set_timing": (C.c_int, [_P, C.c_int]),
    "mdd_ctx_event_record": (C.c_int, [_P, C.c_int]),
    "mdd_ctx_event_elapsed": (C.c_int, [_P, C.c_int, C.c_int, _pd]),
    "mdd_dev_alloc": (C.c_int, [_P, _i64, _PP]),
    "mdd_dev_free": (C.c_int, [_P, C.c_void_p]),
    "mdd_memcpy": (C.c_int, [_P, C.c_void_p, C.c_void_p, _i64, C.c_int]),
    "mdd_csr_from_host": (C.c_int, [_P, _i64, _i64, _i64, _pi32, _pi32, C.c_void_p, C.c_int, _PP]),
    "mdd_csr_info": (C.c_int, [_P, _pi64, _pi64, _pi64, C.POINTER(C.c_int)]),
    "mdd_csr_to_host": (C.c_int, [_P, _pi32, _pi32, C.c_void_p]),
    "mdd_csr_destroy": (None, [_P]),
    "mdd_spmv": (C.c_int, [_P, _P, _pz, _pz]),
    "mdd_spmv_bench": (C.c_int, [_P, _P, C.c_int, _pd]),
    "mdd_space_create": (
        C.c_int,
        [_P, _i32, _i64, _pd, _i64, _pi64, _pi64, _pi64, _i64, _pi64, _i64, _PP],
    ),
    "mdd_space_destroy": (None, [_P]),
    "mdd_space_nnz": (C.c_int, [_P, _pi64]),
    "mdd_space_set_row_window": (C.c_int, [_P, _i64, _i64]),
    "mdd_assemble": (
        C.c_int,
        [_P, C.POINTER(mdd_coeffs), C.c_int, _i64, _pi64, _PP, _PP, _PP, _PP, _PP],
    ),
    "mdd_assemble_rhs": (C.c_int, [_P, _pz, _pz]),
    "mdd_assemble_rhs_gaussian": (C.c_int, [_P, _pd, C.c_double, C.c_double, _pd, _pz]),
    "mdd_element_matrices": (C.c_int, [_P, _i64, _pd, _pd, _pd, _pd, _pd]),
    "mdd_space2_create": (
        C.c_int,
        [_P, _i32, _i64, _pd, _i64, _pi64, _pi64, _i64, _i32, _pd, _pd, _PP],
    ),
    "mdd_element2_matrices": (C.c_int, [_P, _i64, _pd, _pd, _pd]),
    "mdd_free": (None, [C.c_void_p]),
    "mdd_prec_symmetric": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "mdd_extend_overlap": (
        C.c_int,
        [_i32, _i64, _pi64, _i32, _pi64, _pi64, _i32, C.POINTER(_pi64), C.POINTER(_pi64)],
    ),
    "mdd_subdomain_dofs": (
        C.c_int,
        [_i32, _i64, _pi64, _pi64, _i64, _pi64, _i64, _pi64, _i64, _pi64, _i64, _i32, _pi64, _pi64,
         C.POINTER(_pi64), C.POINTER(_pi64)],
    ),
    "mdd_nesting_map": (C.c_int, [_i32, _pd, _pi64, _i32, _pd, _pi64, C.c_double, _pi64]),
    "mdd_coarse_restriction": (
        C.c_int,
        [_i64, _pd, _i64, _pi64, _pi64, _i64, _pi64, _pd, _i64, _pi64, _pi64, _pi64, _pi64, _i64, _pi64,
         C.c_double, C.POINTER(_pi64), C.POINTER(_pi64), C.POINTER(_pd), _pi64],
    ),
    "mdd_prec_create": (C.c_int, [_P, C.POINTER(mdd_prec_desc), _PP, _pi32]),
    "mdd_prec_variant": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, _PP]),
    "mdd_prec_destroy": (None, [_P]),
    "mdd_prec_apply": (C.c_int, [_P, _pz, _pz]),
    "mdd_prec_coarse_apply": (C.c_int, [_P, _pz, _pz]),
    "mdd_prec_stats": (C.c_int, [_P, _pd]),
    "mdd_prec_flop_counts": (C.c_int, [_P, _pd]),
    "mdd_prec_apply_bench": (C.c_int, [_P, C.c_int, C.c_int, _pd]),
    "mdd_comm_unique_id": (C.c_int, [C.c_char_p]),
    "mdd_comm_create": (C.c_int, [_P, C.c_int, C.c_int, C.c_char_p, _PP]),
    "mdd_comm_loopback_group": (C.c_int, [C.c_int, _PP]),
    "mdd_comm_loopback_group_free": (None, [_P]),
    "mdd_comm_create_loopback": (C.c_int, [_P, _P, C.c_int, _PP]),
    "mdd_comm_destroy": (None, [_P]),
    "mdd_comm_abort": (C.c_int, [_P]),
    "mdd_comm_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mdd_prec_local_matrix_size": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "mdd_prec_local_matrix": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _P]),
    "mdd_prec_pivot_ratio": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mdd_prec_set_comm": (C.c_int, [_P, _P]),
    "mdd_prec_set_halo": (C.c_int, [_P, C.c_int64, C.c_int64]),
    "mdd_prec_halo_info": (C.c_int, [_P] + [C.POINTER(C.c_int64)] * 5),
    "mdd_prec_refactor": (C.c_int, [_P, _P, C.POINTER(mdd_coeffs)]),
    "mdd_gmres": (
        C.c_int,
        [
            _P,
            C.POINTER(mdd_gmres_ops),
            _i64,
            _pz,
            _pz,
            C.POINTER(mdd_gmres_cfg),
            _pz,
            _pd,
            _pd,
            _pz,
            _pi32,
            _pi32,
            _pd,
        ],
    ),
}


def _load():
    if not os.path.exists(LIB_PATH):
        # build the native library in-tree (nvcc); there is no CPU fallback
        try:
            import importlib.util

            spec = importlib.util.spec_from_file_location("_mdd_build", os.path.join(os.path.dirname(LIB_PATH),
                                                                                      "build.py"))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            mod.build()
        except Exception as exc:  # noqa: BLE001
            raise ImportError(
                f"{LIB_PATH} is missing and could not be built ({exc}): build it with "
                "`python paper_1711_03789_b200/build.py` (the package has no CPU fallback)"
            ) from exc
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class MddError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int):
    if rc != MDD_OK:
        msg = lib.mdd_last_error().decode("utf-8", "replace")
        raise MddError(rc, msg)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def zptr(a: np.ndarray):
    assert a.dtype == np.complex128 and a.flags.c_contiguous
    return a.ctypes.data_as(_pz)


# ------------------------------------------------------------------ context
class Context:
    """One CUDA device + stream (opaque ``mdd_ctx``)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.mdd_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def synchronize(self):
        check(lib.mdd_ctx_synchronize(self.handle))

    def kernel_launches(self) -> int:
        return int(lib.mdd_ctx_kernel_launches(self.handle))

    def set_timing(self, on: bool):
        check(lib.mdd_ctx_set_timing(self.handle, 1 if on else 0))

    def record(self, slot: int):
        check(lib.mdd_ctx_event_record(self.handle, slot))

    def elapsed_ms(self, s0: int, s1: int) -> float:
        ms = C.c_double()
        check(lib.mdd_ctx_event_elapsed(self.handle, s0, s1, C.byref(ms)))
        return ms.value

    def timers(self):
        out = (C.c_double * 8)()
        check(lib.mdd_ctx_timers(self.handle, out))
        return list(out)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            lib.mdd_ctx_destroy(h)
            self.handle = None


_ctx = None
_ctx_lock = threading.Lock()


def device_count() -> int:
    n = C.c_int(0)
    check(lib.mdd_device_count(C.byref(n)))
    return n.value


_thread_ctx = threading.local()


class use_context:
    """``with use_context(ctx):`` — calls made by this thread use ``ctx``
    instead of the process-wide default (one context per thread, e.g. the
    loopback ranks of tests/test_gpu_distributed.py)."""

    def __init__(self, ctx: "Context"):
        self.ctx = ctx

    def __enter__(self):
        self.prev = getattr(_thread_ctx, "ctx", None)
        _thread_ctx.ctx = self.ctx
        return self.ctx

    def __exit__(self, *exc):
        _thread_ctx.ctx = self.prev


def get_context() -> Context:
    """The calling thread's context (:class:`use_context`), else the
    process-wide default context on ``LOCAL_RANK`` (or device 0)."""
    local = getattr(_thread_ctx, "ctx", None)
    if local is not None:
        return local
    global _ctx
    with _ctx_lock:
        if _ctx is None:
            _ctx = Context(int(os.environ.get("MDD_DEVICE", os.environ.get("LOCAL_RANK", "0"))))
        return _ctx


class DeviceBuffer:
    """Raw device allocation (benchmark plumbing: device-resident inputs)."""

    def __init__(self, ctx: Context, nbytes: int):
        self.ctx = ctx
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        check(lib.mdd_dev_alloc(ctx.handle, self.nbytes, C.byref(p)))
        self.ptr = p

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        check(lib.mdd_memcpy(self.ctx.handle, self.ptr, a.ctypes.data_as(C.c_void_p), a.nbytes, 1))

    def download(self, a: np.ndarray):
        check(lib.mdd_memcpy(self.ctx.handle, a.ctypes.data_as(C.c_void_p), self.ptr, a.nbytes, 2))
        return a

    def __del__(self):
        p = getattr(self, "ptr", None)
        if p:
            lib.mdd_dev_free(self.ctx.handle, p)
            self.ptr = None


def exported_symbols():
    return list(SIGNATURES)


def take_ragged(ptr_p, idx_p, n: int) -> list:
    """Copy a library-allocated ragged array (n+1 offsets + flat int64) into numpy and free it."""
    import numpy as np

    try:
        ptr = np.ctypeslib.as_array(ptr_p, shape=(n + 1,)).copy()
        flat = np.ctypeslib.as_array(idx_p, shape=(max(int(ptr[-1]), 1),))[: int(ptr[-1])].copy()
    finally:
        lib.mdd_free(C.cast(ptr_p, C.c_void_p))
        lib.mdd_free(C.cast(idx_p, C.c_void_p))
    return [flat[ptr[i]: ptr[i + 1]] for i in range(n)]
