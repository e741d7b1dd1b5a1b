"""ctypes binding of libsylvadi_b200.so (the C-ABI in include/sylvadi_b200.h).

The shared library is built in-tree (``python -m paper_2312_02891_b200._build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or no CUDA device is present, every GPU entry point raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
#: SAD_LIB_PATH selects another build of the library (A/B experiments)
LIB_PATH = os.environ.get("SAD_LIB_PATH") or os.path.join(_HERE, "libsylvadi_b200.so")

SAD_OK, SAD_EINVAL, SAD_EBREAKDOWN, SAD_ECUDA, SAD_ENCCL, SAD_ENOMEM = range(6)
SAD_F64, SAD_C128 = 0, 1
SAD_PRECOND_NONE, SAD_PRECOND_JACOBI = 0, 1
SAD_PRECOND_ILU0, SAD_PRECOND_ILUT, SAD_PRECOND_IC0, SAD_PRECOND_ICT = 2, 3, 4, 5
PRECOND_CODES = {"none": 0, "jacobi": 1, "ilu0": 2, "ilut": 3, "ic0": 4, "ict": 5}
SAD_ENGINE_MULTI, SAD_ENGINE_PERSISTENT = 0, 1
SAD_OPT_ENGINE, SAD_OPT_MAX_SMS, SAD_OPT_MIN_ELEMS_PER_THREAD, SAD_OPT_DIRECT_A = 0, 1, 2, 3
SAD_OPT_RESIDENT_CSR = 4
SAD_OPT_DIST_ORTH = 5
SAD_OPT_DEBUG_DELAY = 6

#: every symbol declared in include/sylvadi_b200.h with (restype, argtypes)
_c = ctypes
_vp = _c.c_void_p
_i64 = _c.c_int64
SIGNATURES = {
    "sad_version": (_c.c_int, []),
    "sad_kernel_launches": (_i64, []),
    "sad_gmres_profile": (_c.c_int, [_vp, _c.c_int, _vp]),
    "sad_ctx_create": (_c.c_int, [_c.c_int, _c.POINTER(_vp)]),
    "sad_ctx_destroy": (_c.c_int, [_vp]),
    "sad_last_error": (_c.c_char_p, [_vp]),
    "sad_ctx_num_sms": (_c.c_int, [_vp]),
    "sad_ctx_trim": (_c.c_int, [_vp]),
    "sad_csr_create": (_c.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _c.c_int,
                                  _c.POINTER(_vp)]),
    "sad_csr_destroy": (_c.c_int, [_vp]),
    "sad_csr_nnz": (_i64, [_vp]),
    "sad_op_create": (_c.c_int, [_vp, _vp, _vp, _c.c_double, _c.c_double, _c.c_int,
                                 _c.c_int, _c.POINTER(_vp)]),
    "sad_op_destroy": (_c.c_int, [_vp]),
    "sad_op_get_dinv": (_c.c_int, [_vp, _vp]),
    "sad_op_band_info": (_c.c_int, [_vp, _c.c_int, _vp]),
    "sad_op_apply": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _vp, _vp]),
    "sad_op_apply_host": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _vp, _vp]),
    "sad_op_residual": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _vp, _vp, _vp]),
    "sad_csr_apply": (_c.c_int, [_vp, _c.c_int, _c.c_int, _c.c_int, _vp, _vp, _vp]),
    "sad_gmres_create": (_c.c_int, [_vp, _i64, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                    _c.POINTER(_vp)]),
    "sad_gmres_destroy": (_c.c_int, [_vp]),
    "sad_gmres_bytes": (_i64, [_vp]),
    "sad_gmres_set_option": (_c.c_int, [_vp, _c.c_int, _c.c_int]),
    "sad_gmres_solve": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _c.c_double, _c.c_int, _vp,
                                   _vp, _vp, _vp]),
    "sad_gmres_launch": (_c.c_int, [_vp, _vp, _vp, _vp, _c.c_double, _c.c_int, _vp]),
    "sad_gmres_finish": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "sad_gmres_fixed": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _c.c_int, _vp, _vp, _vp]),
    "sad_gram": (_c.c_int, [_vp, _i64, _c.c_int, _c.c_int, _vp, _vp, _vp, _vp]),
    "sad_axpy": (_c.c_int, [_vp, _i64, _c.c_int, _c.c_int, _c.c_double, _c.c_double,
                            _vp, _vp, _vp]),
    "sad_adi_epilogue": (_c.c_int, [_vp, _i64, _i64, _c.c_int, _c.c_int, _c.c_double,
                                    _c.c_double, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sad_ts_hgemv": (_c.c_int, [_vp, _i64, _i64, _i64, _c.c_int, _vp, _c.c_int, _vp, _vp,
                                _vp]),
    "sad_ts_gemv": (_c.c_int, [_vp, _i64, _i64, _i64, _c.c_int, _vp, _c.c_int, _vp, _vp,
                               _c.c_int, _vp]),
    # row-partitioned solves (per-rank arguments are arrays of nl pointers)
    "sad_comm_unique_id": (_c.c_int, [_vp]),
    "sad_comm_nccl_error": (_c.c_char_p, []),
    "sad_comm_create_nccl": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _c.POINTER(_vp)]),
    "sad_comm_create_local": (_c.c_int, [_vp, _c.c_int, _c.POINTER(_vp)]),
    "sad_comm_destroy": (_c.c_int, [_vp]),
    "sad_comm_size": (_c.c_int, [_vp]),
    "sad_comm_local_ranks": (_c.c_int, [_vp]),
    "sad_halo_create": (_c.c_int, [_vp, _c.c_int, _c.c_int, _i64, _i64, _vp, _vp, _vp,
                                   _c.POINTER(_vp)]),
    "sad_halo_destroy": (_c.c_int, [_vp]),
    "sad_local_csr_create": (_c.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp,
                                        _c.POINTER(_vp)]),
    "sad_local_op_create": (_c.c_int, [_vp, _vp, _c.c_double, _c.c_double, _c.c_int,
                                       _c.POINTER(_vp)]),
    "sad_dist_op_setup": (_c.c_int, [_vp, _c.c_int, _vp, _vp, _vp]),
    "sad_dist_halo_exchange": (_c.c_int, [_vp, _c.c_int, _vp, _vp, _c.c_int, _c.c_int, _vp]),
    "sad_dist_op_apply": (_c.c_int, [_vp, _c.c_int, _vp, _vp, _c.c_int, _c.c_int, _vp, _vp,
                                     _vp]),
    "sad_dist_allreduce": (_c.c_int, [_vp, _c.c_int, _vp, _i64, _vp]),
    "sad_dist_gmres_create": (_c.c_int, [_vp, _i64, _i64, _c.c_int, _c.c_int, _c.c_int,
                                         _c.c_int, _c.POINTER(_vp)]),
    "sad_dist_gmres_solve": (_c.c_int, [_vp, _c.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _c.c_double, _c.c_int, _vp, _vp, _vp, _vp]),
    # device BiCGstab (the reference's own inner solver)
    "sad_bicg_create": (_c.c_int, [_vp, _i64, _c.c_int, _c.c_int, _c.POINTER(_vp)]),
    "sad_bicg_destroy": (_c.c_int, [_vp]),
    "sad_bicg_bytes": (_i64, [_vp]),
    "sad_bicg_solve": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _c.c_double, _c.c_int, _vp, _vp,
                                  _vp, _vp]),
    # device MINRES (the reference's inner solver for Hermitian sides)
    "sad_minres_create": (_c.c_int, [_vp, _i64, _c.c_int, _c.c_int, _c.POINTER(_vp)]),
    "sad_minres_destroy": (_c.c_int, [_vp]),
    "sad_minres_bytes": (_i64, [_vp]),
    "sad_minres_solve": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _c.c_double, _c.c_int, _vp, _vp,
                                    _vp, _vp]),
    # incomplete-factorisation preconditioners
    "sad_pc_create": (_c.c_int, [_vp, _vp, _vp, _c.c_double, _c.c_double, _c.c_int, _c.c_int,
                                 _c.c_double, _c.POINTER(_vp)]),
    "sad_pc_destroy": (_c.c_int, [_vp]),
    "sad_pc_info": (_c.c_int, [_vp, _vp]),
    "sad_pc_get_factor": (_c.c_int, [_vp, _c.c_int, _vp, _vp, _vp]),
    "sad_pc_apply": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _vp, _c.c_int, _vp]),
    "sad_bicg_solve_pc": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c.c_double, _c.c_int, _vp,
                                     _vp, _vp, _vp]),
    "sad_minres_solve_pc": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c.c_double, _c.c_int,
                                       _vp, _vp, _vp, _vp]),
    # native ADI outer loop
    "sad_adi_run": (_c.c_int, [_vp, _vp, _c.c_int, _c.c_int, _i64, _i64, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _c.c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
}


class AdiConfigC(_c.Structure):
    """sad_adi_config (include/sylvadi_b200.h)."""
    _fields_ = [("strategy", _c.c_int), ("kmax", _c.c_int), ("max_inner_iterations", _c.c_int),
                ("outer_tolerance", _c.c_double), ("xi", _c.c_double),
                ("gap_budget", _c.c_double), ("fixed_delta", _c.c_double),
                ("delta_min_A", _c.c_double), ("delta_max_A", _c.c_double),
                ("delta_min_B", _c.c_double), ("delta_max_B", _c.c_double),
                ("has_gap_budget", _c.c_int)]


SAD_ADI_REC = 14
STRATEGY_CODES = {"fixed": 0, "dynamic_mid": 1, "dynamic_mid_bl": 2, "dynamic_b": 3,
                  "dynamic_b_bl": 4}


class FactorizationBreakdown(RuntimeError):
    """Zero Jacobi diagonal, zero pivot or an indefinite matrix for the Cholesky
    kinds (the reference's precond.FactorizationBreakdown)."""


class DeviceError(RuntimeError):
    """CUDA failure inside libsylvadi_b200."""


_LIB = None


def load(path=None):
    """Load the shared library (once) and attach the ctypes signatures."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} not found: build it with `python -m paper_2312_02891_b200._build` "
            "(there is no CPU fallback for the inner-solve path)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("SAD_LIB_PATH") and not hasattr(lib, name):
            continue            # A/B builds of older sources (tools/build_variant.py)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def check(rc, ctx=None):
    """Map a status code to the reference's exception classes."""
    if rc == SAD_OK:
        return
    lib = load()
    msg = lib.sad_last_error(ctx).decode() if ctx else f"status {rc}"
    if rc == SAD_EINVAL:
        raise ValueError(msg)
    if rc == SAD_EBREAKDOWN:
        raise FactorizationBreakdown(msg)
    if rc == SAD_ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


_CTX = {}


def context(device=0):
    """Process-wide context per device (one ctx per device, header contract)."""
    ctx = _CTX.get(device)
    if ctx is None:
        lib = load()
        h = ctypes.c_void_p()
        rc = lib.sad_ctx_create(int(device), ctypes.byref(h))
        if rc != SAD_OK:
            raise DeviceError(f"sad_ctx_create(device={device}) failed with status {rc}")
        ctx = h
        _CTX[device] = ctx
    return ctx
