"""ctypes binding of libctk_b200.so (include/ctk_b200.h).

There is no fallback: if the native library is missing or cannot be loaded, importing the
operator layer raises.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``
(or ``make -C paper_2211_14212_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CTK_B200_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("CTK_B200_LIB") or os.path.join(HERE, "lib", "libctk_b200.so")

CTK_OK, CTK_E_DIMENSION, CTK_E_GEOMETRY, CTK_E_PARAMETER, CTK_E_DEGENERATE, CTK_E_NUMERICAL, CTK_E_CUDA, CTK_E_UNSUPPORTED = range(8)


class GeomDesc(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("source_to_origin", C.c_double),
        ("origin_to_detector", C.c_double),
        ("detector_pixel_size", C.c_double),
        ("nu", C.c_int),
        ("nv", C.c_int),
        ("nx", C.c_int),
        ("ny", C.c_int),
        ("nz", C.c_int),
        ("spacing", C.c_double),
        ("n_angles", C.c_int),
        ("angles", C.POINTER(C.c_double)),
    ]


OBSERVER = C.CFUNCTYPE(None, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p)


class SolverOpts(C.Structure):
    _fields_ = [
        ("max_iters", C.c_int),
        ("stop_on_explicit_residual_increase", C.c_int),
        ("residual_tolerance", C.c_double),
        ("reorth", C.c_int),
        ("ground_truth", C.c_void_p),
        ("iterate_observer", OBSERVER),
        ("observer_user", C.c_void_p),
    ]


class SolveLog(C.Structure):
    _fields_ = [
        ("capacity", C.c_int),
        ("implicit_residual", C.POINTER(C.c_double)),
        ("explicit_residual", C.POINTER(C.c_double)),
        ("relative_error", C.POINTER(C.c_double)),
        ("lambda_", C.POINTER(C.c_double)),
        ("outer_starts", C.POINTER(C.c_int)),
        ("iterations", C.c_int),
        ("n_relative_error", C.c_int),
        ("n_lambda", C.c_int),
        ("n_outer_starts", C.c_int),
        ("iterations_run", C.c_int),
        ("stop_reason", C.c_int),
        ("stored_domain_basis", C.c_int),
        ("stored_range_basis", C.c_int),
        ("warning_iterations", C.POINTER(C.c_int)),
        ("n_warnings", C.c_int),
    ]


class HybridStrategyC(C.Structure):
    _fields_ = [("kind", C.c_int), ("lambda_", C.c_double), ("noise_level", C.c_double)]


ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_double, C.POINTER(C.c_double), C.c_void_p)


class P2POp(C.Structure):
    _fields_ = [("peer", C.c_int), ("is_send", C.c_int), ("d_buf", C.c_void_p), ("count", C.c_size_t)]


EXCHANGE = C.CFUNCTYPE(C.c_int, C.POINTER(P2POp), C.c_int, C.c_int, C.c_void_p, C.c_void_p)


class CommCallbacks(C.Structure):
    _fields_ = [
        ("rank", C.c_int),
        ("nranks", C.c_int),
        ("allreduce_sum", ALLREDUCE),
        ("allgather_f64", ALLGATHER),
        ("user", C.c_void_p),
        ("exchange", EXCHANGE),
    ]


_lib = None


def load():
    """Load libctk_b200.so once; raise (never fall back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libctk_b200.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i, sz, d = C.c_void_p, C.c_int, C.c_size_t, C.c_double
    pd = C.POINTER(C.c_double)
    sig = {
        "ctk_last_error": (i, [C.c_char_p, sz]),
        "ctk_last_error_iteration": (i, []),
        "ctk_abi_version": (i, []),
        "ctk_geom_create": (i, [C.POINTER(GeomDesc), C.POINTER(vp)]),
        "ctk_geom_validate": (i, [C.POINTER(GeomDesc)]),
        "ctk_geom_destroy": (None, [vp]),
        "ctk_geom_sizes": (i, [vp, C.POINTER(sz), C.POINTER(sz)]),
        "ctk_geom_set_projector": (i, [vp, i]),
        "ctk_geom_set_bp_partitions": (i, [vp, i]),
        "ctk_geom_set_slab": (i, [vp, i, i]),
        "ctk_geom_shard_range": (i, [vp]),
        "ctk_geom_range_rows": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i)]),
        "ctk_band_partition": (i, [C.POINTER(GeomDesc), i, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i),
                                   C.POINTER(i), C.POINTER(i)]),
        "ctk_geom_set_stream": (i, [vp, vp]),
        "ctk_geom_attach_comm": (i, [vp, vp]),
        "ctk_geom_last_kernel_ms": (d, [vp]),
        "ctk_ax_f32": (i, [vp, vp, vp, vp]),
        "ctk_ax_f64": (i, [vp, vp, vp, vp]),
        "ctk_atb_f32": (i, [vp, i, vp, vp, vp]),
        "ctk_atb_f64": (i, [vp, i, vp, vp, vp]),
        "ctk_ax_residual_f32": (i, [vp, vp, vp, pd, vp]),
        "ctk_ax_pair_f32": (i, [vp, vp, vp, vp, vp, vp]),
        "ctk_ax_host_f32": (i, [vp, vp, vp]),
        "ctk_ax_host_f64": (i, [vp, vp, vp]),
        "ctk_atb_host_f32": (i, [vp, i, vp, vp]),
        "ctk_atb_host_f64": (i, [vp, i, vp, vp]),
        "ctk_dot_f32": (i, [sz, vp, vp, pd, vp]),
        "ctk_dot_f64": (i, [sz, vp, vp, pd, vp]),
        "ctk_nrm2_f32": (i, [sz, vp, pd, vp]),
        "ctk_nrm2_f64": (i, [sz, vp, pd, vp]),
        "ctk_axpy_f32": (i, [sz, d, vp, vp, vp]),
        "ctk_axpy_f64": (i, [sz, d, vp, vp, vp]),
        "ctk_scal_f32": (i, [sz, d, vp, vp]),
        "ctk_scal_f64": (i, [sz, d, vp, vp]),
        "ctk_shepp_logan_3d_f32": (i, [i, vp, vp]),
        "ctk_shepp_logan_3d_f64": (i, [i, vp, vp]),
        "ctk_make_phantom_f32": (i, [i, i, vp, vp]),
        "ctk_make_phantom_f64": (i, [i, i, vp, vp]),
        "ctk_add_noise_f32": (i, [sz, vp, d, d, C.c_uint64, vp]),
        "ctk_gradient_f32": (i, [i, i, i, vp, vp, vp, vp, vp]),
        "ctk_gradient_f64": (i, [i, i, i, vp, vp, vp, vp, vp]),
        "ctk_gradient_adjoint_f32": (i, [i, i, i, vp, vp, vp, vp, vp]),
        "ctk_gradient_adjoint_f64": (i, [i, i, i, vp, vp, vp, vp, vp]),
        "ctk_tv_weights_f32": (i, [i, i, i, vp, d, vp, vp]),
        "ctk_tv_weights_f64": (i, [i, i, i, vp, d, vp, vp]),
        "ctk_add_noise_f64": (i, [sz, vp, d, d, C.c_uint64, vp]),
        "ctk_solve_dev_f32": (i, [vp, i, i, vp, d, C.POINTER(HybridStrategyC), i, i, i, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)]),
        "ctk_solve_dev_f64": (i, [vp, i, i, vp, d, C.POINTER(HybridStrategyC), i, i, i, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)]),
        "ctk_shard_angles": (i, [i, i, i, C.POINTER(i), C.POINTER(i)]),
        "ctk_shard_slabs": (i, [i, i, i, C.POINTER(i), C.POINTER(i)]),
        "ctk_comm_create": (i, [C.POINTER(CommCallbacks), C.POINTER(vp)]),
        "ctk_nccl_get_unique_id": (i, [vp]),
        "ctk_comm_create_nccl": (i, [vp, i, i, C.POINTER(vp)]),
        "ctk_comm_adopt_nccl": (i, [vp, i, i, C.POINTER(vp)]),
        "ctk_comm_destroy": (None, [vp]),
        "ctk_launch_count": (C.c_uint64, []),
        "ctk_projected_gcv_lambda": (i, [pd, i, d, pd]),
        "ctk_projected_dp_lambda": (i, [pd, i, d, d, pd]),
        "ctk_projected_tikhonov": (i, [pd, i, d, d, pd, pd]),
    }
    for t in ("f32", "f64"):
        sig[f"ctk_cgls_{t}"] = (i, [vp, i, vp, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        sig[f"ctk_lsqr_{t}"] = (i, [vp, i, vp, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        for nm in ("sirt", "ab_gmres", "ba_gmres"):
            sig[f"ctk_{nm}_{t}"] = (i, [vp, i, vp, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        sig[f"ctk_lsmr_{t}"] = (i, [vp, i, vp, d, C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        sig[f"ctk_hybrid_lsqr_{t}"] = (i, [vp, i, vp, C.POINTER(HybridStrategyC), C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        sig[f"ctk_flsqr_tv_{t}"] = (i, [vp, i, vp, C.POINTER(HybridStrategyC), C.POINTER(SolverOpts), vp, C.POINTER(SolveLog)])
        sig[f"ctk_cgls_tv_{t}"] = (i, [vp, i, vp, d, i, i, C.POINTER(SolverOpts), i, vp, C.POINTER(SolveLog)])
    for name, (res, args) in sig.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.environ.get("CTK_B200_LIB"):  # an older build loaded for A/B timing
                continue
            raise
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error():
    lib = load()
    buf = C.create_string_buffer(512)
    code = lib.ctk_last_error(buf, 512)
    return code, buf.value.decode(errors="replace"), lib.ctk_last_error_iteration()
