"""ctypes binding of include/hosweep_b200.h (libhosweep_b200.so).

The library is the product: CUDA kernels for sm_100a plus the C++ host setup.
There is no CPU fallback — loading fails loudly if the library is missing, and
``hsw_create`` returns HSW_ERR_CUDA when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libhosweep_b200.so")

HSW_ABI_VERSION = 4
HSW_OK = 0
STATUS_NAMES = {
    -1: "HSW_ERR_INVALID", -2: "HSW_ERR_MESH", -3: "HSW_ERR_GEOMETRY", -4: "HSW_ERR_ASSEMBLY",
    -5: "HSW_ERR_SOLVER", -6: "HSW_ERR_LOGIC", -7: "HSW_ERR_RANGE", -8: "HSW_ERR_CUDA",
    -9: "HSW_ERR_NOMEM",
}

# every symbol include/hosweep_b200.h declares
EXPORTED = [
    "hsw_last_error", "hsw_create", "hsw_destroy", "hsw_sizes", "hsw_ordering",
    "hsw_total_lagged_edges", "hsw_couplings", "hsw_interior_faces", "hsw_local_solve",
    "hsw_sweep", "hsw_sweep_device", "hsw_direct_oracle", "hsw_source_iteration", "hsw_balance",
    "hsw_balance_resident", "hsw_device_state", "hsw_sweep_resident", "hsw_synchronize", "hsw_stream",
    "hsw_last_launch_count", "hsw_pivot_fallbacks", "hsw_last_sweep_kernel_ms", "hsw_debug_zero_block",
    "hsw_fp64_peak", "hsw_debug_flags", "hsw_set_state", "hsw_debug_profile",
    "hsw_shard_reset", "hsw_shard_sweep", "hsw_shard_sweep_host", "hsw_shard_phi_partial", "hsw_shard_psi_error",
    "hsw_shard_phi_norms", "hsw_shard_advance", "hsw_shard_psi", "hsw_debug_graph_order",
    "hsw_debug_create_zero_block",
]


class hsw_problem_desc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int), ("dim", C.c_int), ("geom_order", C.c_int),
        ("basis_order", C.c_int), ("num_points", C.c_int), ("points", C.c_void_p),
        ("num_elements", C.c_int), ("element_nodes", C.c_void_p), ("element_region", C.c_void_p),
        ("num_boundary_faces", C.c_int), ("boundary_faces", C.c_void_p),
        ("num_ordinates", C.c_int), ("ordinate_weight", C.c_void_p), ("ordinate_dir", C.c_void_p),
        ("num_regions", C.c_int), ("region_ids", C.c_void_p), ("sigma_t", C.c_void_p),
        ("sigma_s", C.c_void_p), ("source_kind", C.c_int), ("source_params", C.c_double * 8),
        ("inflow", C.c_double), ("volume_points", C.c_int), ("face_points", C.c_int),
        ("weighting", C.c_int), ("exact_fas_threshold", C.c_int), ("validate_geometry", C.c_int),
        ("check_local_blocks", C.c_int), ("device", C.c_int),
        ("face_rule", C.c_int), ("romberg_tol", C.c_double), ("romberg_max_levels", C.c_int),
        ("romberg_min_levels", C.c_int), ("ordinate_begin", C.c_int), ("ordinate_end", C.c_int),
    ]


class hsw_si_options(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int), ("criterion", C.c_int),
                ("mode", C.c_int)]


class hsw_si_result(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_error", C.c_double),
                ("final_phi_rel", C.c_double), ("seconds", C.c_double)]


_lib = None


def load():
    """Load libhosweep_b200.so (build it first with paper_1810_11080_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhosweep_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, i64 = C.c_void_p, C.c_int64
    L.hsw_last_error.argtypes = [C.c_char_p, C.c_size_t]
    L.hsw_create.argtypes = [C.POINTER(hsw_problem_desc), C.POINTER(vp)]
    L.hsw_destroy.argtypes = [vp]
    L.hsw_destroy.restype = None
    L.hsw_sizes.argtypes = [vp, vp]
    L.hsw_ordering.argtypes = [vp, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp]
    L.hsw_total_lagged_edges.argtypes = [vp, vp]
    L.hsw_couplings.argtypes = [vp, C.c_int, vp, vp, C.c_int, vp]
    L.hsw_interior_faces.argtypes = [vp, vp, C.c_int, vp]
    L.hsw_local_solve.argtypes = [vp, C.c_int, C.c_int, vp, vp]
    L.hsw_sweep.argtypes = [vp, C.c_int, vp, vp, vp]
    L.hsw_sweep_device.argtypes = [vp, C.c_int, vp, vp, vp]
    L.hsw_direct_oracle.argtypes = [vp, C.c_int, vp, vp]
    L.hsw_source_iteration.argtypes = [vp, C.POINTER(hsw_si_options), C.POINTER(hsw_si_result), vp, vp, vp, vp, vp]
    L.hsw_balance.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int, vp]
    L.hsw_balance_resident.argtypes = [vp, vp, vp, vp, C.c_int, vp]
    L.hsw_device_state.argtypes = [vp, vp, vp, vp]
    L.hsw_sweep_resident.argtypes = [vp]
    L.hsw_synchronize.argtypes = [vp]
    L.hsw_stream.argtypes = [vp]
    L.hsw_stream.restype = vp
    L.hsw_last_launch_count.argtypes = [vp]
    L.hsw_last_launch_count.restype = i64
    L.hsw_pivot_fallbacks.argtypes = [vp]
    L.hsw_pivot_fallbacks.restype = i64
    L.hsw_last_sweep_kernel_ms.argtypes = [vp]
    L.hsw_last_sweep_kernel_ms.restype = C.c_double
    L.hsw_debug_zero_block.argtypes = [vp, C.c_int, C.c_int]
    L.hsw_debug_create_zero_block.argtypes = [C.c_int, C.c_int]
    L.hsw_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.hsw_debug_flags.argtypes = [vp, C.c_int]
    L.hsw_set_state.argtypes = [vp, vp, vp]
    L.hsw_debug_profile.argtypes = [vp, vp]
    L.hsw_shard_reset.argtypes = [vp]
    L.hsw_shard_sweep.argtypes = [vp, C.c_int, C.c_int, vp]
    L.hsw_shard_sweep_host.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
    L.hsw_shard_phi_partial.argtypes = [vp, C.c_int, C.c_int, vp, vp]
    L.hsw_shard_psi_error.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_double)]
    L.hsw_shard_phi_norms.argtypes = [vp, vp, vp, vp]
    L.hsw_shard_advance.argtypes = [vp, vp]
    L.hsw_shard_psi.argtypes = [vp, C.c_int, C.c_int, vp]
    L.hsw_debug_graph_order.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, vp, C.POINTER(C.c_double)]
    _lib = L
    return L


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    load().hsw_last_error(buf, 4096)
    return buf.value.decode(errors="replace")
