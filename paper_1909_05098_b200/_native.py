"""ctypes binding of libfedheat_b200.so (include/fedheat_b200.h).

There is no fallback: if the library is missing or cannot load, every entry
point raises `NativeLibraryError` -- the engine never silently computes on
the CPU.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import DeviceError, FedheatError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FH_LIB") or os.path.join(_HERE, "libfedheat_b200.so")
MAX_KNOTS = 32
CHUNK_SIZE = 4096

ASSEMBLY = {"exact": 0, "tiled": 1, "atomic": 2}

f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class NativeLibraryError(FedheatError, RuntimeError):
    """libfedheat_b200.so is missing or failed to load (run __graft_entry__.build())."""


class FhCurve(C.Structure):
    _fields_ = [("n", C.c_int32), ("x", f64p), ("y", f64p)]


class FhMaterial(C.Structure):
    _fields_ = [("density", FhCurve), ("specific_heat", FhCurve), ("conductivity", FhCurve),
                ("perfusion", FhCurve), ("perfusion_rate", C.c_double), ("blood_specific_heat", C.c_double),
                ("arterial_temperature", C.c_double), ("metabolic_rate", C.c_double)]


class FhMesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("coords", f64p), ("n_tets", C.c_int64), ("tets", i64p),
                ("n_hexes", C.c_int64), ("hexes", i64p)]


class FhSource(C.Structure):
    _fields_ = [("kind", C.c_int32), ("amp", C.c_double), ("sigma", C.c_double), ("cap", C.c_double),
                ("x0", C.c_double * 3), ("vel", C.c_double * 3), ("t0", C.c_double), ("t1", C.c_double)]


class FhBoundary(C.Structure):
    _fields_ = [
        ("n_dirichlet", C.c_int64), ("dirichlet_nodes", i64p), ("dirichlet_values", f64p),
        ("n_loads", C.c_int64), ("load_offsets", i64p), ("load_nodes", i64p), ("load_power", f64p),
        ("load_t0", f64p), ("load_t1", f64p), ("q_static", f64p), ("n_sources", C.c_int32),
        ("sources", C.POINTER(FhSource)), ("n_robin", C.c_int64), ("robin_nodes", i64p),
        ("robin_hA", f64p), ("robin_hAT", f64p),
    ]


# fh_options tuning knobs (include/fedheat_b200.h); 0 = the measured default
TUNING_FIELDS = ("exact_resident", "resident_ctas", "tile_mode", "tile_stages", "tet_rows", "launch_order",
                 "kind_split", "hex_color", "first_touch", "allow_nondeterministic", "lean_kernels",
                 "resident_sync")


class FhOptions(C.Structure):
    _fields_ = [
        ("precision", C.c_int32), ("assembly", C.c_int32), ("td_mode", C.c_int32), ("device", C.c_int32),
        ("runaway_limit", C.c_double), ("n_materials", C.c_int32), ("materials", C.POINTER(FhMaterial)),
        ("element_region", i32p), ("element_kfactor", f64p), ("part_nodes", C.c_int32),
        ("n_domains", C.c_int32), ("domain_lo", C.c_int32), ("domain_hi", C.c_int32), ("slab_axis", C.c_int32),
    ] + [(name, C.c_int32) for name in TUNING_FIELDS]


# fh_transport (host halo exchange instead of NCCL)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p, C.POINTER(C.c_int64),
                          C.c_void_p, C.POINTER(C.c_int64), C.c_int32)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_uint64))


class FhTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("exchange", EXCHANGE_FN), ("allreduce_min_u64", ALLREDUCE_FN)]


class FhReport(C.Structure):
    _fields_ = [("steps_done", C.c_int64), ("fail_step", C.c_int64), ("fail_node", C.c_int64),
                ("fail_value", C.c_double), ("time", C.c_double), ("step_index", C.c_int64)]


class FhLayout(C.Structure):
    _fields_ = [("n_parts", C.c_int64), ("n_slots", C.c_int64), ("n_nodes_owned", C.c_int64),
                ("n_elements", C.c_int64), ("step_bytes", C.c_int64), ("canonical_bytes", C.c_int64),
                ("kernels_per_step", C.c_int32), ("max_part_nodes", C.c_int32),
                ("resident_ctas", C.c_int32), ("resident_threads", C.c_int32)]


# every symbol include/fedheat_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = [
    "fh_last_error", "fh_version", "fh_device_count", "fh_eval_curve_nodes", "fh_lumped_capacity_nodes",
    "fh_element_mean_nodal", "fh_scatter_net_loads", "fh_nodal_update", "fh_create", "fh_destroy",
    "fh_set_temperature", "fh_get_temperature", "fh_get_inflow", "fh_keep_inflow", "fh_reset_properties", "fh_step",
    "fh_step_timed", "fh_step_timed_flush", "fh_step_host", "fh_step_host_async", "fh_host_wait", "fh_set_q_static", "fh_set_sources", "fh_set_probes", "fh_get_probes", "fh_critical_dt", "fh_scatter_loads",
    "fh_get_precompute", "fh_get_layout", "fh_stream", "fh_get_node_order", "fh_nccl_unique_id", "fh_nccl_library",
    "fh_attach_nccl", "fh_attach_transport", "fh_halo_info", "fh_halo_lists", "fh_halo_export", "fh_halo_import", "fh_get_owned",
    "fh_plan_create", "fh_plan_info", "fh_plan_arrays", "fh_plan_destroy", "fh_mesh_parse", "fh_mesh_text_info",
    "fh_mesh_text_arrays", "fh_mesh_text_set", "fh_mesh_text_destroy", "fh_format_f64", "fh_format_i64",
]

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as err:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {err}") from err
    L.fh_last_error.restype = C.c_char_p
    L.fh_stream.restype = C.c_void_p
    L.fh_stream.argtypes = [C.c_void_p]
    L.fh_create.argtypes = [C.POINTER(FhMesh), C.POINTER(FhBoundary), C.POINTER(FhOptions), C.POINTER(C.c_void_p)]
    L.fh_destroy.argtypes = [C.c_void_p]
    L.fh_set_temperature.argtypes = [C.c_void_p, f64p, C.c_int64, C.c_int64, C.c_double]
    L.fh_get_temperature.argtypes = [C.c_void_p, f64p, C.c_int64]
    L.fh_get_inflow.argtypes = [C.c_void_p, f64p, C.c_int64]
    L.fh_keep_inflow.argtypes = [C.c_void_p, C.c_int32]
    L.fh_reset_properties.argtypes = [C.c_void_p]
    L.fh_step.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(FhReport)]
    L.fh_step_timed.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(FhReport), C.POINTER(C.c_float)]
    L.fh_step_timed_flush.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_size_t,
                                      C.POINTER(FhReport), C.POINTER(C.c_float)]
    L.fh_step_host.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, C.c_int64, C.c_double, C.POINTER(FhReport)]
    L.fh_step_host_async.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, C.c_int64, C.c_double, C.c_int32]
    L.fh_host_wait.argtypes = [C.c_void_p, C.c_int32, C.POINTER(FhReport)]
    L.fh_set_sources.argtypes = [C.c_void_p, C.POINTER(FhSource), C.c_int32]
    L.fh_set_q_static.argtypes = [C.c_void_p, f64p, C.c_int64]
    L.fh_set_probes.argtypes = [C.c_void_p, i64p, C.c_int64, C.c_int64, C.c_int64]
    L.fh_get_probes.argtypes = [C.c_void_p, f64p, C.c_int64, i64p]
    L.fh_critical_dt.argtypes = [C.c_void_p, f64p, C.c_int64, f64p]
    L.fh_scatter_loads.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, f64p]
    L.fh_get_precompute.argtypes = [C.c_void_p, f64p, f64p]
    L.fh_get_layout.argtypes = [C.c_void_p, C.POINTER(FhLayout)]
    L.fh_get_node_order.argtypes = [C.c_void_p, i64p, C.c_int64]
    L.fh_eval_curve_nodes.argtypes = [f64p, f64p, C.c_int64, f64p, C.c_int64, f64p]
    L.fh_lumped_capacity_nodes.argtypes = [f64p, f64p, C.c_int64, f64p, f64p, C.c_int64, f64p, f64p, C.c_int64, f64p]
    L.fh_element_mean_nodal.argtypes = [i64p, i64p, C.c_int64, f64p, C.c_int64, f64p]
    L.fh_scatter_net_loads.argtypes = [i64p, i64p, f64p, i64p, C.c_int64, f64p, f64p, C.c_int64, C.c_int64, f64p]
    L.fh_nodal_update.argtypes = [f64p, f64p, f64p, f64p, f64p, f64p, f64p, C.c_int64, C.c_double]
    L.fh_nccl_unique_id.argtypes = [C.c_char_p]
    L.fh_nccl_library.argtypes = [C.c_char_p]
    # one NCCL per process: prefer the copy PyTorch bundles (found without
    # importing torch), so that the library's dlopen and a later `import torch`
    # agree on the version behind the libnccl.so.2 soname
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations if spec else []):
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                L.fh_nccl_library(cand.encode())
                break
    except Exception:  # pragma: no cover - best effort, the sonames remain
        pass
    L.fh_attach_nccl.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32]
    L.fh_attach_transport.argtypes = [C.c_void_p, C.POINTER(FhTransport)]
    i32o = C.POINTER(C.c_int32)
    L.fh_halo_info.argtypes = [C.c_void_p, i32o, i32o, i32o, i64p, i64p, i64p, i64p]
    L.fh_halo_lists.argtypes = [C.c_void_p, i32p, i64p, i64p, i64p, i64p]
    L.fh_halo_export.argtypes = [C.c_void_p, f64p]
    L.fh_halo_import.argtypes = [C.c_void_p, f64p]
    L.fh_get_owned.argtypes = [C.c_void_p, C.POINTER(C.c_uint8), C.c_int64]
    L.fh_plan_create.argtypes = [C.POINTER(FhMesh), C.POINTER(FhBoundary), C.POINTER(FhOptions), C.c_int32,
                                 C.c_int32, C.POINTER(C.c_void_p)]
    L.fh_plan_info.argtypes = [C.c_void_p, i64p, C.c_int32]
    L.fh_plan_arrays.argtypes = [C.c_void_p, i64p, i64p, i32p, i64p, i64p, i64p, i64p]
    L.fh_plan_destroy.argtypes = [C.c_void_p]
    L.fh_mesh_parse.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p), i64p]
    L.fh_mesh_text_info.argtypes = [C.c_void_p, i64p, i64p, i64p, C.POINTER(C.c_int32)]
    L.fh_mesh_text_arrays.argtypes = [C.c_void_p, f64p, i64p, i64p]
    L.fh_mesh_text_set.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64, i64p, i64p]
    L.fh_mesh_text_destroy.argtypes = [C.c_void_p]
    L.fh_format_f64.argtypes = [f64p, C.c_int64, C.c_int64, C.c_char, C.c_char_p, C.c_int32, C.c_char_p,
                                C.c_int64, i64p]
    L.fh_format_i64.argtypes = [i64p, C.c_int64, C.c_int64, C.c_char, C.c_char_p, C.c_int32, C.c_char_p,
                                C.c_int64, i64p]
    _lib = L
    return L


def check(status: int) -> None:
    if status:
        raise_for_status(int(status), lib().fh_last_error().decode())


def ptr(a, t=f64p):
    return None if a is None else a.ctypes.data_as(t)


def device_count() -> int:
    n = C.c_int(0)
    check(lib().fh_device_count(C.byref(n)))
    return int(n.value)


def require_gpu() -> None:
    if device_count() < 1:
        raise DeviceError("no CUDA device visible: the engine runs on B200 GPUs only (no CPU fallback)")


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
