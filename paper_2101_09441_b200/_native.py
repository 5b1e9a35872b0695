"""ctypes binding of the C ABI in include/dbl_b200.h (libdbl_b200.so).

There is no fallback: if the shared library is missing or no CUDA device is
usable, every call raises DeviceError.  The library is built in-tree by
paper_2101_09441_b200/build.py.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import STATUS_ERRORS, DeviceError

LIB_PATH = os.environ.get("DBL_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libdbl_b200.so")

P = ctypes.c_void_p
u8p = ctypes.POINTER(ctypes.c_uint8)
u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32

MEM_HOST, MEM_DEVICE = 0, 1


class Config(ctypes.Structure):
    _fields_ = [("k", u32), ("k_prime", u32), ("strategy", i32),
                ("leaf_threshold", u64), ("hash_seed", u64)]


class UpdateStatsC(ctypes.Structure):
    _fields_ = [("visited", u32), ("labels_changed", u32), ("early_terminated", u32),
                ("inserted", u32)]


class BatchStatsC(ctypes.Structure):
    _fields_ = [("requested", u64), ("inserted", u64), ("certified", u64),
                ("labels_changed", u64), ("levels", u32), ("delta_merged", u32),
                ("fix_items", u64), ("fix_edges", u64)]


class BuildWorkC(ctypes.Structure):
    _fields_ = [("n", u64), ("m", u64), ("record_bytes", u32), ("flags", u32), ("sweeps", u32),
                ("steps", u32), ("fix_levels", u32), ("fix_runs", u32), ("bu_tests", u64),
                ("bu_probes", u64), ("td_vertices", u64), ("td_edges", u64), ("union_records", u64),
                ("fix_items", u64), ("fix_edges", u64)]


# name -> argtypes (restype is always dbl_status / c_int unless listed)
_SIGS = {
    "dbl_graph_create": [u32, P, P, u64, i32, i32, ctypes.POINTER(P)],
    "dbl_graph_free": [P],
    "dbl_graph_info": [P, ctypes.POINTER(u32), ctypes.POINTER(u64)],
    "dbl_graph_degrees": [P, P, P],
    "dbl_graph_has_edges": [P, P, P, u64, P],
    "dbl_graph_edges": [P, P, P],
    "dbl_graph_adjacency": [P, i32, P, P],
    "dbl_graph_add_edges": [P, P, P, u64, ctypes.POINTER(u64)],
    "dbl_graph_add_vertices": [P, u32],
    "dbl_leaf_hash": [P, u64, u32, u64, P, i32],
    "dbl_select_landmarks": [P, u32, i32, P],
    "dbl_select_leaves": [P, u64, u32, u64, P, P, u32, P, P],
    "dbl_index_build": [P, ctypes.POINTER(Config), P, P, P, P, P, u32, ctypes.POINTER(P)],
    "dbl_index_create": [P, ctypes.POINTER(Config), P, P, P, P, P, u32, ctypes.POINTER(P)],
    "dbl_index_rebuild": [P, P],
    "dbl_index_build_words": [P, P, P, u32],
    "dbl_index_free": [P],
    "dbl_index_info": [P, ctypes.POINTER(u32), ctypes.POINTER(Config)],
    "dbl_index_metadata": [P, P, P, P],
    "dbl_index_export": [P, P, P, P, P],
    "dbl_index_import": [P, P, P, P, P],
    "dbl_index_equal": [P, P, ctypes.POINTER(ctypes.c_int)],
    "dbl_index_grow": [P, u32],
    "dbl_index_records": [P, ctypes.POINTER(P), ctypes.POINTER(u32)],
    "dbl_index_pack_words": [P, P, u32, P, P],
    "dbl_index_unpack_words": [P, P, u32, P, P],
    "dbl_label_tests": [P, P, P, u64, P, P],
    "dbl_index_digest": [P, P, P, P],
    "dbl_query_one": [P, P, u32, u32, u32, P],
    "dbl_query": [P, P, P, P, u64, u32, P, P, i32],
    "dbl_query_async": [P, P, P, P, u64, u32, P, P],
    "dbl_query_multi": [P, P, u32, P, P, u64, u32, P, P, i32],
    "dbl_sync": [P],
    "dbl_query_counters": [P, P],
    "dbl_release_cached_memory": [],
    "dbl_stream": [P, ctypes.POINTER(P)],
    "dbl_insert_edge": [P, P, u32, u32, ctypes.POINTER(UpdateStatsC)],
    "dbl_insert_edges": [P, P, P, P, u64, i32, ctypes.POINTER(BatchStatsC)],
    "dbl_work_model": [P, P, P, P, P],
    "dbl_build_work_stats": [P, ctypes.POINTER(BuildWorkC)],
    "dbl_graph_instrument": [P, i32],
    "dbl_verify": [P, P, i32, u64, ctypes.POINTER(u64), P, P, P, P],
    "dbl_rmat_generate": [u32, u64, u64, ctypes.c_double, ctypes.c_double, ctypes.c_double, P, P, i32],
    "dbl_last_timings": [P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                         ctypes.POINTER(ctypes.c_float)],
}

_lib = None


def lib():
    """Load libdbl_b200.so (raises DeviceError if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"native library missing: {LIB_PATH} (run "
                              f"`python -m paper_2101_09441_b200.build`)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.dbl_last_error.restype = ctypes.c_char_p
        L.dbl_last_error.argtypes = []
        L.dbl_version.restype = ctypes.c_int
        L.dbl_kernel_launches.restype = ctypes.c_uint64
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS) + ["dbl_last_error", "dbl_version", "dbl_kernel_launches"]


def check(status: int) -> None:
    if status:
        msg = lib().dbl_last_error().decode(errors="replace")
        raise STATUS_ERRORS.get(status, DeviceError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def device_inputs_ready(*tensors) -> None:
    """The engine orders its stream after the legacy default stream (where torch
    produces tensors unless told otherwise); tensors made on another current
    stream are waited for here."""
    import torch
    for t in tensors:
        if t is not None and getattr(t, "is_cuda", False):
            cur = torch.cuda.current_stream(t.device)
            if cur != torch.cuda.default_stream(t.device):
                cur.synchronize()
            return


def check_device_ids(u, v, device: int) -> None:
    """Validate CUDA id tensors handed to kernels that read uint32 words.

    The kernels take raw pointers, so an int64 tensor would be read as lo/hi
    word pairs and a short `v` read out of bounds: require int32/uint32,
    contiguous, on the graph's device, and equal lengths.
    """
    import torch
    ok_types = {torch.int32}
    if hasattr(torch, "uint32"):
        ok_types.add(torch.uint32)
    for name, t in (("u", u), ("v", v)):
        if not (hasattr(t, "is_cuda") and t.is_cuda):
            raise TypeError(f"{name} must be a CUDA tensor when the other one is")
        if t.dtype not in ok_types:
            raise TypeError(f"{name} must be an int32 or uint32 tensor of vertex ids, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if t.device.index != device:
            raise ValueError(f"{name} lives on {t.device}, the graph on cuda:{device}")
        if t.dim() != 1:
            raise ValueError(f"{name} must be one-dimensional")
    if u.numel() != v.numel():
        raise ValueError(f"u and v differ in length ({u.numel()} vs {v.numel()})")


def ptr(a) -> ctypes.c_void_p | None:
    """Address of a numpy array / torch tensor (host or device) or None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    raise TypeError(f"cannot take the address of {type(a)!r}")


def u32_array(x) -> np.ndarray:
    a = np.asarray(x)
    if a.dtype != np.uint32:
        if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
            from .errors import VertexRangeError
            raise VertexRangeError("vertex id outside the uint32 range")
        a = a.astype(np.uint32)
    return np.ascontiguousarray(a)


def kernel_launches() -> int:
    return int(lib().dbl_kernel_launches())
