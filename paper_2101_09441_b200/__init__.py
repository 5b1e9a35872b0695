"""B200-native DBL reachability engine (drop-in for dblreach's hot path).

Reference: /root/reference/pkg/src/dblreach (pure Python).  This package
keeps its index API -- build_index, query / query_batch, insert_edge -- and
runs every step on the GPU through the C ABI in include/dbl_b200.h
(libdbl_b200.so, hand-written sm_100a CUDA).  There is no CPU fallback: a
missing library or device raises DeviceError.
"""
from .errors import (ConfigError, DblError, DeviceError, EdgeListFormatError,
                     IndexGraphMismatchError, MissingEdgeError, NotFittedError,
                     VertexRangeError, WorkloadExhaustedError)
from .graph import DynamicGraph, as_device_graph, load_edge_list
from .labels import (DblIndex, IndexConfig, LandmarkSet, LandmarkStrategy, LeafSets,
                     bl_contain, build_index, dl_intersec, leaf_hash, leaf_hash_batch,
                     rebuild_in_place, rebuild_index, select_landmarks, select_leaves)
from .queries import (BL_ONLY, DEFAULT_FLAGS, DL_ONLY, AnsweredBy, BatchStats, Outcomes,
                      QueryFlags, QueryOutcome, default_workers, explain, query, query_batch,
                      query_codes)
from .updates import BatchUpdateStats, UpdateStats, insert_edge, insert_edges, insert_vertex
from .snapshot import SnapshotFormatError, load_index, save_index, sniff_snapshot
from .verify import LabelViolation, VerifyReport, verify_labels
from .estimator import DblReachability

__version__ = "0.1.0"

__all__ = [
    "DblReachability", "LabelViolation", "SnapshotFormatError", "VerifyReport", "load_index",
    "save_index", "sniff_snapshot", "verify_labels",
    "AnsweredBy", "BL_ONLY", "BatchStats", "BatchUpdateStats", "ConfigError", "DEFAULT_FLAGS",
    "DL_ONLY", "DblError", "DblIndex", "DeviceError", "DynamicGraph", "EdgeListFormatError",
    "IndexConfig", "IndexGraphMismatchError", "LandmarkSet", "LandmarkStrategy", "LeafSets",
    "MissingEdgeError", "NotFittedError", "Outcomes", "QueryFlags", "QueryOutcome",
    "UpdateStats", "VertexRangeError", "WorkloadExhaustedError", "as_device_graph", "load_edge_list",
    "bl_contain", "build_index", "default_workers", "dl_intersec", "explain", "insert_edge",
    "insert_edges", "insert_vertex", "leaf_hash", "leaf_hash_batch", "query", "query_batch",
    "query_codes", "rebuild_in_place", "rebuild_index", "select_landmarks", "select_leaves",
]
