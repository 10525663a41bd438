"""B200-native triplet merge tree + 0-dimensional persistence diagram (arXiv 2301.10838).

The hot path runs in libmt_b200.so (hand-written sm_100a CUDA kernels behind the
C ABI of include/mt.h); ``_lib`` is its thin ctypes binding.  Importing this
package does not load the library; the first call does, and fails loudly if it
is missing (there is no CPU fallback).
"""
from ._lib import (MT_FLAG_SPLIT_TREE, PAIR_DTYPE, MergeTree, MTError, load, mt_compute, mt_create,
                   mt_destroy, mt_diagram, mt_diagram_view, mt_kernel_times, mt_last_error,
                   mt_last_launch_count, mt_set_diagram_output, mt_set_profiling, mt_workspace_bytes,
                   pairs_to_numpy)

__all__ = ["MergeTree", "MTError", "MT_FLAG_SPLIT_TREE", "PAIR_DTYPE", "load", "mt_compute", "mt_create",
           "mt_destroy", "mt_diagram", "mt_diagram_view", "mt_kernel_times", "mt_last_error",
           "mt_last_launch_count", "mt_set_diagram_output", "mt_set_profiling", "mt_workspace_bytes",
           "pairs_to_numpy"]
