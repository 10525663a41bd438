"""Host-to-host steps over the C ABI (``mt_compute_host``): a stream of fields in pinned host
memory in, their triplet stores and diagrams back in pinned host memory out.

The library overlaps, step by step on three CUDA streams of its own, the host->device copy of
field i+1, the computation of field i and the device->host copies of the outputs of field i-1
(double-buffered device staging that this object owns as a torch tensor).  This module is
argument marshalling only; every copy and every step of the computation is issued by
libmt_b200.so.
"""
from __future__ import annotations

import torch

from . import _lib


class HostPipeline:
    def __init__(self, dims, conn: int, device=None):
        self.mt = _lib.MergeTree(dims, conn, device)
        self.n = self.mt.n
        nbytes = _lib.mt_host_staging_bytes(self.mt.ctx)
        self.staging = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.mt.device)
        self._sp = (self.staging.data_ptr() + 255) // 256 * 256
        self._sb = nbytes

    def run(self, f_hosts, T_hosts, rec_hosts, split: bool = False, stream=None):
        """f_hosts[i] (pinned float32, n) -> T_hosts[i] (pinned int64, n), rec_hosts[i] (pinned int32
        (cap, 4)); returns [(n_pairs, n_essential)] per field.  Synchronous."""
        cap = min(r.shape[0] for r in rec_hosts) if rec_hosts else 0
        return _lib.mt_compute_host(self.mt.ctx, [f.data_ptr() for f in f_hosts], [t.data_ptr() for t in T_hosts],
                                    [r.data_ptr() for r in rec_hosts], cap,
                                    _lib.MT_FLAG_SPLIT_TREE if split else 0, self._sp, self._sb, stream)
