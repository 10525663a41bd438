"""Host-to-host pipeline over the C ABI: a stream of fields in pinned host memory in, their
triplet stores and diagrams back in pinned host memory out.

Three CUDA streams overlap, step by step, the host->device copy of field i+1, the computation of
field i and the device->host copies of the outputs of field i-1 (double-buffered device buffers,
the diagram written straight into a registered device buffer by `mt_set_diagram_output`).  This is
argument marshalling and stream plumbing only; every step of the computation runs in
libmt_b200.so.
"""
from __future__ import annotations

import torch

from . import _lib


class HostPipeline:
    def __init__(self, dims, conn: int, device=None):
        self.mt = _lib.MergeTree(dims, conn, device)
        dev = self.mt.device
        n = self.mt.n
        self.n = n
        cap = (n + 1) // 2 + 2
        self.f_dev = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(2)]
        self.T_dev = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(2)]
        self.rec_dev = [torch.empty((cap, 4), dtype=torch.int32, device=dev) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.h2d_done = [torch.cuda.Event() for _ in range(2)]
        self.comp_done = [torch.cuda.Event() for _ in range(2)]
        self.d2h_done = [torch.cuda.Event() for _ in range(2)]
        for e in self.comp_done + self.d2h_done:
            e.record(self.s_comp)

    def _h2d(self, i, f_host):
        b = i % 2
        self.s_h2d.wait_event(self.comp_done[b])          # compute i-2 no longer reads f_dev[b]
        with torch.cuda.stream(self.s_h2d):
            self.f_dev[b].copy_(f_host, non_blocking=True)
        self.h2d_done[b].record(self.s_h2d)

    def run(self, f_hosts, T_hosts, rec_hosts, split: bool = False):
        """f_hosts[i] (pinned float32, n) -> T_hosts[i] (pinned int64, n), rec_hosts[i] (pinned int32
        (cap, 4)); returns [(n_pairs, n_essential)] per field.  Synchronises at the end."""
        k = len(f_hosts)
        counts = []
        if k:
            self._h2d(0, f_hosts[0])
        for i in range(k):
            b = i % 2
            self.s_comp.wait_event(self.h2d_done[b])
            self.s_comp.wait_event(self.d2h_done[b])     # outputs of step i-2 copied out
            _lib.mt_set_diagram_output(self.mt.ctx, self.rec_dev[b].data_ptr(), self.rec_dev[b].shape[0])
            _lib.mt_compute(self.mt.ctx, self.f_dev[b].data_ptr(), self.T_dev[b].data_ptr(),
                            _lib.MT_FLAG_SPLIT_TREE if split else 0, self.s_comp)
            self.comp_done[b].record(self.s_comp)
            if i + 1 < k:
                self._h2d(i + 1, f_hosts[i + 1])           # overlaps the computation of field i
            st, npairs, ness = _lib.mt_diagram(self.mt.ctx, 0, 0, self.s_comp)   # waits for field i
            if st != _lib.MT_OK:
                raise _lib.MTError(st, "mt_diagram")
            counts.append((npairs, ness))
            self.s_d2h.wait_event(self.comp_done[b])
            with torch.cuda.stream(self.s_d2h):
                T_hosts[i].copy_(self.T_dev[b], non_blocking=True)
                rec_hosts[i][: npairs + ness].copy_(self.rec_dev[b][: npairs + ness], non_blocking=True)
            self.d2h_done[b].record(self.s_d2h)            # overlaps the computation of field i+1
        torch.cuda.synchronize(self.mt.device)
        _lib.mt_set_diagram_output(self.mt.ctx, 0, 0)
        return counts
