"""One run_workload step fed from host memory (rs_feeder_*; workload.cpp:506-581).

The data loader's pinned token ids + sequence lengths go host -> device on a
copy stream that runs ahead of the compute, the gradients are
pseudo_sparse_grad on the device, the step runs, and only the step's
embedding checksum comes back.  Used by bench.py's end-to-end measurement.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from ._lib import check
from .table import SparseStep, _stream


class Feeder:
    def __init__(self, max_tokens: int, max_seqs: int, dim: int):
        self._h = C.c_void_p()
        check(L.lib().rs_feeder_create(max_tokens, max_seqs, dim, C.byref(self._h)), "Feeder")
        self.dim = dim
        self.result = torch.zeros(1, dtype=torch.float64).pin_memory()

    def step(self, st: SparseStep, h_ids: torch.Tensor, h_lengths: torch.Tensor, step: int,
             first_sample_id: int = 1) -> None:
        """h_ids / h_lengths: pinned int64 host tensors of one batch."""
        check(L.lib().rs_feeder_step(self._h, st.ws.handle, st.table.handle, h_ids.data_ptr(), h_ids.numel(),
                                     h_lengths.data_ptr(), h_lengths.numel(), first_sample_id, step,
                                     C.byref(st.params.c()), self.result.data_ptr(), _stream()), "feeder_step")

    def dist_step(self, sharded, params, h_ids: torch.Tensor, h_lengths: torch.Tensor, step: int,
                  first_sample_id: int = 1) -> None:
        check(L.lib().rs_feeder_dist_step(self._h, sharded._c, sharded.shard.handle, h_ids.data_ptr(), h_ids.numel(),
                                          h_lengths.data_ptr(), h_lengths.numel(), first_sample_id, step,
                                          C.byref(params.c()), self.result.data_ptr(), _stream()),
              "feeder_dist_step")

    def checksum(self) -> float:
        torch.cuda.current_stream().synchronize()
        return float(self.result[0])

    def close(self):
        if self._h:
            L.lib().rs_feeder_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
