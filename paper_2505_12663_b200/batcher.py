"""Dynamic sequence balancing (host mirror of seq_batcher.hpp).

``closest_prefix`` / ``SequenceBatcher`` (seq_batcher.cpp:22-78, PAPER.md
Alg. 1), ``imbalance_report``, ``weighted_grad_combine`` and the rank
partition run in librsgpu's host code (batcher.cu); same argument meaning
and errors as the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import check

ROUND_ROBIN, COST_LPT = 0, 1


@dataclass
class SequenceSample:
    sample_id: int = 0
    feature_ids: list = field(default_factory=list)
    label: float = 0.0

    def token_count(self) -> int:
        return len(self.feature_ids)


def closest_prefix(cumsums, target: int) -> int:
    c = np.ascontiguousarray(cumsums, np.uint64)
    k = C.c_uint64()
    check(L.lib().rs_closest_prefix(c.ctypes.data if len(c) else None, len(c), int(target), C.byref(k)),
          "closest_prefix")
    return k.value


class SequenceBatcher:
    """SequenceBatcher(target_tokens, source): source(chunk: list) -> bool
    appends SequenceSample objects (ChunkSource, seq_batcher.hpp:38)."""

    def __init__(self, target_tokens: int, source, max_chunk: int = 1 << 16):
        self._source = source
        self._objs = {}
        self._next = 0
        self._err = None

        def pull(ctx, ids, toks, cap, n_out):
            try:
                chunk = []
                more = bool(source(chunk))
                if not more:
                    n_out[0] = 0
                    return 0
                if len(chunk) > cap:
                    raise L.ConfigError("SequenceBatcher: chunk larger than max_chunk")
                for i, s in enumerate(chunk):
                    ids[i] = self._next
                    toks[i] = s.token_count()
                    self._objs[self._next] = s
                    self._next += 1
                n_out[0] = len(chunk)
                return 1
            except Exception as e:  # surfaced after the C call returns
                self._err = e
                n_out[0] = 0
                return 0

        self._cb = L.rs_chunk_source(pull)
        self._h = C.c_void_p()
        check(L.lib().rs_seq_batcher_create(int(target_tokens), self._cb, None, max_chunk, C.byref(self._h)),
              "SequenceBatcher")
        self._target = int(target_tokens)
        self._cap = max_chunk

    def next_batch(self):
        """Next batch (list of samples) in arrival order, or None when done."""
        cap = len(self._objs) + self._cap
        ids = np.zeros(max(cap, 1), np.uint64)
        n = C.c_uint64()
        st = L.lib().rs_seq_batcher_next(self._h, ids.ctypes.data, None, cap, C.byref(n))
        if self._err is not None:
            e, self._err = self._err, None
            raise e
        check(st, "next_batch")
        if n.value == 0:
            return None
        return [self._objs.pop(int(i)) for i in ids[: n.value]]

    def target_tokens(self) -> int:
        return self._target

    def buffered_tokens(self) -> int:
        return L.lib().rs_seq_batcher_buffered_tokens(self._h)

    def buffered_samples(self) -> int:
        return L.lib().rs_seq_batcher_buffered_samples(self._h)

    def __del__(self):
        try:
            if self._h:
                L.lib().rs_seq_batcher_destroy(self._h)
                self._h = None
        except Exception:
            pass


def partition_sequences(lengths, world: int, policy: int = COST_LPT, a: float = 1.0, b: float = 0.01):
    """-> (rank per sequence, cost per rank)."""
    ln = np.ascontiguousarray(lengths, np.uint64)
    ranks = np.zeros(max(len(ln), 1), np.uint32)
    load = np.zeros(world, np.float64)
    check(L.lib().rs_partition_sequences(ln.ctypes.data, len(ln), world, policy, a, b, ranks.ctypes.data,
                                         load.ctypes.data), "partition_sequences")
    return ranks[: len(ln)], load


@dataclass
class ImbalanceReport:
    max_tokens: int
    min_tokens: int
    spread: float


def imbalance_report(per_worker_tokens) -> ImbalanceReport:
    t = np.ascontiguousarray(per_worker_tokens, np.uint64)
    mx, mn, sp = C.c_uint64(), C.c_uint64(), C.c_double()
    check(L.lib().rs_imbalance_report(t.ctypes.data if len(t) else None, len(t), C.byref(mx), C.byref(mn),
                                      C.byref(sp)), "imbalance_report")
    return ImbalanceReport(mx.value, mn.value, sp.value)


def weighted_grad_combine(batch_sizes, grads) -> np.ndarray:
    bs = np.ascontiguousarray(batch_sizes, np.uint64)
    g = np.ascontiguousarray(grads, np.float64)
    if len(bs) == 0 or g.ndim != 2 or g.shape[0] != len(bs):
        raise L.ConfigError("weighted_grad_combine: need matching, non-empty inputs")
    out = np.zeros(g.shape[1], np.float64)
    check(L.lib().rs_weighted_grad_combine(bs.ctypes.data, g.ctypes.data, len(bs), g.shape[1], out.ctypes.data),
          "weighted_grad_combine")
    return out


def weighted_grad_allreduce(batch_size: int, grad, group=None):
    """The dense side of a step across ranks (workload.cpp:583-601 +
    weighted_grad_combine, seq_batcher.cpp:80-138): every rank contributes
    its per-sample mean gradient weighted by its batch size; one all-reduce
    of [b * g, b] (f64, NCCL on GPU tensors / gloo on CPU) gives
    sum_i b_i g_i / sum_i b_i on every rank.  The reduction order is the
    collective's, so the result matches weighted_grad_combine to f64
    rounding, not bit for bit."""
    import torch
    import torch.distributed as dist
    g = torch.as_tensor(grad, dtype=torch.float64)
    if batch_size < 1:
        raise L.ConfigError("weighted_grad_combine: batch sizes must be >= 1")
    buf = torch.empty(g.numel() + 1, dtype=torch.float64, device=g.device)
    buf[:-1] = g.reshape(-1) * float(batch_size)
    buf[-1] = float(batch_size)
    dist.all_reduce(buf, group=group)
    return (buf[:-1] * (1.0 / buf[-1])).reshape(g.shape)
