"""Row-sharded embedding step over the GPUs of one node (host mirror).

Mirrors SimCluster / distributed_lookup (exchange_sim.hpp:61-107) with
DedupMode::kTwoStage, but every "worker" is a process on its own B200:
``ShardedTable`` owns this rank's shard (keys with hash64(key) % W == rank)
and runs the step whose ID / embedding / gradient exchanges are peer stores
over NVLink issued by the kernels themselves (librsgpu ``rs_dist_*``).
torch.distributed is used only to bootstrap (exchange the CUDA IPC handles)
and to gather trace rows.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from ._lib import check
from .table import EmbedTable, TableConfig, _ptr, _stream, as_keys


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All-gather one opaque handle per rank, returned in rank order."""
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, handle, group=group)
    return out


class ShardedTable:
    def __init__(self, config: TableConfig, max_tokens: int, group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.group = group
        self.shard = EmbedTable(config)
        self.dim = config.embedding_dim
        self.max_tokens = max_tokens
        self._c = C.c_void_p()
        check(L.lib().rs_comm_create(self.rank, self.world, max_tokens, self.dim, C.byref(self._c)), "rs_comm_create")
        h = (C.c_char * 64)()
        check(L.lib().rs_comm_ipc_handle(self._c, h), "ipc handle")
        handles = exchange_handles(bytes(h), group)
        buf = (C.c_char * (64 * self.world)).from_buffer_copy(b"".join(handles))
        check(L.lib().rs_comm_open(self._c, buf), "rs_comm_open")

    def owner_of(self, keys: np.ndarray) -> np.ndarray:
        from .table import hash64_batch, keys_to_numpy
        return (keys_to_numpy(hash64_batch(keys)) % np.uint64(self.world)).astype(np.int64)

    def insert_owned(self, keys, emb: torch.Tensor) -> None:
        """Insert the rows whose keys this rank owns (keys/emb given for all ranks)."""
        keys = np.asarray(keys, np.uint64)
        mine = np.nonzero(self.owner_of(keys) == self.rank)[0]
        if len(mine):
            self.shard.insert(keys[mine], emb[torch.from_numpy(mine).to(emb.device)])

    def forward(self, ids, out: torch.Tensor | None = None) -> torch.Tensor:
        k = as_keys(ids)
        if out is None:
            out = torch.empty((k.numel(), self.dim), dtype=torch.float32, device="cuda")
        check(L.lib().rs_dist_forward(self._c, self.shard.handle, _ptr(k), k.numel(), _ptr(out), _stream()),
              "rs_dist_forward")
        return out

    def backward(self, grads: torch.Tensor, params) -> None:
        g = grads.contiguous()
        check(L.lib().rs_dist_backward(self._c, self.shard.handle, _ptr(g), g.shape[0], C.byref(params.c()),
                                       _stream()), "rs_dist_backward")

    def trace_row(self) -> dict:
        ids = np.zeros(self.world, np.uint64)
        embs = np.zeros(self.world, np.uint64)
        lk, rq, rv = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(L.lib().rs_comm_trace(self._c, ids.ctypes.data, embs.ctypes.data, C.byref(lk), C.byref(rq),
                                    C.byref(rv)), "rs_comm_trace")
        return dict(ids_sent=ids, embs_sent=embs, lookups=lk.value, ids_requested=rq.value, ids_received=rv.value)

    def trace(self) -> dict:
        """ExchangeTrace of the last step (all ranks; rows = src)."""
        rows = [None] * self.world
        dist.all_gather_object(rows, self.trace_row(), group=self.group)
        return dict(ids_sent=np.stack([r["ids_sent"] for r in rows]),
                    embs_sent=np.stack([r["embs_sent"] for r in rows]),  # [owner][requester]
                    lookups=np.array([r["lookups"] for r in rows], np.uint64),
                    ids_requested=sum(r["ids_requested"] for r in rows),
                    ids_received=sum(r["ids_received"] for r in rows))

    def close(self):
        if self._c:
            L.lib().rs_comm_destroy(self._c)
            self._c = C.c_void_p()
