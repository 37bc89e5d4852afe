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
from .table import EmbedTable, TableConfig, _ptr, _stream, as_keys, shard_of_batch


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

    def owner_of(self, keys) -> torch.Tensor:
        """shard_of(id, W) = hash64(id) % W per key (exchange_sim.cpp:82-85), on the device."""
        return shard_of_batch(keys, self.world)

    def insert_owned(self, keys, emb: torch.Tensor) -> None:
        """Insert the rows whose keys this rank owns (keys/emb given for all ranks)."""
        k = as_keys(keys)
        mine = torch.nonzero(self.owner_of(k) == self.rank).flatten()
        if mine.numel():
            self.shard.insert(k[mine], emb.to("cuda")[mine])

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

    def step(self, ids, grads: torch.Tensor, params, out: torch.Tensor | None = None,
             checksum: torch.Tensor | None = None) -> torch.Tensor:
        """forward + backward in one call (rs_dist_step); returns the gathered rows.
        checksum (float64, device or pinned host): receives the f64 sum of the
        rows (rs_dist_step_checksum, summed inside the gather kernel)."""
        k = as_keys(ids)
        g = grads.contiguous()
        if out is None:
            out = torch.empty((k.numel(), self.dim), dtype=torch.float32, device="cuda")
        if checksum is not None:
            assert checksum.dtype == torch.float64
            check(L.lib().rs_dist_step_checksum(self._c, self.shard.handle, _ptr(k), k.numel(), _ptr(g), _ptr(out),
                                                C.byref(params.c()), _ptr(checksum), _stream()),
                  "rs_dist_step_checksum")
            return out
        check(L.lib().rs_dist_step(self._c, self.shard.handle, _ptr(k), k.numel(), _ptr(g), _ptr(out),
                                   C.byref(params.c()), _stream()), "rs_dist_step")
        return out

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

    # phases of rs_comm_phase_ms; in the fused step "gather" is the fused
    # gather + segment-reduce + sums-to-owners pass and "req_reduce" is 0
    PHASES = ("req_dedup", "send_ids", "wait_ids", "owner_dedup", "owner_table_respond", "wait_embs", "gather",
              "req_reduce", "wait_grads", "owner_update")

    def barrier(self) -> None:
        """Device-side barrier of the group on the current stream."""
        check(L.lib().rs_comm_barrier(self._c, _stream()), "rs_comm_barrier")

    def set_profiling(self, on: bool) -> None:
        check(L.lib().rs_comm_set_profiling(self._c, int(on)), "rs_comm_set_profiling")

    def phase_ms(self) -> dict:
        ms = (C.c_double * len(self.PHASES))()
        cnt = C.c_uint64()
        check(L.lib().rs_comm_phase_ms(self._c, ms, len(self.PHASES), C.byref(cnt)), "rs_comm_phase_ms")
        return {k: ms[i] for i, k in enumerate(self.PHASES)}

    def close(self):
        if self._c:
            L.lib().rs_comm_destroy(self._c)
            self._c = C.c_void_p()


class LocalShardGroup:
    """W logical ranks of the sharded step on the current GPU (one process).

    The reference's SimCluster (exchange_sim.hpp:63-75: W shards in one
    process, distributed_lookup exchange_sim.cpp:117-233) run on the sharded
    step's own kernels, arena layout and flag protocol
    (rs_comm_create_local / rs_dist_group_*): every rank's phases are enqueued
    on one stream in data-flow order, so the W-rank data path -- owner
    routing, stage-2 dedup, find-or-insert at the owner, the embedding and
    gradient exchanges, the owner's ordered update -- is exercised on one GPU.
    shards[r] owns the keys with hash64(key) % W == r."""

    def __init__(self, config: TableConfig, world: int, max_tokens: int):
        self.world, self.dim, self.max_tokens = world, config.embedding_dim, max_tokens
        self.shards = [EmbedTable(config) for _ in range(world)]
        self._cs = (C.c_void_p * world)()
        check(L.lib().rs_comm_create_local(world, max_tokens, self.dim, self._cs), "rs_comm_create_local")
        self._ts = (C.c_void_p * world)(*[s.handle for s in self.shards])

    def insert_all(self, keys, emb: torch.Tensor) -> None:
        """Insert every row into the shard that owns its key."""
        k = as_keys(keys)
        own = shard_of_batch(k, self.world)
        e = emb.to("cuda")
        for r in range(self.world):
            sel = torch.nonzero(own == r).flatten()
            if sel.numel():
                self.shards[r].insert(k[sel], e[sel])

    def _arrays(self, ids):
        ks = [as_keys(i) for i in ids]
        n = (C.c_uint64 * self.world)(*[k.numel() for k in ks])
        return ks, n

    def forward(self, ids: list) -> list:
        ks, n = self._arrays(ids)
        outs = [torch.empty((k.numel(), self.dim), dtype=torch.float32, device="cuda") for k in ks]
        pi = (C.c_void_p * self.world)(*[_ptr(k) for k in ks])
        po = (C.c_void_p * self.world)(*[_ptr(o) for o in outs])
        check(L.lib().rs_dist_group_forward(self._cs, self._ts, self.world, pi, n, po, _stream()),
              "rs_dist_group_forward")
        self._keep = ks
        return outs

    def backward(self, grads: list, params) -> None:
        gs = [g.to("cuda", torch.float32).contiguous() for g in grads]
        n = (C.c_uint64 * self.world)(*[g.shape[0] for g in gs])
        pg = (C.c_void_p * self.world)(*[_ptr(g) for g in gs])
        check(L.lib().rs_dist_group_backward(self._cs, self._ts, self.world, pg, n, C.byref(params.c()), _stream()),
              "rs_dist_group_backward")
        torch.cuda.current_stream().synchronize()  # keeps gs alive until the kernels read them

    def step(self, ids: list, grads: list, params) -> list:
        ks, n = self._arrays(ids)
        gs = [g.to("cuda", torch.float32).contiguous() for g in grads]
        outs = [torch.empty((k.numel(), self.dim), dtype=torch.float32, device="cuda") for k in ks]
        pi = (C.c_void_p * self.world)(*[_ptr(k) for k in ks])
        pg = (C.c_void_p * self.world)(*[_ptr(g) for g in gs])
        po = (C.c_void_p * self.world)(*[_ptr(o) for o in outs])
        check(L.lib().rs_dist_group_step(self._cs, self._ts, self.world, pi, n, pg, po, C.byref(params.c()),
                                         _stream()), "rs_dist_group_step")
        torch.cuda.current_stream().synchronize()
        return outs

    def trace(self) -> dict:
        """ExchangeTrace of the last step (rows = src), as ShardedTable.trace()."""
        rows = []
        for r in range(self.world):
            ids = np.zeros(self.world, np.uint64)
            embs = np.zeros(self.world, np.uint64)
            lk, rq, rv = C.c_uint64(), C.c_uint64(), C.c_uint64()
            check(L.lib().rs_comm_trace(self._cs[r], ids.ctypes.data, embs.ctypes.data, C.byref(lk), C.byref(rq),
                                        C.byref(rv)), "rs_comm_trace")
            rows.append(dict(ids_sent=ids, embs_sent=embs, lookups=lk.value, ids_requested=rq.value,
                             ids_received=rv.value))
        return dict(ids_sent=np.stack([r["ids_sent"] for r in rows]),
                    embs_sent=np.stack([r["embs_sent"] for r in rows]),
                    lookups=np.array([r["lookups"] for r in rows], np.uint64),
                    ids_requested=sum(r["ids_requested"] for r in rows),
                    ids_received=sum(r["ids_received"] for r in rows))

    def close(self):
        for r in range(self.world):
            if self._cs[r]:
                L.lib().rs_comm_destroy(self._cs[r])
                self._cs[r] = None
