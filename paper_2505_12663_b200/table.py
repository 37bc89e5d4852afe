"""Host mirror of the reference table / dedup / optimizer API over the C-ABI.

Mirrors /root/reference/proj/include/recsparse/{embed_table,exchange_sim,
sparse_update}.hpp: same class names, argument meaning and error behaviour
(exceptions of the same taxonomy), but batched and device-resident: keys are
torch int64 tensors holding the u64 bit patterns, rows are CUDA tensors.
Everything executes in librsgpu.so kernels; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from ._lib import check


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def as_keys(keys) -> torch.Tensor:
    """u64 ids (numpy uint64 / python ints / int64 tensor) -> CUDA int64 tensor (same bits)."""
    if isinstance(keys, torch.Tensor):
        if keys.dtype == torch.uint64:
            keys = keys.view(torch.int64)
        return keys.to(device="cuda", dtype=torch.int64).contiguous()
    a = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64)).view(np.int64)
    return torch.from_numpy(a.copy()).to("cuda")


def keys_to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


_OPT = {"none": L.RS_OPT_NONE, "adam": L.RS_OPT_ADAM, "adagrad": L.RS_OPT_ADAGRAD}


@dataclass
class TableConfig:
    """TableConfig (embed_table.hpp:28-36) + GPU extensions (optimizer state, bound)."""
    capacity: int = 1024
    embedding_dim: int = 16
    thread_groups: int = 1
    max_load_factor: float = 0.75
    chunk_rows: int = 1024
    optimizer: str = "adam"
    initial_rows: int = 0
    max_keys: int = 0

    def c(self) -> L.rs_table_config:
        if self.optimizer not in _OPT:
            raise L.ConfigError(f"unknown optimizer {self.optimizer!r}")
        return L.rs_table_config(self.capacity, self.embedding_dim, self.thread_groups,
                                 self.max_load_factor, self.chunk_rows, _OPT[self.optimizer],
                                 self.initial_rows, self.max_keys)


@dataclass
class AdamParams:
    """AdamParams (sparse_update.hpp:26-31)."""
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def c(self):
        return L.rs_optimizer_params(L.RS_OPT_ADAM, self.lr, self.beta1, self.beta2, self.eps)


@dataclass
class AdagradParams:
    """Adagrad (no reference counterpart): acc += g^2; w -= lr*g/(sqrt(acc)+eps)."""
    lr: float = 0.01
    eps: float = 1e-8

    def c(self):
        return L.rs_optimizer_params(L.RS_OPT_ADAGRAD, self.lr, 0.0, 0.0, self.eps)


class EmbedTable:
    """Dynamic hash embedding table on the GPU (EmbedTable, embed_table.hpp:73-211)."""

    def __init__(self, config: TableConfig):
        self.config = config
        self._h = C.c_void_p()
        check(L.lib().rs_table_create(C.byref(config.c()), C.byref(self._h)), "EmbedTable")
        self.dim = config.embedding_dim

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            L.lib().rs_table_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- observers (embed_table.hpp:108-118); synchronizing
    def info(self) -> L.rs_table_info:
        out = L.rs_table_info()
        check(L.lib().rs_table_stats(self._h, C.byref(out)), "stats")
        return out

    def capacity(self) -> int:
        return self.info().capacity

    def occupied(self) -> int:
        return self.info().occupied

    def tombstones(self) -> int:
        return self.info().tombstones

    def tick(self) -> int:
        return self.info().tick

    def load_factor(self) -> float:
        i = self.info()
        return (i.occupied + i.tombstones) / i.capacity

    # -- batched operations
    def insert(self, keys, emb: torch.Tensor) -> None:
        k = as_keys(keys)
        emb = emb.to(device="cuda", dtype=torch.float32).contiguous()
        if emb.numel() != k.numel() * self.dim:
            raise L.ConfigError("insert: embedding length != embedding_dim")
        check(L.lib().rs_table_insert(self._h, _ptr(k), k.numel(), _ptr(emb), _stream()), "insert")

    def find(self, keys) -> torch.Tensor:
        k = as_keys(keys)
        rows = torch.empty(k.numel(), dtype=torch.int64, device="cuda")
        check(L.lib().rs_table_find(self._h, _ptr(k), k.numel(), _ptr(rows), _stream()), "find")
        return rows

    def lookup_batch(self, keys) -> torch.Tensor:
        k = as_keys(keys)
        out = torch.empty((k.numel(), self.dim), dtype=torch.float32, device="cuda")
        check(L.lib().rs_table_lookup(self._h, _ptr(k), k.numel(), _ptr(out), _stream()), "lookup_batch")
        return out

    def ensure(self, keys) -> torch.Tensor:
        k = as_keys(keys)
        rows = torch.empty(k.numel(), dtype=torch.int64, device="cuda")
        check(L.lib().rs_table_ensure(self._h, _ptr(k), k.numel(), _ptr(rows), _stream()), "ensure")
        return rows

    def remove(self, keys) -> torch.Tensor:
        k = as_keys(keys)
        out = torch.empty(k.numel(), dtype=torch.uint8, device="cuda")
        check(L.lib().rs_table_remove(self._h, _ptr(k), k.numel(), _ptr(out), _stream()), "remove")
        return out.bool()

    def expand(self) -> int:
        nc = C.c_uint64()
        check(L.lib().rs_table_expand(self._h, C.byref(nc), _stream()), "expand")
        return nc.value

    def evict(self, k: int) -> int:
        ev = C.c_uint64()
        check(L.lib().rs_table_evict(self._h, k, C.byref(ev), _stream()), "evict")
        return ev.value

    def gather_rows(self, rows: torch.Tensor) -> torch.Tensor:
        rows = rows.to(device="cuda", dtype=torch.int64).contiguous()
        out = torch.empty((rows.numel(), self.dim), dtype=torch.float32, device="cuda")
        check(L.lib().rs_table_gather_rows(self._h, _ptr(rows), rows.numel(), _ptr(out), _stream()),
              "gather_rows")
        return out

    def export(self) -> dict:
        """Live entries sorted by key: keys(u64), emb, m, v, step, ts (numpy)."""
        torch.cuda.synchronize()
        n = C.c_uint64()
        check(L.lib().rs_table_export(self._h, 0, None, None, None, None, None, None, C.byref(n)), "export")
        k = n.value
        d = self.dim
        keys = np.zeros(max(k, 1), np.uint64)
        emb = np.zeros((max(k, 1), d), np.float32)
        m = np.zeros((max(k, 1), d), np.float32)
        v = np.zeros((max(k, 1), d), np.float32)
        step = np.zeros(max(k, 1), np.uint64)
        ts = np.zeros(max(k, 1), np.uint64)
        if k:
            check(L.lib().rs_table_export(self._h, k, keys.ctypes.data, emb.ctypes.data, m.ctypes.data,
                                          v.ctypes.data, step.ctypes.data, ts.ctypes.data, C.byref(n)),
                  "export")
        return dict(keys=keys[:k], emb=emb[:k], m=m[:k], v=v[:k], step=step[:k], ts=ts[:k])

    def import_entries(self, keys, emb, m=None, v=None, step=None, ts=None) -> None:
        keys = np.ascontiguousarray(keys, np.uint64)
        n = len(keys)
        emb = np.ascontiguousarray(emb, np.float32)
        arr = lambda a, t: None if a is None else np.ascontiguousarray(a, t)
        m, v = arr(m, np.float32), arr(v, np.float32)
        step, ts = arr(step, np.uint64), arr(ts, np.uint64)
        p = lambda a: None if a is None else a.ctypes.data
        check(L.lib().rs_table_import(self._h, n, p(keys), p(emb), p(m), p(v), p(step), p(ts)), "import")


class Workspace:
    """Per-stream scratch of the dedup / step kernels (max_tokens ids per call)."""

    def __init__(self, max_tokens: int):
        self._h = C.c_void_p()
        self.max_tokens = max_tokens
        check(L.lib().rs_workspace_create(max_tokens, C.byref(self._h)), "Workspace")

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            L.lib().rs_workspace_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def results(self):
        """device pointers of the last forward: (unique, inverse, n_unique, rows)."""
        u, inv, n, r = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.lib().rs_workspace_results(self._h, C.byref(u), C.byref(inv), C.byref(n), C.byref(r)),
              "results")
        return u.value, inv.value, n.value, r.value


def stage1_dedup(ids, ws: Workspace | None = None):
    """stage1_dedup (exchange_sim.cpp:87-98): (unique ids int64-bits, inverse int32), CUDA tensors."""
    k = as_keys(ids)
    n = k.numel()
    ws = ws or Workspace(max(n, 1))
    uniq = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    inv = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    nu = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(L.lib().rs_dedup(ws.handle, _ptr(k), n, _ptr(uniq), _ptr(inv), _ptr(nu), _stream()), "dedup")
    m = int(nu.item())
    return uniq[:m], inv[:n]


class SparseStep:
    """One shard's fused training step: dedup -> find-or-insert -> gather (forward),
    segment-reduce + optimizer (backward).  Reference caller: run_workload
    (workload.cpp:506-581) with distributed_lookup at W = 1."""

    def __init__(self, table: EmbedTable, max_tokens: int, params=None):
        self.table = table
        self.ws = Workspace(max_tokens)
        self.params = params or AdagradParams()

    def forward(self, ids: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        k = as_keys(ids)
        if out is None:
            out = torch.empty((k.numel(), self.table.dim), dtype=torch.float32, device="cuda")
        check(L.lib().rs_forward(self.ws.handle, self.table.handle, _ptr(k), k.numel(), _ptr(out), _stream()),
              "forward")
        return out

    def backward(self, grads: torch.Tensor) -> None:
        g = grads.contiguous()
        n = g.shape[0]
        check(L.lib().rs_backward(self.ws.handle, self.table.handle, _ptr(g), n, C.byref(self.params.c()),
                                  _stream()), "backward")

    def _check(self, ids, grads, out):
        """The C-ABI reads raw device pointers: reject anything it would misread."""
        d = self.table.dim
        ok = (isinstance(ids, torch.Tensor) and ids.is_cuda and ids.dtype in (torch.int64, torch.uint64)
              and ids.is_contiguous() and ids.dim() == 1)
        n = ids.numel() if ok else -1
        for t in (grads, out):
            ok = ok and (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                         and tuple(t.shape) == (n, d))
        if not ok:
            raise L.ConfigError("SparseStep: ids must be a contiguous 1-D int64 CUDA tensor of n keys (as_keys), "
                              "grads / out contiguous float32 CUDA tensors of shape (n, embedding_dim)")

    def step(self, ids: torch.Tensor, grads: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        self._check(ids, grads, out)
        check(L.lib().rs_step(self.ws.handle, self.table.handle, _ptr(ids), ids.numel(), _ptr(grads),
                              _ptr(out), C.byref(self.params.c()), _stream()), "step")
        return out

    def step_checksum(self, ids: torch.Tensor, grads: torch.Tensor, out: torch.Tensor,
                      checksum: torch.Tensor) -> torch.Tensor:
        """step() + checksum[0] (device float64) = sum of every value written to
        out (run_workload's emb_checksum, workload.cpp:547-549), summed in the
        gather kernel."""
        assert checksum.dtype == torch.float64 and checksum.is_cuda
        self._check(ids, grads, out)
        check(L.lib().rs_step_checksum(self.ws.handle, self.table.handle, _ptr(ids), ids.numel(), _ptr(grads),
                                       _ptr(out), C.byref(self.params.c()), _ptr(checksum), _stream()),
              "step_checksum")
        return out

    def last_unique(self) -> torch.Tensor:
        """unique ids of the last forward, indexed like accumulate()'s rows."""
        n = C.c_uint64()
        check(L.lib().rs_workspace_unique(self.ws.handle, None, 0, C.byref(n)), "last_unique")
        out = torch.empty(max(n.value, 1), dtype=torch.int64, device="cuda")
        check(L.lib().rs_workspace_unique(self.ws.handle, _ptr(out), out.numel(), C.byref(n)), "last_unique")
        return out[: n.value]

    def accumulate(self, grads: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
        """aggregated grads of the last forward's unique ids (first-occurrence order)."""
        g = grads.contiguous()
        n = g.shape[0]
        sums = torch.empty((n, self.table.dim), dtype=torch.float32, device="cuda")
        check(L.lib().rs_accumulate(self.ws.handle, _ptr(g), n, _ptr(sums), _stream()), "accumulate")
        return sums


def sparse_update(table: EmbedTable, ws: Workspace, ids: torch.Tensor, grads: torch.Tensor, params) -> None:
    """GradAccumulator::accumulate + apply (sparse_update.cpp:45-83) for one window."""
    k = as_keys(ids)
    g = grads.contiguous()
    check(L.lib().rs_sparse_update(ws.handle, table.handle, _ptr(k), k.numel(), _ptr(g), C.byref(params.c()),
                                   _stream()), "sparse_update")


def apply_aggregated(table: EmbedTable, keys, sums: torch.Tensor, params) -> None:
    """GradAccumulator::apply given the pending map (sparse_update.cpp:58-83)."""
    k = as_keys(keys)
    s = sums.to(device="cuda", dtype=torch.float32).contiguous()
    check(L.lib().rs_apply_aggregated(table.handle, _ptr(k), k.numel(), _ptr(s), C.byref(params.c()),
                                      _stream()), "apply_aggregated")


def hash64_batch(keys) -> torch.Tensor:
    k = as_keys(keys)
    out = torch.empty_like(k)
    check(L.lib().rs_hash64_batch(_ptr(k), k.numel(), _ptr(out), _stream()), "hash64_batch")
    return out


def shard_of_batch(ids, world: int) -> torch.Tensor:
    k = as_keys(ids)
    out = torch.empty(k.numel(), dtype=torch.int32, device="cuda")
    check(L.lib().rs_shard_of_batch(_ptr(k), k.numel(), world, _ptr(out), _stream()), "shard_of")
    return out
