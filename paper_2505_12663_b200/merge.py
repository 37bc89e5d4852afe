"""Automatic table merging, pooled feature lookup and per-token routing
(host mirror of merge_registry.hpp and run_workload's routing).

Same names, argument meaning and errors as the reference:
``plan_merge`` (merge_registry.cpp:69-110), ``MergeGroup.encode_global_id``
(:48-51), ``HashTableCollection.lookup`` / ``collection_lookup``
(:112-176), ``catalog_from`` (workload.cpp:171-185).  Planning runs in
librsgpu's host code, lookups and routing in its sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import torch

from . import _lib as L
from ._lib import check
from .table import EmbedTable, TableConfig, _ptr, _stream, as_keys


class Pooling(IntEnum):
    NONE = 0
    SUM = 1
    MEAN = 2


@dataclass
class FeatureConfig:
    feature_name: str
    embedding_dim: int
    lookup_tables: list = field(default_factory=list)
    pooling: Pooling = Pooling.NONE

    def c(self):
        """rs_feature_config (the returned tuple keeps the strings alive)."""
        names = [t.encode() for t in self.lookup_tables]
        arr = (C.c_char_p * max(1, len(names)))(*names)
        cf = L.rs_feature_config(self.feature_name.encode(), self.embedding_dim, arr, len(names), int(self.pooling))
        return cf, (names, arr)


def encode_tagged_id(k_bits: int, index: int, index_limit: int, raw_id: int) -> int:
    """merge_registry.cpp:23-33 (host scalar form)."""
    if index > index_limit:
        raise L.RangeError("encode_tagged_id: table index out of range")
    shift = 63 - k_bits
    if raw_id >> shift:
        raise L.RangeError("encode_tagged_id: raw id exceeds payload width")
    return (index << shift) | raw_id


def decode_tagged_id(k_bits: int, index_limit: int, tagged_id: int):
    """merge_registry.cpp:35-46 (host scalar form)."""
    if tagged_id >> 63:
        raise L.RangeError("decode_tagged_id: top bit must be zero")
    shift = 63 - k_bits
    index = tagged_id >> shift
    if index > index_limit:
        raise L.RangeError("decode_tagged_id: table index out of range")
    return index, tagged_id & ((1 << shift) - 1)


@dataclass
class MergeGroup:
    embedding_dim: int
    member_tables: list
    table_index_of: dict
    k_bits: int

    def encode_global_id(self, table_index: int, raw_id: int) -> int:
        return encode_tagged_id(self.k_bits, table_index, len(self.member_tables), raw_id)

    def decode_global_id(self, global_id: int):
        return decode_tagged_id(self.k_bits, len(self.member_tables), global_id)

    def max_raw_id(self) -> int:
        return (1 << (63 - self.k_bits)) - 1


class MergePlan:
    """MergePlan (merge_registry.hpp:62-69) over an rs_merge_plan handle."""

    def __init__(self, handle):
        self._h = handle
        lib = L.lib()
        self.groups = []
        self.group_of_table = {}
        for g in range(lib.rs_merge_plan_groups(handle)):
            dim, k, m = C.c_uint32(), C.c_uint32(), C.c_uint32()
            check(lib.rs_merge_plan_group(handle, g, C.byref(dim), C.byref(k), C.byref(m)), "plan group")
            members = [lib.rs_merge_plan_member(handle, g, i).decode() for i in range(1, m.value + 1)]
            self.groups.append(MergeGroup(dim.value, members, {t: i + 1 for i, t in enumerate(members)}, k.value))
            for t in members:
                self.group_of_table[t] = g

    def group_index_for(self, table_name: str) -> int:
        g, i = C.c_uint32(), C.c_uint32()
        check(L.lib().rs_merge_plan_find(self._h, table_name.encode(), C.byref(g), C.byref(i)), "group_index_for")
        return g.value

    def group_for(self, table_name: str) -> MergeGroup:
        return self.groups[self.group_index_for(table_name)]

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                L.lib().rs_merge_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass


def plan_merge(configs) -> MergePlan:
    cfs = [f.c() for f in configs]
    arr = (L.rs_feature_config * max(1, len(cfs)))(*[c for c, _ in cfs])
    h = C.c_void_p()
    check(L.lib().rs_plan_merge(arr, len(cfs), C.byref(h)), "plan_merge")
    return MergePlan(h)


class _TableView(EmbedTable):
    """Non-owning EmbedTable over a collection's group table."""

    def __init__(self, handle, config: TableConfig):
        self.config = config
        self._h = C.c_void_p(handle)
        self.dim = config.embedding_dim

    def close(self):
        self._h = C.c_void_p()


class HashTableCollection:
    """HashTableCollection (merge_registry.hpp:90-105): one device table per group."""

    def __init__(self, plan: MergePlan, prototype: TableConfig):
        self._plan = plan
        self._h = C.c_void_p()
        check(L.lib().rs_collection_create(plan.handle, C.byref(prototype.c()), C.byref(self._h)),
              "HashTableCollection")
        self._tables = []
        for g in plan.groups:
            cfg = TableConfig(**{**prototype.__dict__, "embedding_dim": g.embedding_dim})
            self._tables.append(_TableView(L.lib().rs_collection_table(self._h, len(self._tables)), cfg))

    def plan(self) -> MergePlan:
        return self._plan

    def table(self, group: int) -> EmbedTable:
        return self._tables[group]

    def group_count(self) -> int:
        return len(self._tables)

    def lookup(self, feature: FeatureConfig, raw_ids) -> torch.Tensor:
        k = as_keys(raw_ids)
        out = torch.empty((k.numel(), feature.embedding_dim), dtype=torch.float32, device="cuda")
        cf, keep = feature.c()
        check(L.lib().rs_collection_lookup(self._h, C.byref(cf), _ptr(k), k.numel(), _ptr(out), _stream()),
              "collection_lookup")
        return out

    def close(self):
        if self._h:
            for t in self._tables:
                t.close()
            L.lib().rs_collection_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def collection_lookup(coll: HashTableCollection, feature: FeatureConfig, raw_ids) -> torch.Tensor:
    return coll.lookup(feature, raw_ids)


def catalog_from(features):
    """TableCatalog (workload.cpp:171-185): names in first-appearance order,
    ordinal (1-based) per name, k_bits = max(1, bit_width(#tables))."""
    names, ordinal_of = [], {}
    for f in features:
        for t in f.lookup_tables:
            if t not in ordinal_of:
                names.append(t)
                ordinal_of[t] = len(names)
    return names, ordinal_of, max(1, len(names).bit_length())


class Router:
    """run_workload's per-token routing (workload.cpp:431-447, 506-531) on the GPU."""

    def __init__(self, plan: MergePlan, catalog_names):
        self.plan = plan
        self.n_groups = len(plan.groups)
        names = [n.encode() for n in catalog_names]
        arr = (C.c_char_p * max(1, len(names)))(*names)
        self._h = C.c_void_p()
        check(L.lib().rs_router_create(plan.handle, arr, len(names), C.byref(self._h)), "Router")

    def route(self, tagged, gids: torch.Tensor | None = None, pos: torch.Tensor | None = None):
        """-> (gids int64 [n], pos int32 [n], counts list): group 0's tokens in
        token order, then group 1's, ...  Synchronizes (range errors raise)."""
        k = as_keys(tagged)
        n = k.numel()
        if gids is None:
            gids = torch.empty(n, dtype=torch.int64, device="cuda")
        if pos is None:
            pos = torch.empty(n, dtype=torch.int32, device="cuda")
        counts = (C.c_uint64 * self.n_groups)()
        check(L.lib().rs_route_tagged(self._h, _ptr(k), n, _ptr(gids), _ptr(pos), counts, _stream()), "route")
        return gids, pos, list(counts)

    def route_async(self, tagged: torch.Tensor, gids: torch.Tensor, pos: torch.Tensor) -> None:
        """Same routing, no synchronization (group sizes known to the caller;
        range errors are not reported)."""
        check(L.lib().rs_route_tagged(self._h, _ptr(tagged), tagged.numel(), _ptr(gids), _ptr(pos), None,
                                      _stream()), "route")

    def __del__(self):
        try:
            if self._h:
                L.lib().rs_router_destroy(self._h)
                self._h = None
        except Exception:
            pass
