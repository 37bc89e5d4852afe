"""CPU restatement of the reference's table merging, pooling and per-token
routing (TEST INFRASTRUCTURE ONLY -- imported by tests/ and smoke(); never by
the product).

Follows /root/reference/proj/src/merge_registry.cpp and workload.cpp:
  * plan_merge            merge_registry.cpp:69-110
  * encode / decode       merge_registry.cpp:23-51 (oracle.c or_encode/decode)
  * collection_lookup     merge_registry.cpp:112-158 (per raw id, per lookup
                          table in order: ensure(gid) then pool; mean = sum *
                          (1.0f / n))
  * catalog_from          workload.cpp:171-185
  * route_tagged          workload.cpp:431-447 (cluster/member maps) and
                          :506-531 (per token decode + re-encode into the
                          group's id space, requests in token order)
Pinned against the compiled reference (oracle/_ref, ref_plan_merge /
ref_collection_*) in tests/test_merge.py.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

NONE, SUM, MEAN = 0, 1, 2


class ConfigError(ValueError):
    pass


class RangeError(ValueError):
    pass


@dataclass
class Feature:
    name: str
    dim: int
    tables: list
    pooling: int = NONE


@dataclass
class Group:
    dim: int
    members: list = field(default_factory=list)
    index_of: dict = field(default_factory=dict)
    k_bits: int = 0


def bit_width(x: int) -> int:
    return int(x).bit_length()


def plan_merge(features):
    """merge_registry.cpp:69-110 -- groups by dim in first-appearance order."""
    groups, group_of_table, group_of_dim, seen = [], {}, {}, set()
    for f in features:
        if not f.name:
            raise ConfigError("feature with empty name")
        if f.name in seen:
            raise ConfigError("duplicate feature name: " + f.name)
        seen.add(f.name)
        if f.dim == 0:
            raise ConfigError(f"feature {f.name}: embedding_dim must be >= 1")
        if not f.tables:
            raise ConfigError(f"feature {f.name}: lookup_tables must be non-empty")
        for t in f.tables:
            if t in group_of_table:
                if groups[group_of_table[t]].dim != f.dim:
                    raise ConfigError("logical table " + t + " referenced with conflicting embedding dims")
                continue
            if f.dim not in group_of_dim:
                group_of_dim[f.dim] = len(groups)
                groups.append(Group(f.dim))
            g = groups[group_of_dim[f.dim]]
            g.members.append(t)
            g.index_of[t] = len(g.members)
            group_of_table[t] = group_of_dim[f.dim]
    for g in groups:
        g.k_bits = bit_width(len(g.members))  # ceil(log2(m + 1)) for m >= 1
    return groups, group_of_table


def encode(k_bits: int, index: int, limit: int, raw: int) -> int:
    """encode_tagged_id (merge_registry.cpp:23-33)."""
    if index > limit:
        raise RangeError("encode_tagged_id: table index out of range")
    shift = 63 - k_bits
    if raw >> shift:
        raise RangeError("encode_tagged_id: raw id exceeds payload width")
    return (index << shift) | raw


def decode(k_bits: int, limit: int, tagged: int):
    """decode_tagged_id (merge_registry.cpp:35-46)."""
    if tagged >> 63:
        raise RangeError("decode_tagged_id: top bit must be zero")
    shift = 63 - k_bits
    index = tagged >> shift
    if index > limit:
        raise RangeError("decode_tagged_id: table index out of range")
    return index, tagged & ((1 << shift) - 1)


def collection_lookup(o, groups, group_of_table, tables, feature, raw_ids):
    """merge_registry.cpp:112-158 on oracle tables (one or_table per group)."""
    if feature.pooling == NONE and len(feature.tables) != 1:
        raise ConfigError(f"feature {feature.name}: pooling=none requires exactly one lookup table")
    if len(tables) != len(groups):
        raise ConfigError("collection_lookup: one table per plan group required")
    resolved = []
    for name in feature.tables:
        if name not in group_of_table:
            raise ConfigError("unknown logical table: " + name)
        g = group_of_table[name]
        resolved.append((g, groups[g].index_of[name]))
    dim = feature.dim
    out = np.zeros((len(raw_ids), dim), np.float32)
    for t, raw in enumerate(np.asarray(raw_ids, np.uint64)):
        pooled = np.zeros(dim, np.float32)
        for g, idx in resolved:
            grp = groups[g]
            gid = encode(grp.k_bits, idx, len(grp.members), int(raw))
            row = o.table_ensure(tables[g], gid)
            emb = np.ctypeslib.as_array(o.table_emb(tables[g], row), (grp.dim,))
            if feature.pooling == NONE:
                pooled[:] = emb
            else:
                pooled += emb
        if feature.pooling == MEAN:
            pooled *= np.float32(1.0) / np.float32(len(resolved))
        out[t] = pooled
    return out


def catalog_from(features):
    """workload.cpp:171-185: ordinal (1-based) of every logical table, k bits."""
    names, ordinal_of = [], {}
    for f in features:
        for t in f.tables:
            if t not in ordinal_of:
                names.append(t)
                ordinal_of[t] = len(names)
    return names, ordinal_of, max(1, bit_width(len(names)))


def route_maps(features):
    """workload.cpp:431-447 with merging on: group and member index per ordinal."""
    groups, gof = plan_merge(features)
    names, _, _ = catalog_from(features)
    group_of_ord = np.zeros(len(names) + 1, np.uint32)
    member_of_ord = np.zeros(len(names) + 1, np.uint32)
    for ord_, name in enumerate(names, start=1):
        group_of_ord[ord_] = gof[name]
        member_of_ord[ord_] = groups[gof[name]].index_of[name]
    return groups, group_of_ord, member_of_ord


def route_tagged(tagged, features):
    """workload.cpp:506-531: per token decode the catalog tag, re-encode into
    the merged group's id space; per group the ids in token order and their
    token positions."""
    groups, group_of_ord, member_of_ord = route_maps(features)
    names, _, cat_k = catalog_from(features)
    per_ids = [[] for _ in groups]
    per_pos = [[] for _ in groups]
    for t, x in enumerate(np.asarray(tagged, np.uint64)):
        ordinal, raw = decode(cat_k, len(names), int(x))
        g = int(group_of_ord[ordinal])
        grp = groups[g]
        per_ids[g].append(encode(grp.k_bits, int(member_of_ord[ordinal]), len(grp.members), raw))
        per_pos[g].append(t)
    return ([np.array(x, np.uint64) for x in per_ids], [np.array(x, np.int64) for x in per_pos])


def route_tagged_np(tagged, features):
    """route_tagged, vectorised (numpy) for large token counts; same result."""
    groups, group_of_ord, member_of_ord = route_maps(features)
    names, _, cat_k = catalog_from(features)
    x = np.asarray(tagged, np.uint64)
    assert not np.any(x >> np.uint64(63)), "decode_tagged_id: top bit must be zero"
    ords = (x >> np.uint64(63 - cat_k)).astype(np.int64)
    assert ords.max(initial=0) <= len(names), "decode_tagged_id: table index out of range"
    raw = x & np.uint64((1 << (63 - cat_k)) - 1)
    g = group_of_ord[ords]
    ids, pos = [], []
    for gi, grp in enumerate(groups):
        sel = np.nonzero(g == gi)[0]
        sh = np.uint64(63 - grp.k_bits)
        assert not np.any(raw[sel] >> sh), "encode_tagged_id: raw id exceeds payload width"
        ids.append((member_of_ord[ords[sel]].astype(np.uint64) << sh) | raw[sel])
        pos.append(sel.astype(np.int64))
    return ids, pos


def spec_string(features) -> str:
    """features -> the ref shim's text spec (oracle/ref_shim.cpp parse_features)."""
    return ";".join(f"{f.name}|{f.dim}|{f.pooling}|{','.join(f.tables)}" for f in features)


def ref_plan(ref, features):
    """The compiled reference's plan_merge as [(dim, k, members)] or ConfigError."""
    buf = C.create_string_buffer(1 << 16)
    fn = ref.lib.ref_plan_merge
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64]
    st = fn(spec_string(features).encode(), buf, len(buf))
    if st:
        raise ConfigError(f"reference plan_merge status {st}")
    out = []
    for part in buf.value.decode().split("|") if buf.value else []:
        dim, k, members = part.split(":")
        out.append((int(dim), int(k), members.split(",")))
    return out
