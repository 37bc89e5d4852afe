"""ctypes bindings for the CPU checker (TEST INFRASTRUCTURE ONLY).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg.  Two libraries:

* ``liboracle.so`` -- the C restatement (oracle.c), built from this directory;
* ``_ref/librsref.so`` -- the unmodified reference compiled from
  /root/reference/proj sources (built here, travels prebuilt to the GPU box).

Both expose the same shapes of calls; ``Oracle`` wraps either one
(``prefix`` "or_" or "ref_") with numpy-friendly helpers.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "librsref.so")
REF_ROOT = os.environ.get("RS_REF_ROOT", "/root/reference/proj")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
vp = C.c_void_p


def build(ref: bool = True) -> None:
    """Build liboracle.so (and _ref/librsref.so when the reference sources exist)."""
    targets = ["all"]
    if ref and os.path.isdir(os.path.join(REF_ROOT, "src")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, f"REF_ROOT={REF_ROOT}", "-j8", *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(LIB_REF)


def _sig(lib, prefix):
    def f(name, res, *args):
        fn = getattr(lib, prefix + name)
        fn.restype = res
        fn.argtypes = list(args)
        return fn

    return f


class Oracle:
    """numpy wrapper over liboracle (prefix 'or_') or librsref (prefix 'ref_')."""

    def __init__(self, which: str = "oracle"):
        if which == "oracle":
            if not os.path.exists(LIB_ORACLE):
                build(ref=False)
            self.lib = C.CDLL(LIB_ORACLE)
            self.p = "or_"
        else:
            if not os.path.exists(LIB_REF):
                build(ref=True)
            if not os.path.exists(LIB_REF):
                raise FileNotFoundError("reference library unavailable: " + LIB_REF)
            self.lib = C.CDLL(LIB_REF)
            self.p = "ref_"
        self.is_ref = which != "oracle"
        f = _sig(self.lib, self.p)
        f("hash64", C.c_uint64, C.c_uint64)
        f("probe_step", C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64))
        f("table_create", C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_uint32,
          C.POINTER(vp))
        f("table_destroy", None, vp)
        for n in ("capacity", "occupied", "tombstones", "tick"):
            f("table_" + n, C.c_uint64, vp)
        f("table_insert", C.c_int64, vp, C.c_uint64, f32p)
        f("table_lookup", C.c_int64, vp, C.c_uint64)
        f("table_find", C.c_int64, vp, C.c_uint64)
        f("table_ensure", C.c_int64, vp, C.c_uint64)
        f("table_remove", C.c_int, vp, C.c_uint64)
        f("table_expand", C.c_uint64, vp)
        f("stage1_dedup", C.c_uint64 if self.is_ref else C.c_size_t, u64p, C.c_uint64, u64p, i64p)
        f("stage2_dedup", C.c_uint64, u64p, u64p, C.c_uint64, u64p, u64p, u64p, u64p)
        f("shard_of", C.c_uint64, C.c_uint64, C.c_uint64)
        f("cluster_create", C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_double,
          C.c_uint32, C.c_int, C.POINTER(vp))
        f("cluster_destroy", None, vp)
        f("cluster_shard", vp, vp, C.c_uint64)
        f("distributed_lookup", C.c_int, vp, u64p, u64p, f32p, u64p, u64p, u64p, u64p)
        f("accumulate", C.c_uint64, u64p, f32p, C.c_uint64, C.c_uint32, u64p, f32p)
        f("adam_row", None, f32p, f32p, f32p, C.POINTER(C.c_uint64), f32p, C.c_uint32, C.c_double,
          C.c_double, C.c_double, C.c_double)
        f("encode_tagged_id", C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
          C.POINTER(C.c_uint64))
        f("decode_tagged_id", C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
          C.POINTER(C.c_uint64))
        f("closest_prefix", C.c_uint64, u64p, C.c_uint64, C.c_uint64)
        f("sequence_batches", C.c_uint64, u64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p)
        f("generate_workload", C.c_int64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
          C.c_double, C.c_double, C.c_uint32, u64p, u64p, u64p, C.c_uint64)
        f("pseudo_sparse_grad", None, C.c_uint64, C.c_uint64, f32p, C.c_uint32)
        if self.is_ref:
            f("table_export_slots", C.c_uint64, vp, vp, vp, vp, vp, vp, vp)
            f("table_lookup_batch", None, vp, u64p, C.c_uint64, f32p, C.c_int)
            f("table_row", None, vp, C.c_int64, C.c_int, f32p)
            f("accumulate_apply_adam", C.c_uint64, vp, u64p, f32p, C.c_uint64, C.c_double,
              C.c_double, C.c_double, C.c_double, C.c_int)
            f("c1_step", C.c_double, vp, u64p, f32p, C.c_uint64, C.c_int, C.c_double, C.c_double,
              vp)
            f("dist_step", C.c_double, vp, u64p, u64p, f32p, C.c_int, C.c_double, C.c_double)
            f("write_workload_file", C.c_int, C.c_char_p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
              C.c_double, C.c_double, C.c_uint32, u64p)
            f("read_workload_file", C.c_int64, C.c_char_p, u64p, np.ctypeslib.ndpointer(np.float64), u64p, u64p,
              C.c_uint64, C.POINTER(C.c_uint64))
            f("omp_max_threads", C.c_int)
        else:
            f("table_export", C.c_size_t, vp, vp, vp, vp, vp, vp, vp)
            f("table_lookup_batch", None, vp, u64p, C.c_size_t, f32p)
            f("table_emb", C.POINTER(C.c_float), vp, C.c_int64)
            f("table_ensure_batch", C.c_int64, vp, u64p, C.c_size_t, C.c_uint64, C.c_uint64, vp)
            f("table_evict_oldest", C.c_size_t, vp, C.c_size_t)
            f("adagrad_row", None, f32p, f32p, C.POINTER(C.c_uint64), f32p, C.c_uint32,
              C.c_double, C.c_double)
            f("apply", C.c_size_t, vp, u64p, f32p, C.c_size_t, C.c_int, C.c_double, C.c_double,
              C.c_double, C.c_double)
            f("bit_width", C.c_uint32, C.c_uint64)
            f("cost_partition", None, u64p, C.c_size_t, C.c_size_t, C.c_double, C.c_double, u32p)

    def __getattr__(self, name):
        return getattr(self.lib, self.p + name)

    # ---- numpy helpers -------------------------------------------------------
    def stage1(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        uniq = np.zeros(max(len(ids), 1), np.uint64)
        inv = np.zeros(max(len(ids), 1), np.int64)
        n = self.stage1_dedup(ids, len(ids), uniq, inv)
        return uniq[:n].copy(), inv[: len(ids)].copy()

    def stage2(self, lists):
        counts = np.array([len(x) for x in lists], np.uint64)
        recv = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint64) for x in lists])
                                    if len(lists) else np.zeros(0, np.uint64), dtype=np.uint64)
        tot = int(counts.sum())
        uniq = np.zeros(tot + 1, np.uint64)
        off = np.zeros(tot + 2, np.uint64)
        src = np.zeros(tot + 1, np.uint64)
        pos = np.zeros(tot + 1, np.uint64)
        if tot == 0:
            recv = np.zeros(1, np.uint64)
        n = self.stage2_dedup(recv, counts, len(lists), uniq, off, src, pos)
        return uniq[:n].copy(), off[: n + 1].copy(), src[:tot].copy(), pos[:tot].copy()

    def accumulate_np(self, ids, grads, dim):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        grads = np.ascontiguousarray(grads, dtype=np.float32).reshape(-1)
        n = len(ids)
        out_ids = np.zeros(max(n, 1), np.uint64)
        out = np.zeros(max(n, 1) * dim, np.float32)
        k = self.accumulate(ids if n else np.zeros(1, np.uint64),
                            grads if n else np.zeros(dim, np.float32), n, dim, out_ids, out)
        return out_ids[:k].copy(), out[: k * dim].reshape(k, dim).copy()

    def generate(self, seed, num_sequences, mean_len, max_len, sigma, zipf, vocab):
        vocab = np.ascontiguousarray(vocab, dtype=np.uint64)
        lengths = np.zeros(num_sequences, np.uint64)
        cap = int(num_sequences * max(mean_len, 1) * 4 + 1024)
        while True:
            ids = np.zeros(cap, np.uint64)
            t = self.generate_workload(seed, num_sequences, mean_len, max_len, sigma, zipf,
                                       len(vocab), vocab, lengths, ids, cap)
            if t >= 0:
                return lengths, ids[:t].copy()
            if cap > num_sequences * max_len:
                raise ValueError("bad workload config")
            cap *= 2

    def grads(self, sample_id, step, dim):
        out = np.zeros(dim, np.float32)
        self.pseudo_sparse_grad(sample_id, step, out, dim)
        return out

    def token_grads(self, lengths, step, dim, first_sample_id=1):
        """per-token grads: pseudo_sparse_grad(sample_id, step) repeated over the
        sample's tokens (workload.cpp:519-526)."""
        lengths = np.asarray(lengths, np.int64)
        per = np.zeros((len(lengths), dim), np.float32)
        for i in range(len(lengths)):
            self.pseudo_sparse_grad(first_sample_id + i, step, per[i], dim)
        return np.repeat(per, lengths, axis=0)


class Table:
    """Handle over an oracle/ref EmbedTable."""

    def __init__(self, o: Oracle, capacity, dim, groups=1, lf=0.75, chunk_rows=1024, handle=None):
        self.o = o
        self.dim = dim
        self.owned = handle is None
        if handle is None:
            h = vp()
            st = o.table_create(capacity, dim, groups, lf, chunk_rows, C.byref(h))
            if st != 0:
                raise ValueError("table config error")
            handle = h.value
        self.h = handle

    def __del__(self):
        if getattr(self, "owned", False) and self.h:
            self.o.table_destroy(self.h)
            self.h = None

    def insert(self, key, emb):
        return self.o.table_insert(self.h, key, np.ascontiguousarray(emb, np.float32))

    def export(self):
        """live entries sorted by key -> dict of arrays"""
        o, d = self.o, self.dim
        n = int(o.table_occupied(self.h))
        keys = np.zeros(n + 1, np.uint64)
        emb = np.zeros((n + 1) * d, np.float32)
        m = np.zeros((n + 1) * d, np.float32)
        v = np.zeros((n + 1) * d, np.float32)
        step = np.zeros(n + 1, np.uint64)
        ts = np.zeros(n + 1, np.uint64)
        ptrs = [a.ctypes.data for a in (keys, emb, m, v, step, ts)]
        if o.is_ref:
            k = o.table_export_slots(self.h, *ptrs)
        else:
            k = o.table_export(self.h, *ptrs)
        assert k == n
        res = dict(keys=keys[:n], emb=emb[: n * d].reshape(n, d), m=m[: n * d].reshape(n, d),
                   v=v[: n * d].reshape(n, d), step=step[:n], ts=ts[:n])
        if o.is_ref:  # slot order -> key order
            order = np.argsort(res["keys"], kind="stable")
            res = {k2: a[order] for k2, a in res.items()}
        return res
