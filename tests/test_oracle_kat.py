"""The C restatement (oracle/oracle.c) against the reference's own known-answer
vectors (tests/golden/kat.json, transcribed with file:line citations)."""
import ctypes as C

import numpy as np
import pytest

from oracle.bind import Table


def test_hash64_kat(oracle, kat):
    for k, h in kat["hash64"]["cases"]:
        assert oracle.hash64(k) == h


def test_probe_step_kat(oracle, kat):
    out = C.c_uint64()
    for key, cap, g, want in kat["probe_step"]["cases"]:
        assert oracle.probe_step(key, cap, g, C.byref(out)) == 0
        assert out.value == want
    for key, cap, g in kat["probe_step"]["errors"]["cases"]:
        assert oracle.probe_step(key, cap, g, C.byref(out)) == 1


def test_stage1_kat(oracle, kat):
    for ids, uniq, inv in kat["stage1_dedup"]["cases"]:
        u, i = oracle.stage1(np.array(ids, np.uint64))
        assert u.tolist() == uniq and i.tolist() == inv


def test_stage2_kat(oracle, kat):
    for lists, uniq, origins in kat["stage2_dedup"]["cases"]:
        u, off, src, pos = oracle.stage2(lists)
        assert u.tolist() == uniq
        got = [[[int(src[o]), int(pos[o])] for o in range(off[k], off[k + 1])] for k in range(len(u))]
        assert got == origins


def test_encode_kat(oracle, kat):
    e = kat["encode_tagged_id"]
    out = C.c_uint64()
    for idx, raw, want in e["encode"]:
        assert oracle.encode_tagged_id(e["k_bits"], idx, e["index_limit"], raw, C.byref(out)) == 0
        assert out.value == want
    for idx, raw in e["overflow"]:
        assert oracle.encode_tagged_id(e["k_bits"], idx, e["index_limit"], raw, C.byref(out)) == 2
    for idx, raw in e["bad_index"]:
        assert oracle.encode_tagged_id(e["k_bits"], idx, e["index_limit"], raw, C.byref(out)) == 1
    i, x = C.c_uint32(), C.c_uint64()
    for tagged, idx, raw in e["decode"]:
        assert oracle.decode_tagged_id(e["k_bits"], e["index_limit"], tagged, C.byref(i), C.byref(x)) == 0
        assert (i.value, x.value) == (idx, raw)
    assert oracle.decode_tagged_id(2, 3, 1 << 63, C.byref(i), C.byref(x)) == 1
    for m, k in kat["plan_merge"]["k_bits"]:
        assert oracle.bit_width(m) == k


def test_adam_kat(oracle, kat):
    a = kat["adam_one_step"]
    w = np.array([a["w"]], np.float32)
    m = np.zeros(1, np.float32)
    v = np.zeros(1, np.float32)
    step = C.c_uint64(0)
    oracle.adam_row(w, m, v, C.byref(step), np.array([a["g"]], np.float32), 1, a["lr"], a["beta1"],
                    a["beta2"], a["eps"])
    assert step.value == 1
    assert abs(float(w[0]) - a["w_out"]) < a["tol"][0]
    assert abs(float(m[0]) - a["m_out"]) < a["tol"][1]
    assert abs(float(v[0]) - a["v_out"]) < a["tol"][2]


def test_accumulate_kat(oracle, kat):
    for ids, grads, dim, want_ids, want in kat["accumulate"]["cases"]:
        i, s = oracle.accumulate_np(np.array(ids, np.uint64), np.array(grads, np.float32), dim)
        assert i.tolist() == want_ids
        assert s.reshape(-1).tolist() == want


def test_closest_prefix_kat(oracle, kat):
    for cums, target, want in kat["closest_prefix"]["cases"]:
        assert oracle.closest_prefix(np.array(cums, np.uint64), len(cums), target) == want


def test_table_threshold_and_load_factor_kat(oracle, kat):
    k = kat["table_threshold"]
    t = Table(oracle, k["capacity"], k["dim"], lf=k["lf"], chunk_rows=4)
    for key in range(k["inserts_before"]):
        t.insert(key, np.full(4, key, np.float32))
    assert oracle.table_capacity(t.h) == k["capacity"]
    t.insert(6, np.full(4, 6, np.float32))
    assert oracle.table_capacity(t.h) == k["capacity_after_7th"]
    k = kat["table_load_factor"]
    t = Table(oracle, k["capacity"], 4, chunk_rows=4)
    for key in k["insert"]:
        t.insert(key, np.zeros(4, np.float32))
    for key in k["remove"]:
        assert oracle.table_remove(t.h, key) == 1
    assert oracle.table_occupied(t.h) == k["occupied"]
    assert oracle.table_tombstones(t.h) == k["tombstones"]
