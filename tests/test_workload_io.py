"""Workload text ingest: rs_workload_write / rs_workload_read
against the reference's own generate_workload_file / read_workload_file
(workload.cpp:280-339), compiled from its sources (oracle/_ref).  Host code of
librsgpu.so: runs without a GPU."""
import numpy as np
import pytest

import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import workload as W


def _ref_read(ref, path, n_seq_cap=100000, tok_cap=1 << 22):
    import ctypes as C
    sid = np.zeros(n_seq_cap, np.uint64)
    lab = np.zeros(n_seq_cap, np.float64)
    ln = np.zeros(n_seq_cap, np.uint64)
    ids = np.zeros(tok_cap, np.uint64)
    nt = C.c_uint64()
    n = ref.read_workload_file(str(path).encode(), sid, lab, ln, ids, tok_cap, C.byref(nt))
    return n, sid[:max(n, 0)], lab[:max(n, 0)], ln[:max(n, 0)], ids[: nt.value]


@pytest.mark.parametrize("tables,vocab", [(1, [1 << 20]), (3, [1000, 50, 7])])
def test_write_is_byte_identical_and_read_matches_reference(ref, tmp_path, tables, vocab):
    args = (7, 300, 32.0, 512, 1.0, 1.1)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    W.write_workload_file(ours, *args, vocab)
    assert ref.write_workload_file(str(theirs).encode(), *args, tables, np.asarray(vocab, np.uint64)) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    sid, lab, ln, ids = W.read_workload_file(theirs)
    n, rsid, rlab, rln, rids = _ref_read(ref, theirs)
    assert n == 300
    np.testing.assert_array_equal(sid, rsid)
    np.testing.assert_array_equal(lab.astype(np.float32), rlab.astype(np.float32))  # SequenceSample::label is float
    np.testing.assert_array_equal(ln, rln)
    np.testing.assert_array_equal(ids, rids)
    # the file holds exactly the generator's batch
    gl, gids = W.generate(*args, vocab)
    np.testing.assert_array_equal(ln, gl)
    np.testing.assert_array_equal(ids, gids)


def test_read_errors_and_comments_like_reference(ref, tmp_path):
    good = tmp_path / "good.txt"
    good.write_text("# header\n\n5\t0.5000\t1 2 3\n# mid comment\n9\t0.2500\t42\n")
    sid, lab, ln, ids = W.read_workload_file(good)
    assert sid.tolist() == [5, 9] and ln.tolist() == [3, 1] and ids.tolist() == [1, 2, 3, 42]
    assert _ref_read(ref, good)[0] == 2
    for text in ("5\t0.5\t\n", "x y 1 2\n", "7\n"):
        bad = tmp_path / "bad.txt"
        bad.write_text(text)
        with pytest.raises(P.IoError, match=":1:"):
            W.read_workload_file(bad)
        assert _ref_read(ref, bad)[0] == -3  # IoError in the reference too
    with pytest.raises(P.IoError):
        W.read_workload_file(tmp_path / "missing.txt")
