"""The reference's own unit suites relinked against the GPU build.

oracle/Makefile (`make -C oracle suites`) compiles the reference's test
sources where they lie (proj/tests/test_{hash,sparse_update,exchange_sim,
embed_table}.cpp, unchanged) with a minimal GoogleTest-compatible harness
(oracle/gtest_shim) twice:
  *.ref -- linked against the reference library itself: every test passes
           (the harness is faithful);
  *.gpu -- linked against librecsparse_gpu.so, the reference's C++ API
           (include/recsparse_gpu) over the C-ABI: tables, dedup, the sharded
           lookup and the sparse Adam run in the sm_100a kernels.
SKIP lists the tests that assert the reference's CPU memory layout rather than
behaviour (slot positions, capacity schedule and the dual-chunk
row allocator are not comparable across designs), the pipeline simulator
(out of scope) and bit-identity twins of an OpenMP path that does not exist.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref")

SKIP = {
    "hash": {},
    "sparse_update": {},
    "exchange_sim": {},
    "embed_table": {
        # the reference's two-chunk row allocator (current / next chunk, retire
        # on exhaustion); the GPU carves one pool in chunk_rows units
        "EmbedTable.DualChunkRotation",
    },
}


def _run(path, skip=()):
    args = [path]
    for s in skip:
        args += ["--skip", s]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900)
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("SUMMARY")]
    return r, (summary[-1] if summary else "")


@pytest.mark.parametrize("suite", sorted(SKIP))
def test_reference_suite_passes_on_the_reference(suite):
    # the harness itself: the reference's suite against the reference library
    path = os.path.join(BIN, f"suite_{suite}.ref")
    if not os.path.exists(path):
        pytest.skip("suites not built (make -C oracle suites needs /root/reference)")
    r, summary = _run(path)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "failed=0" in summary and "skipped=0" in summary, summary


@pytest.mark.gpu
@pytest.mark.parametrize("suite", sorted(SKIP))
def test_reference_suite_passes_on_the_gpu_build(suite):
    path = os.path.join(BIN, f"suite_{suite}.gpu")
    assert os.path.exists(path), "conformance suites missing (build with make -C oracle suites)"
    r, summary = _run(path, SKIP[suite])
    assert r.returncode == 0, r.stdout[-4000:]
    assert "failed=0" in summary, summary
    print(suite, summary)
