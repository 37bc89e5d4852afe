"""Sharded step: host bootstrap on CPU (gloo, world 2) and the
NVLink peer-store step on >= 2 GPUs against the oracle (tests/dist_worker.py)."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _handles_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    from paper_2505_12663_b200.dist import exchange_handles
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    got = exchange_handles(bytes([rank]) * 64)
    q.put((rank, got))
    dist.destroy_process_group()


def test_handle_exchange_gloo_world2():
    # the IPC-handle bootstrap returns every rank's 64-byte handle in rank order
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_handles_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r] == [bytes([0]) * 64, bytes([1]) * 64]


def test_shard_of_matches_oracle(oracle):
    # owner routing: shard_of = hash64(id) % W (exchange_sim.cpp:82-85)
    import numpy as np
    ids = np.random.default_rng(3).integers(0, 1 << 63, 1000).astype(np.uint64)
    for W in (1, 2, 3, 8):
        want = [oracle.shard_of(int(i), W) for i in ids]
        got = [int(oracle.hash64(int(i))) % W for i in ids]
        assert want == got


@pytest.mark.gpu
@pytest.mark.parametrize("opt,dim", [("adam", 32), ("adagrad", 64), ("adam", 128)])
def test_sharded_step_vs_oracle(opt, dim):
    # one process per GPU over CUDA IPC + NVLink; on a 1-GPU box the same worker
    # runs at W = 1 (the bootstrap and the arena mapped as its own peer).  The
    # W-rank data path on one GPU is tests/test_dist_local.py.
    n = torch.cuda.device_count()
    w = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={w}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), opt, str(dim)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    errs = [ln for ln in (r.stdout + r.stderr).splitlines()
            if ("rror" in ln or "assert" in ln.lower() or "Mismatch" in ln) and "frame #" not in ln]
    assert r.returncode == 0, "\n".join(errs[:40]) + "\n" + r.stdout[-3000:]
    assert f"DIST OK world={w}" in r.stdout
