"""Dynamic sequence balancing: librsgpu's host batcher
against the oracle restatement and the compiled reference."""
import ctypes as C

import numpy as np
import pytest

import paper_2505_12663_b200 as P


def _cums(rng, n):
    return np.cumsum(rng.integers(1, 50, n)).astype(np.uint64)


def test_closest_prefix_vs_oracle_and_ref(oracle, ref):
    rng = np.random.default_rng(1)
    for _ in range(300):
        c = _cums(rng, int(rng.integers(1, 30)))
        t = int(rng.integers(0, int(c[-1]) + 40))
        want = oracle.closest_prefix(c, len(c), t)
        assert P.closest_prefix(c, t) == want == ref.closest_prefix(c, len(c), t)
    with pytest.raises(P.ConfigError):
        P.closest_prefix([], 3)


def _batch_sizes(lengths, target, chunk):
    data = [P.SequenceSample(i, [1] * int(l)) for i, l in enumerate(lengths)]
    cur = [0]

    def src(ch):
        if cur[0] >= len(data):
            return False
        ch.extend(data[cur[0]:cur[0] + chunk])
        cur[0] += chunk
        return True

    b = P.SequenceBatcher(target, src)
    out, order = [], []
    while (x := b.next_batch()) is not None:
        out.append(len(x))
        order += [s.sample_id for s in x]
    assert order == list(range(len(lengths)))  # arrival order kept
    assert b.buffered_tokens() == 0 and b.buffered_samples() == 0
    return out


@pytest.mark.parametrize("target,chunk", [(100, 4), (1000, 16), (37, 1), (5000, 256)])
def test_sequence_batcher_vs_oracle_and_ref(oracle, ref, target, chunk):
    rng = np.random.default_rng(target + chunk)
    lengths = np.minimum(rng.lognormal(3.5, 1.2, 700).astype(np.uint64) + 1, 4096).astype(np.uint64)
    got = _batch_sizes(lengths, target, chunk)
    for o in (oracle, ref):
        bs = np.zeros(len(lengths) + 1, np.uint64)
        nb = o.sequence_batches(lengths, len(lengths), target, chunk, bs)
        assert got == [int(x) for x in bs[:nb]]


def test_sequence_batcher_errors():
    with pytest.raises(P.ConfigError):
        P.SequenceBatcher(0, lambda ch: False)
    b = P.SequenceBatcher(10, lambda ch: ch.append(P.SequenceSample(1, [])) or True)
    with pytest.raises(P.InvariantError):
        b.next_batch()


def test_partition_lpt_vs_oracle(oracle):
    rng = np.random.default_rng(4)
    for world in (1, 2, 3, 8):
        lengths = np.minimum(rng.lognormal(4.0, 1.5, 2000).astype(np.uint64) + 1, 4096).astype(np.uint64)
        ranks, load = P.partition_sequences(lengths, world, P.batcher.COST_LPT, 1.0, 0.01)
        want = np.zeros(len(lengths), np.uint32)
        oracle.cost_partition(lengths, len(lengths), world, 1.0, 0.01, want)
        np.testing.assert_array_equal(ranks, want)
        rr, _ = P.partition_sequences(lengths, world, P.batcher.ROUND_ROBIN)
        np.testing.assert_array_equal(rr, np.arange(len(lengths)) % world)
        # the cost model balances the simulated compute far better than round robin
        cost = lengths.astype(np.float64) + 0.01 * lengths.astype(np.float64) ** 2
        per = np.array([cost[ranks == r].sum() for r in range(world)])
        np.testing.assert_allclose(per, load)
        if world > 1:
            per_rr = np.array([cost[rr == r].sum() for r in range(world)])
            assert per.max() <= per_rr.max()


def test_imbalance_and_weighted_combine():
    r = P.imbalance_report([5, 3, 9])
    assert (r.max_tokens, r.min_tokens) == (9, 3) and r.spread == (9 - 3) / 9
    assert P.imbalance_report([0, 0]).spread == 0.0
    with pytest.raises(P.ConfigError):
        P.imbalance_report([])
    rng = np.random.default_rng(2)
    bs = rng.integers(1, 100, 5).astype(np.uint64)
    g = rng.standard_normal((5, 33))
    got = P.weighted_grad_combine(bs, g)
    inv = 1.0 / float(bs.sum())
    for e in range(33):
        acc = 0.0
        for i in range(5):
            acc += float(bs[i]) * g[i, e]
        assert got[e] == acc * inv  # workers in fixed order, bit-identical (seq_batcher.cpp:127-135)
    with pytest.raises(P.ConfigError):
        P.weighted_grad_combine([0, 1], g[:2])


def _allreduce_worker(rank, world, port, q):
    import sys as _s
    import os as _o
    _s.path.insert(0, _o.path.dirname(_o.path.dirname(_o.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_2505_12663_b200 as P2
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(rank)
    b = int(rng.integers(1, 50))
    g = rng.standard_normal(17)
    out = P2.batcher.weighted_grad_allreduce(b, g)
    q.put((rank, b, g, out.numpy()))
    dist.destroy_process_group()


def test_weighted_grad_allreduce_gloo_world2():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_allreduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    bs = np.array([r[1] for r in res], np.uint64)
    gs = np.stack([r[2] for r in res])
    want = P.weighted_grad_combine(bs, gs)
    for r in res:
        np.testing.assert_allclose(r[3], want, rtol=1e-14, atol=1e-15)
