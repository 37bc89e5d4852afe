#!/usr/bin/env python
"""Benchmark of the sparse-embedding hot path (BASELINE.json metric).

Metric: unique-ID lookups+updates per second (one step = dedup -> table
find-or-insert -> jagged gather -> segment-reduce + Adagrad update of one
batch), whole job over all ranks.  Default workload = BASELINE config 1:
one dynamic table, dim 64, 2^20 keys pre-populated, batch 1024 jagged
sequences (lognormal, mean 128, max 4096), Zipf(1.1) ids, Adagrad.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation
(oracle/_ref/librsref.so, compiled from /root/reference sources; else the C
restatement) on the host cores, same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C1 = dict(workload="config1: 1 dynamic table dim 64, 2^20 keys, batch 1024 seqs (mean 128, max 4096, sigma 1.0), "
                   "Zipf 1.1, dedup+lookup+Adagrad", dim=64, vocab=1 << 20, seqs=1024, mean=128.0, max_len=4096,
          sigma=1.0, zipf=1.1, seed=1, capacity=1 << 22)
C4 = dict(workload="config4: row-sharded table of 100M pre-populated keys, dim 128, Zipf 1.1 over 1e8, per-rank batch "
                   "1024 seqs (mean 128, max 4096, sigma 1.0), dedup+lookup+Adagrad, ids/embeddings/gradients over NVLink",
          dim=128, vocab=100_000_000, seqs=1024, mean=128.0, max_len=4096, sigma=1.0, zipf=1.1, seed=4,
          capacity=None)
C5 = dict(workload="config5: long-tail sequences (lognormal sigma 1.5, mean 128, max 4096), a pool of 1024 x N "
                   "sequences per step assigned to the N ranks by the cost model (LPT on a*len + b*len^2, "
                   "CostModel defaults a=1, b=0.01), sharded 2^20-key table dim 64, dedup+lookup+Adagrad",
          dim=64, vocab=1 << 20, seqs=1024, mean=128.0, max_len=4096, sigma=1.5, zipf=1.1, seed=5,
          capacity=1 << 22, pooled=True)
TAG1 = np.uint64(1 << 62)
L2_FLUSH_BYTES = 512 << 20
_E2E_HOST_MS = None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    def __init__(self, index=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {getattr(N, k, 0): k for k in (
            "nvmlClocksEventReasonGpuIdle", "nvmlClocksEventReasonSwPowerCap", "nvmlClocksEventReasonHwSlowdown",
            "nvmlClocksEventReasonHwThermalSlowdown", "nvmlClocksEventReasonSwThermalSlowdown",
            "nvmlClocksEventReasonHwPowerBrakeSlowdown", "nvmlClocksEventReasonApplicationsClocksSetting",
            "nvmlClocksEventReasonSyncBoost")}
        short = {"nvmlClocksEventReasonSwPowerCap": "sw_power_cap", "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
                 "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
                 "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
                 "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake",
                 "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks",
                 "nvmlClocksEventReasonSyncBoost": "sync_boost", "nvmlClocksEventReasonGpuIdle": "gpu_idle"}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if bit and r & bit and name in short:
                        self.reasons.add(short[name])
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.N:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"})}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def n_batches(warmup):
    """Distinct batches both arms cycle through (step k uses batch k % nb): even,
    so each batch always meets the same scratch parity (one captured graph
    each), at most 6, and every one of them runs during the W warm-up steps --
    no graph is ever captured inside the timed region."""
    return max(2, min(6, warmup - warmup % 2))


def batch_seed(cfg, rank, b):
    return cfg["seed"] + 1000 * rank + b


def bench_config(cfg, world, nb, sharded):
    """The `config` object, identical in both arms (--impl ours / reference)."""
    c = {"workload": cfg["workload"] + ("; row-sharded over the ranks (owner = hash64 % N), per-rank batch"
                                        if sharded else ""),
         "embedding_dim": cfg["dim"], "table_keys": cfg["vocab"], "optimizer": "adagrad (lr 0.01, eps 1e-8)",
         "batches": nb, "batch_seeds": f"{cfg['seed']} + 1000*rank + b, b < {nb}",
         "parallelism": f"row-sharded x{world}" if sharded else "single"}
    return c


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2505_12663_b200 as P
    from paper_2505_12663_b200 import workload as W

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dim, vocab = cfg["dim"], cfg["vocab"]

    # table: every key pre-populated with pseudo_sparse_grad(k, 0) rows (bench_main.cpp:105-108)
    cap = cfg["capacity"] or 1 << int(np.ceil(np.log2((vocab + (1 << 20)) / 0.6)))
    table = P.EmbedTable(P.TableConfig(capacity=cap, embedding_dim=dim, optimizer="adagrad",
                                       chunk_rows=1 << 16, initial_rows=vocab + (1 << 20)))
    for lo in range(0, vocab, 1 << 24):
        raw = torch.arange(lo, min(vocab, lo + (1 << 24)), dtype=torch.int64, device="cuda")
        table.insert(raw + int(TAG1), W.pseudo_grads(raw, 0, dim))
    del raw
    # distinct batches (weak scaling: each rank its own seed stream)
    nb = n_batches(args.warmup)
    batches = []
    for b in range(nb):
        lengths, ids = W.generate(batch_seed(cfg, rank, b), cfg["seqs"], cfg["mean"], cfg["max_len"],
                                  cfg["sigma"], cfg["zipf"], [vocab])
        batches.append((lengths, ids))
    max_t = max(len(i) for _, i in batches)
    step = P.SparseStep(table, max_t, P.AdagradParams(lr=0.01, eps=1e-8))
    dev = []
    for b, (lengths, ids) in enumerate(batches):
        d_ids = P.as_keys(ids)
        d_g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), b, dim)
        dev.append((d_ids, d_g, torch.empty((len(ids), dim), device="cuda")))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    lib = P.lib()

    def one(b):
        d_ids, d_g, out = dev[b % nb]
        step.step(d_ids, d_g, out)

    # warm-up: W steps, every batch at least once (one CUDA graph per batch
    # buffer set is captured on first use -- never inside the timed region)
    for w in range(args.warmup):
        one(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- device-timed steps (inputs resident in HBM, L2 flushed between
    # steps).  All K steps are enqueued back to back; each step is bracketed
    # by its own CUDA events, the flush in between is outside the brackets.
    uniq_per_batch = [int(np.unique(ids).size) for _, ids in batches]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.rs_kernel_launches()
    syncs0 = table.info().host_syncs
    with Clocks(local) as clk:
        h0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            one(args.warmup + k)
            evs[k][1].record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # host enqueue time per step
        torch.cuda.synchronize()
    launches = lib.rs_kernel_launches() - launches0
    syncs = table.info().host_syncs - syncs0
    # host time to issue the step alone (no flush launch, no event records): the
    # timed loop's host time also covers the 512 MiB flush kernel and 2 events
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    for k in range(args.steps):
        one(args.warmup + k)
    host_step_ms = (time.perf_counter() - h1) * 1e3 / args.steps
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in evs]
    uniq = sum(uniq_per_batch[(args.warmup + k) % nb] for k in range(args.steps))
    toks = sum(dev[(args.warmup + k) % nb][0].numel() for k in range(args.steps))
    assert _n_unique(step) == uniq_per_batch[(args.warmup + args.steps - 1) % nb], "device n_unique mismatch"
    t_sum = sum(times) / 1e3
    if world > 1:
        tt = torch.tensor([t_sum], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        uu = torch.tensor([uniq, toks], dtype=torch.float64, device="cuda")
        dist.all_reduce(uu)
        t_job, uniq_job, toks_job = tt.item(), uu[0].item(), uu[1].item()
    else:
        t_job, uniq_job, toks_job = t_sum, uniq, toks
    value = uniq_job / t_job

    # ---- per-kernel shares (separate pass with phase events, same inputs)
    phases = phase_times(step, dev, nb, args, flush, P)
    # ---- in-graph kernel spans (device %globaltimer per block, a separate
    # workspace with the timeline on)
    in_graph = graph_timeline(table, dev, nb, flush, P, max_t)

    # ---- end to end through the public API with HOST buffers
    e2e = e2e_pass(args, cfg, batches, step, P, W, rank)

    # ---- roofline of the dominant kernel: algorithmic bytes per launch / its
    # CUDA-event duration (bytes per unit: SURVEY.md §8d)
    hbm, how = peaks()
    D = dim
    T_avg, U_avg = toks / args.steps, uniq / args.steps
    # tokens / ids of the CSR path (<= 64 occurrences) and of the hot path
    T_hot = U_hot = 0.0
    for k in range(args.steps):
        _, cnt = np.unique(batches[(args.warmup + k) % nb][1], return_counts=True)
        T_hot += float(cnt[cnt > 64].sum()) / args.steps
        U_hot += float((cnt > 64).sum()) / args.steps
    T_csr, U_csr = T_avg - T_hot, U_avg - U_hot
    # SURVEY §8(d) per-phase compulsory bytes: ids 8T + dedup out 8U + 4T +
    # slot probe 16U; per id: gather read 4D + Adagrad state r/w 16D; per
    # token: forward write 4D + gradient read 4D
    algo = {
        "dedup_probe": 12 * T_avg + 24 * U_avg,
        "csr_update": 8 * D * T_csr + 20 * D * U_csr,
        "hot_update": 8 * D * T_hot + 20 * D * U_hot,
        "checksum": 0.0,
    }
    dom = max(algo, key=lambda k: phases.get(k) or 0.0)
    traffic = traffic_ctx = None
    try:  # dram bytes of the same kernel from the committed ncu --set full capture
        import glob
        tf = sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")))[-1]
        with open(tf) as f:
            tj = json.load(f)
        traffic = tj.get(dom)
        traffic_ctx = tj.get("in_context", {}).get(dom)  # --cache-control none: the step's real L2 state
    except Exception:
        traffic = traffic_ctx = None
    ach = algo[dom] / (phases[dom] / 1e3) / 1e9 if phases.get(dom) else None
    step_bytes = 12 * T_avg + 24 * U_avg + 8 * D * T_avg + 20 * D * U_avg
    res = {
        "metric": "unique-ID lookups+updates/sec",
        "value": value,
        "unit": "unique-ids/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_job / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 rows, f64 optimizer math, u64 ids",
        "data": "synthetic: the reference's generator (mt19937_64, truncated lognormal lengths, Zipf 1.1 ids), "
                "pseudo_sparse_grad gradients",
        "config": bench_config(cfg, world, nb, False),
        "shape": {"tokens_per_step_per_rank": T_avg, "unique_per_step_per_rank": U_avg},
        "l2": "flushed (512 MiB write) between timed steps",
        "table_host_syncs_in_timed_region": int(syncs),
        "tokens_per_s": toks_job / t_job,
        "host_enqueue_ms_per_step": host_ms,
        "host_issue_ms_per_step": host_step_ms,
        "host_note": "host_enqueue = host time per timed iteration (flush launch + 2 event records + the step); "
                     "host_issue = the step's own host time (graph launch, capacity bookkeeping, no sync); "
                     "the device timing brackets only the step",
        "step_hbm_gbs": step_bytes * world / (t_job / args.steps) / 1e9,
        "step_roofline_frac": step_bytes / (t_job / args.steps) / 1e9 / hbm,
        "kernel_ms": phases,
        "kernel_ms_note": "eager, one kernel group after another (no graph, no concurrency), L2 flushed",
        "kernel_gbs": {k: (algo[k] / (phases[k] / 1e3) / 1e9 if phases.get(k) else None) for k in algo},
        "kernel_span_in_graph_us": in_graph,
        "roofline": {"bound": "hbm", "kernel": dom,
                     "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": (ach / hbm) if ach else None,
                     "traffic": traffic, "traffic_in_context": traffic_ctx, "peak_source": how,
                     "algorithmic_bytes_per_launch": algo[dom]},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg is C1:
        res["cpu_baseline"] = cpu_baseline(cfg, batches, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_sharded(args, cfg):
    """N > 1: the row-sharded step, weak scaling.  Each rank owns
    the keys with hash64(id) % N == rank of the same 2^20-key table, draws its
    own config-1 batch, and runs forward (two-stage dedup, ids and embeddings
    exchanged by NVLink peer stores) + backward (pre-reduced grads to the
    owners, Adagrad on the owner shard).  value = sum over ranks of each rank's
    unique ids / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_2505_12663_b200 as P
    from paper_2505_12663_b200 import workload as W
    from paper_2505_12663_b200.dist import ShardedTable

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dim, vocab = cfg["dim"], cfg["vocab"]
    nb = n_batches(args.warmup)
    balance = None
    if cfg.get("pooled"):
        # config 5: one pool of sequences per step, every rank computes the same
        # assignment (rs_partition_sequences) and takes its share
        policy = P.batcher.COST_LPT if args.balance == "lpt" else P.batcher.ROUND_ROBIN
        batches, spreads, cost_spreads = [], [], []
        for b in range(nb):
            lengths, ids = W.generate(cfg["seed"] + b, cfg["seqs"] * world, cfg["mean"], cfg["max_len"],
                                      cfg["sigma"], cfg["zipf"], [vocab])
            ranks, load = P.partition_sequences(lengths, world, policy, 1.0, 0.01)
            starts = np.concatenate([[0], np.cumsum(lengths.astype(np.int64))])
            mine = np.nonzero(ranks == rank)[0]
            ids_r = np.concatenate([ids[starts[i]:starts[i + 1]] for i in mine]) if len(mine) else ids[:0]
            batches.append((lengths[mine], ids_r))
            tok = np.array([lengths[ranks == r].sum() for r in range(world)], np.uint64)
            spreads.append(P.imbalance_report(tok).spread)
            cost_spreads.append(float((load.max() - load.min()) / load.max()) if load.max() > 0 else 0.0)
        balance = {"policy": args.balance, "token_spread_mean": float(np.mean(spreads)),
                   "cost_spread_mean": float(np.mean(cost_spreads))}
    else:
        batches = [W.generate(batch_seed(cfg, rank, b), cfg["seqs"], cfg["mean"], cfg["max_len"], cfg["sigma"],
                              cfg["zipf"], [vocab]) for b in range(nb)]
    mt = torch.tensor([max(len(i) for _, i in batches)], dtype=torch.int64, device="cuda")
    dist.all_reduce(mt, op=dist.ReduceOp.MAX)  # the arena layout must agree on every rank
    max_t = int(mt.item())
    nflat = world * max_t
    # shard sized for its keys + the W * max_tokens new-key headroom of a step
    rows = vocab // world + vocab // (8 * world) + 8 * nflat
    cap = cfg["capacity"] * 2 if cfg.get("capacity") else 1 << int(np.ceil(np.log2(rows / 0.6)))
    st = ShardedTable(P.TableConfig(capacity=cap, embedding_dim=dim, optimizer="adagrad",
                                    chunk_rows=1 << 16, initial_rows=rows), max_tokens=max_t)
    for lo in range(0, vocab, 1 << 24):  # every rank inserts the keys it owns
        raw = torch.arange(lo, min(vocab, lo + (1 << 24)), dtype=torch.int64, device="cuda")
        st.insert_owned(raw + int(TAG1), W.pseudo_grads(raw, 0, dim))
    del raw
    torch.cuda.synchronize()
    params = P.AdagradParams(lr=0.01, eps=1e-8)
    dev = []
    for b, (lengths, ids) in enumerate(batches):
        d_g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), b, dim)
        dev.append((P.as_keys(ids), d_g, torch.empty((len(ids), dim), device="cuda")))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    lib = P.lib()

    def one(b):
        d_ids, d_g, out = dev[b % nb]
        st.step(d_ids, d_g, params, out)

    for w in range(args.warmup):  # every batch's graph captured before timing (W >= nb)
        one(w)
    torch.cuda.synchronize()
    dist.barrier()
    uniq_b = [int(np.unique(ids).size) for _, ids in batches]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.rs_kernel_launches()
    host_call = 0.0
    with Clocks(local) as clk:
        h0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            st.barrier()  # device barrier: no rank's flush leaks into another rank's step bracket
            evs[k][0].record(stream)
            h1 = time.perf_counter()
            one(args.warmup + k)
            host_call += time.perf_counter() - h1
            evs[k][1].record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # host enqueue time per step
        torch.cuda.synchronize()
    launches = lib.rs_kernel_launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    per_rank = [None] * world
    dist.all_gather_object(per_rank, {"sum_ms": sum(step_ms), "median_ms": statistics.median(step_ms),
                                      "host_enqueue_ms_per_step": host_ms,
                                      "host_step_call_ms": host_call * 1e3 / args.steps})
    t_sum = sum(step_ms) / 1e3
    uniq = sum(uniq_b[(args.warmup + k) % nb] for k in range(args.steps))
    toks = sum(dev[(args.warmup + k) % nb][0].numel() for k in range(args.steps))
    tr = st.trace()  # last step's ExchangeTrace (all ranks)
    timeline = dist_timeline(st, one, flush, lib, P) if os.environ.get("RS_TRACE") == "1" else None
    # per-phase device time (separate pass, CUDA events between the phases)
    st.set_profiling(True)
    for k in range(max(3, min(args.steps, 10))):
        flush.zero_()
        one(k)
    phases = st.phase_ms()
    st.set_profiling(False)
    tt = torch.tensor([t_sum], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    uu = torch.tensor([uniq, toks], dtype=torch.float64, device="cuda")
    dist.all_reduce(uu)
    t_job, uniq_job, toks_job = tt.item(), uu[0].item(), uu[1].item()
    ms = t_job / args.steps * 1e3

    # NVLink bytes of the last step: ids (8 B) + grads (4D) to every other
    # owner, embeddings (4D) back from every owner; max over ranks
    ids_sent, embs_sent = tr["ids_sent"].astype(np.float64), tr["embs_sent"].astype(np.float64)
    off = 1.0 - np.eye(world)
    out_bytes = (ids_sent * off).sum(1) * (8 + 4 * dim) + (embs_sent * off).sum(1) * 4 * dim
    nvl_max = float(out_bytes.max())

    # end to end: host ids + grads -> device, the step, gathered rows -> host
    e2e = e2e_sharded(args, cfg, batches, st, params, P, W)
    hbm, how = peaks()
    T_avg, U_avg = toks / args.steps, uniq / args.steps
    D = dim
    step_bytes = 12 * T_avg + 24 * U_avg + 8 * D * T_avg + 20 * D * U_avg
    ach = step_bytes / (ms / 1e3) / 1e9
    res = {
        "metric": "unique-ID lookups+updates/sec",
        "value": uniq_job / t_job,
        "unit": "unique-ids/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 rows, f64 optimizer math, u64 ids",
        "data": "synthetic: the reference's generator (mt19937_64, truncated lognormal lengths, Zipf 1.1 ids), "
                "pseudo_sparse_grad gradients",
        "config": bench_config(cfg, world, nb, True),
        "shape": {"tokens_per_step_per_rank": T_avg, "unique_per_step_per_rank": U_avg},
        "exchange": "NVLink peer stores from the producing kernels (CUDA IPC arena)",
        "l2": "flushed (512 MiB write) between timed steps, then a device barrier of all ranks",
        "tokens_per_s": toks_job / t_job,
        "kernel_ms_rank0": phases,
        **({"timeline_us_rank0": timeline} if timeline else {}),
        "step_ms_rank0": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        "per_rank": per_rank,
        "balance": balance,
        "table_host_syncs_rank0": int(st.shard.info().host_syncs),
        "roofline": {"bound": "hbm", "kernel": "sharded step (all kernels of one rank)", "achieved": ach,
                     "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None, "peak_source": how,
                     "algorithmic_bytes_per_launch": step_bytes},
        "nvlink": {"bytes_per_step_max_rank": nvl_max, "achieved_gbs": nvl_max / (ms / 1e3) / 1e9,
                   "peak_gbs_per_direction": 900.0,
                   "trace_last_step": {"ids_sent": tr["ids_sent"].tolist(), "embs_sent": tr["embs_sent"].tolist(),
                                       "lookups": tr["lookups"].tolist()}},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.barrier()
    st.close()
    dist.destroy_process_group()


def e2e_sharded(args, cfg, batches, st, params, P, W):
    import torch
    import torch.distributed as dist
    n = max(200, args.steps)  # ~0.15 ms per step: enough steps (~30 ms) to average the host-fed pipeline
    uniq_b = [int(np.unique(ids).size) for _, ids in batches]
    t, uniq, h2d, d2h = workload_e2e(batches, cfg["dim"], lambda f, hi, hl, k: f.dist_step(st, params, hi, hl, k),
                                     n, uniq_b, barrier=dist.barrier)
    v = torch.tensor([t, uniq], dtype=torch.float64, device="cuda")
    tmax = v[:1].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(v)
    return {"value": v[1].item() / tmax.item(), "unit": "unique-ids/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": tmax.item() / n * 1e3,
            "io": "H2D token ids + sequence lengths; gradients generated in-step on the device "
                  "(pseudo_sparse_grad per sample, as run_workload does); D2H the step's embedding checksum"}


C2 = dict(workload="config2: 8 tables (dim 64: 1e7/1e6/1e6/1e5 keys; dim 128: 1e6/1e6/1e5/1e4 keys) auto-merged "
                   "into 2 physical tables, batch 4096 seqs (mean 256, max 4096, sigma 1.0), Zipf 1.1, per-token "
                   "catalog decode + group re-encode on the device, dedup+lookup+Adagrad per group",
          tables=[("t0", 64, 10_000_000), ("t1", 64, 1_000_000), ("t2", 64, 1_000_000), ("t3", 64, 100_000),
                  ("t4", 128, 1_000_000), ("t5", 128, 1_000_000), ("t6", 128, 100_000), ("t7", 128, 10_000)],
          seqs=4096, mean=256.0, max_len=4096, sigma=1.0, zipf=1.1, seed=2)


def run_c2(args, cfg):
    """Config 2 on one GPU: catalog-tagged tokens routed into the two merged
    groups (rs_route_tagged: decode + re-encode + stable partition), then one
    fused step per group table.  value = unique ids of both groups / time."""
    import torch

    import paper_2505_12663_b200 as P
    from paper_2505_12663_b200 import workload as W

    torch.cuda.set_device(0)
    feats = [P.FeatureConfig(n + "_f", d, [n]) for n, d, _ in cfg["tables"]]
    plan = P.plan_merge(feats)
    names, _, cat_k = P.catalog_from(feats)
    router = P.Router(plan, names)
    vocab = [v for _, _, v in cfg["tables"]]
    tables, steps = [], []
    for g in plan.groups:
        members = g.member_tables
        nkeys = sum(v for n, _, v in cfg["tables"] if n in members)
        cap = 1 << int(np.ceil(np.log2(nkeys / 0.5)))
        t = P.EmbedTable(P.TableConfig(capacity=cap, embedding_dim=g.embedding_dim, optimizer="adagrad",
                                       chunk_rows=1 << 16, initial_rows=nkeys + (1 << 21)))
        for name in members:  # pre-populate every key of every member table
            v = next(v for n, _, v in cfg["tables"] if n == name)
            for lo in range(0, v, 1 << 22):
                raw = torch.arange(lo, min(v, lo + (1 << 22)), dtype=torch.int64, device="cuda")
                t.insert(raw | (g.table_index_of[name] << (63 - g.k_bits)), W.pseudo_grads(raw, 0, g.embedding_dim))
        tables.append(t)
    nb = 4
    batches = []
    for b in range(nb):
        lengths, tagged = W.generate(cfg["seed"] + b, cfg["seqs"], cfg["mean"], cfg["max_len"], cfg["sigma"],
                                     cfg["zipf"], vocab)
        d_tag = P.as_keys(tagged)
        gids, pos, counts = router.route(d_tag)  # counts: a property of the batch (data-prep time)
        sample_of = torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)).cuda()
        per = []
        off = 0
        for g, cnt in zip(plan.groups, counts):
            sel = pos[off:off + cnt].long()
            grads = W.pseudo_grads(sample_of[sel], b, g.embedding_dim)
            per.append((off, cnt, grads, torch.empty((cnt, g.embedding_dim), device="cuda"),
                        int(np.unique(P.keys_to_numpy(gids[off:off + cnt])).size)))
            off += cnt
        batches.append((d_tag, gids, pos, per))
    for g, t in enumerate(tables):
        steps.append(P.SparseStep(t, max(b[3][g][1] for b in batches), P.AdagradParams(lr=0.01, eps=1e-8)))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    lib = P.lib()

    def one(k):
        d_tag, gids, pos, per = batches[k % nb]
        router.route_async(d_tag, gids, pos)
        for g, (off, cnt, grads, out, _) in enumerate(per):
            steps[g].step(gids[off:off + cnt], grads, out)

    args.warmup = max(args.warmup, 2 * nb)
    for w in range(args.warmup):
        one(w)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.rs_kernel_launches()
    with Clocks(0) as clk:
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            one(args.warmup + k)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    launches = lib.rs_kernel_launches() - launches0
    ms = [a.elapsed_time(b) for a, b in evs]
    t = sum(ms) / 1e3
    uniq = sum(sum(p[4] for p in batches[(args.warmup + k) % nb][3]) for k in range(args.steps))
    toks = sum(batches[(args.warmup + k) % nb][0].numel() for k in range(args.steps))
    hbm, how = peaks()
    T, U = toks / args.steps, uniq / args.steps
    byt = 0.0
    for g, grp in enumerate(plan.groups):
        Tg = sum(batches[(args.warmup + k) % nb][3][g][1] for k in range(args.steps)) / args.steps
        Ug = sum(batches[(args.warmup + k) % nb][3][g][4] for k in range(args.steps)) / args.steps
        D = grp.embedding_dim
        byt += 12 * Tg + 24 * Ug + 8 * D * Tg + 20 * D * Ug
    byt += 8 * T * 2 + 4 * T  # routing: tagged ids in, group ids + positions out
    ach = byt / (t / args.steps) / 1e9
    res = {"metric": "unique-ID lookups+updates/sec", "value": uniq / t, "unit": "unique-ids/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f32 rows, f64 optimizer math, u64 ids",
           "data": "synthetic: the reference's generator over 8 tagged tables, pseudo_sparse_grad gradients",
           "config": {"workload": cfg["workload"], "tokens_per_step": T, "unique_per_step": U,
                      "groups": [(g.embedding_dim, g.member_tables) for g in plan.groups],
                      "l2": "flushed (512 MiB write) between timed steps"},
           "tokens_per_s": toks / t,
           "roofline": {"bound": "hbm", "kernel": "whole step (route + 2 group steps)", "achieved": ach,
                        "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None, "peak_source": how,
                        "algorithmic_bytes_per_launch": byt},
           "gpu_launches": int(launches), "clocks": clk.summary()}
    print(json.dumps(res), flush=True)


C3 = dict(workload="config3: insert/evict-heavy stream: bounded table (max_keys 2^22, starts full), dim 128, "
                   "batch 1024 seqs (mean 128, max 4096, sigma 1.0), Zipf 1.1 over the resident ids with 20% of "
                   "each batch's unique ids replaced by never-seen ids; every batch inserts and evicts the oldest "
                   "(tick, key)", dim=128, bound=1 << 22, seqs=1024, mean=128.0, max_len=4096, sigma=1.0, zipf=1.1,
          seed=3, new_frac=0.2)


def run_c3(args, cfg):
    """Config 3 on one GPU: the fused step on a bounded table (probe, evict the
    oldest (tick, key) beyond the bound, insert the misses, gather, reduce,
    update).  value = unique ids / time."""
    import torch

    import paper_2505_12663_b200 as P
    from paper_2505_12663_b200 import workload as W

    torch.cuda.set_device(0)
    dim, bound = cfg["dim"], cfg["bound"]
    table = P.EmbedTable(P.TableConfig(capacity=1 << int(np.ceil(np.log2(bound / 0.6))), embedding_dim=dim,
                                       optimizer="adagrad", chunk_rows=1 << 16, initial_rows=bound + (1 << 20),
                                       max_keys=bound))
    for lo in range(0, bound, 1 << 22):  # starts full at the bound
        raw = torch.arange(lo, min(bound, lo + (1 << 22)), dtype=torch.int64, device="cuda")
        table.ensure(raw + int(TAG1))
    rng = np.random.default_rng(cfg["seed"])
    fresh = np.uint64((1 << 62) + bound)
    nb = 6
    batches = []
    for b in range(nb + args.steps + max(args.warmup, 3)):  # new ids never repeat across steps
        lengths, ids = W.generate(cfg["seed"] + b, cfg["seqs"], cfg["mean"], cfg["max_len"], cfg["sigma"],
                                  cfg["zipf"], [bound])
        u, inv = np.unique(ids, return_inverse=True)
        pick = rng.random(len(u)) < cfg["new_frac"]
        u = u.copy()
        u[pick] = fresh + np.arange(int(pick.sum()), dtype=np.uint64)
        fresh += np.uint64(int(pick.sum()))
        batches.append((lengths, u[inv], len(u), int(pick.sum())))
    max_t = max(len(x[1]) for x in batches)
    step = P.SparseStep(table, max_t, P.AdagradParams(lr=0.01, eps=1e-8))
    out = torch.empty((max_t, dim), device="cuda")
    dev = []
    for b, (lengths, ids, nu, nnew) in enumerate(batches):
        dev.append((P.as_keys(ids), W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)),
                                                   b, dim), nu, nnew))
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    lib = P.lib()
    k0 = max(args.warmup, 3)
    for k in range(k0):
        d_ids, d_g, _, _ = dev[k]
        step.step(d_ids, d_g, out[:d_ids.numel()])
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.rs_kernel_launches()
    syncs0 = table.info().host_syncs
    with Clocks(0) as clk:
        for k in range(args.steps):
            d_ids, d_g, _, _ = dev[k0 + k]
            flush.zero_()
            evs[k][0].record(stream)
            step.step(d_ids, d_g, out[:d_ids.numel()])
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    launches = lib.rs_kernel_launches() - launches0
    ms = [a.elapsed_time(b) for a, b in evs]
    t = sum(ms) / 1e3
    uniq = sum(dev[k0 + k][2] for k in range(args.steps))
    new = sum(dev[k0 + k][3] for k in range(args.steps))
    syncs = table.info().host_syncs - syncs0
    toks = sum(dev[k0 + k][0].numel() for k in range(args.steps))
    assert table.occupied() == bound
    hbm, how = peaks()
    T, U, Nn = toks / args.steps, uniq / args.steps, new / args.steps
    byt = 12 * T + 24 * U + 8 * dim * T + 20 * dim * U + Nn * (16 + 16 + 16 + 8 * dim)  # + evict/insert slots, row init
    ach = byt / (t / args.steps) / 1e9
    res = {"metric": "unique-ID lookups+updates/sec", "value": uniq / t, "unit": "unique-ids/s", "n_gpus": 1,
           "steps": args.steps, "warmup": k0, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32 rows, f64 optimizer math, u64 ids",
           "data": "synthetic: the reference's generator + a monotone counter of never-seen ids",
           "config": {"workload": cfg["workload"], "tokens_per_step": T, "unique_per_step": U,
                      "new_ids_per_step": Nn, "evictions_per_step": Nn,
                      "l2": "flushed (512 MiB write) between timed steps"},
           "roofline": {"bound": "hbm", "kernel": "whole step", "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm, "traffic": None, "peak_source": how, "algorithmic_bytes_per_launch": byt},
           "victim_selection": "stamp log (evict.cu k_lg_*): the live records from the log head, no slot scan; "
                               "device radix select over (tick, key) slot scan when the log is off (RS_EVICT_LOG=0)",
           "step_ms": {"min": min(ms), "median": float(np.median(ms)), "max": max(ms)},
           "table_host_syncs_in_timed_region": int(syncs),
           "gpu_launches": int(launches), "clocks": clk.summary()}
    print(json.dumps(res), flush=True)


def _n_unique(step):
    import ctypes

    import paper_2505_12663_b200 as P
    n = ctypes.c_uint64()
    P._lib.check(P.lib().rs_workspace_n_unique(step.ws.handle, ctypes.byref(n)), "n_unique")
    return n.value


# the fast step's eager phases (rs_workspace_phase_ms): dedup + probe (KA);
# the CSR ids' forward + ordered reduce + Adagrad (scratch clean, heavy and
# light kernels); the hot ids' tile partials + finish; the checksum (0 here)
PHASES = ["dedup_probe", "csr_update", "hot_update", "checksum"]
TRACE_NAMES = ["dedup_probe", "csr_light", "hot_tiles", "hot_finish", "scratch_clean", "csr_heavy"]


DIST_TRACE_NAMES = TRACE_NAMES + ["req_gather", "req_grad_flags", "own_wait_ids", "own_dedup", "own_table_respond",
                                   "req_wait_rows", "own_wait_grads", "own_update_done", "own_update"]


def dist_timeline(st, one, flush, lib, P):
    """Sharded step device timeline (diagnostics, RS_TRACE=1 for the whole
    run): per kernel slot of this rank the median over 6 graph-replayed steps
    of start / end relative to the requester dedup's first block (us)."""
    import ctypes
    import torch
    n = ctypes.c_uint64()
    buf = np.zeros(16 * 4096 * 2, np.uint64)
    rows = {name: [] for name in DIST_TRACE_NAMES}
    for k in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        st.barrier()
        P._lib.check(lib.rs_comm_timeline(st._c, buf.ctypes.data, buf.size, ctypes.byref(n)), "timeline")
        one(k)
        torch.cuda.synchronize()
        P._lib.check(lib.rs_comm_timeline(st._c, buf.ctypes.data, buf.size, ctypes.byref(n)), "timeline")
        if not n.value:
            return None
        t = buf.reshape(16, 4096, 2).astype(np.float64)
        t0 = t[0, :, 0][t[0, :, 1] > 0].min()
        if os.environ.get("RS_TRACE_DUMP") and k == 5:  # raw per-block spans of the last step (us)
            np.save(f"{os.environ['RS_TRACE_DUMP']}_rank{st.rank}.npy", np.where(t > 0, (t - t0) / 1e3, np.nan))
            np.save(f"{os.environ['RS_TRACE_DUMP']}_rank{st.rank}_t0.npy", np.array([t0]))
        for i, name in enumerate(DIST_TRACE_NAMES):
            ok = t[i, :, 1] > 0
            if ok.any():
                rows[name].append(((t[i, ok, 0].min() - t0) / 1e3, (t[i, ok, 1].max() - t0) / 1e3))
    out = {}
    for name, v in rows.items():
        if v:
            a = np.array(v)
            out[name] = {"start_us": round(float(np.median(a[:, 0])), 2), "end_us": round(float(np.median(a[:, 1])), 2)}
    return out


def graph_timeline(table, dev, nb, flush, P, max_t):
    """Kernel spans inside the step's CUDA graph: a second workspace with the
    device timeline (RS_TRACE=1 at its first step: per block the first warp
    start / last warp end, %globaltimer), L2 flushed before each step; per
    kernel the median over 6 steps of start / end relative to the first
    kernel's first block (us)."""
    import ctypes
    os.environ["RS_TRACE"] = "1"
    try:
        st = P.SparseStep(table, max_t, P.AdagradParams(lr=0.01, eps=1e-8))
        for k in range(2 * nb):
            st.step(*dev[k % nb])
    finally:
        del os.environ["RS_TRACE"]
    lib = P.lib()
    n = ctypes.c_uint64()
    buf = np.zeros(16 * 4096 * 2, np.uint64)
    rows = {name: [] for name in TRACE_NAMES}
    for k in range(6):
        flush.zero_()
        import torch
        torch.cuda.synchronize()
        P._lib.check(lib.rs_workspace_trace(st.ws.handle, buf.ctypes.data, buf.size, ctypes.byref(n)), "trace")
        st.step(*dev[k % nb])
        torch.cuda.synchronize()
        P._lib.check(lib.rs_workspace_trace(st.ws.handle, buf.ctypes.data, buf.size, ctypes.byref(n)), "trace")
        if not n.value:
            return None
        t = buf.reshape(16, 4096, 2).astype(np.float64)
        t0 = t[0, :, 0][t[0, :, 1] > 0].min()
        for i, name in enumerate(TRACE_NAMES):
            ok = t[i, :, 1] > 0
            if ok.any():
                rows[name].append(((t[i, ok, 0].min() - t0) / 1e3, (t[i, ok, 1].max() - t0) / 1e3))
    out = {}
    for name, v in rows.items():
        if v:
            a = np.array(v)
            out[name] = {"start_us": round(float(np.median(a[:, 0])), 2), "end_us": round(float(np.median(a[:, 1])), 2)}
    return out


def phase_times(step, dev, nb, args, flush, P):
    """Mean device time per kernel group of rs_step, from CUDA events recorded
    by librsgpu on the launching stream between the kernels (profiling mode
    runs the same kernels without the graph)."""
    import ctypes
    lib = P.lib()
    P._lib.check(lib.rs_workspace_set_profiling(step.ws.handle, 1), "profiling")
    reps = max(3, min(args.steps, 10))
    for k in range(reps):
        d_ids, d_g, out = dev[k % nb]
        flush.zero_()
        step.step(d_ids, d_g, out)
    ms = (ctypes.c_double * 8)()
    cnt = ctypes.c_uint64()
    P._lib.check(lib.rs_workspace_phase_ms(step.ws.handle, ms, 8, ctypes.byref(cnt)), "phase_ms")
    P._lib.check(lib.rs_workspace_set_profiling(step.ws.handle, 0), "profiling")
    return {name: ms[i] for i, name in enumerate(PHASES)}


def pipelined_e2e(host, dim, run_step, n, uniq_b, barrier=None):
    """End to end through the public API with HOST buffers, pipelined the way
    a data loader drives it: step k's ids + grads go host->device on a copy
    stream, the step runs on the compute stream once they landed, its
    gathered rows go device->host on a second copy stream -- so H2D of step
    k+1, compute of step k and D2H of step k-1 overlap (PCIe is full duplex).
    Two device buffer sets; every copy of every step is inside the timed
    region (first H2D start -> last D2H end)."""
    import torch
    comp = torch.cuda.current_stream()
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    max_t = max(h[0].numel() for h in host)
    sets = [(torch.empty(max_t, dtype=torch.int64, device="cuda"),
             torch.empty((max_t, dim), dtype=torch.float32, device="cuda"),
             torch.empty((max_t, dim), dtype=torch.float32, device="cuda")) for _ in range(2)]
    in_free = [torch.cuda.Event() for _ in range(2)]
    out_free = [torch.cuda.Event() for _ in range(2)]
    for e in in_free + out_free:
        e.record(comp)

    def issue(k):
        h_ids, g, h_out = host[k % len(host)]
        T, b = h_ids.numel(), k % 2
        d_ids, d_g, d_out = sets[b]
        sh.wait_event(in_free[b])
        with torch.cuda.stream(sh):
            d_ids[:T].copy_(h_ids, non_blocking=True)
            d_g[:T].copy_(g, non_blocking=True)
        landed = torch.cuda.Event()
        landed.record(sh)
        comp.wait_event(landed)
        comp.wait_event(out_free[b])
        run_step(d_ids[:T], d_g[:T], d_out[:T])
        in_free[b].record(comp)
        done = torch.cuda.Event()
        done.record(comp)
        sd.wait_event(done)
        with torch.cuda.stream(sd):
            h_out[:T].copy_(d_out[:T], non_blocking=True)
        out_free[b].record(sd)

    warm = 2 * len(host)  # every (batch, buffer set, scratch parity) graph captured before timing
    for k in range(warm):
        issue(k)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(sh)
    for k in range(warm, warm + n):
        issue(k)
    t1.record(sd)
    torch.cuda.synchronize()
    t = t0.elapsed_time(t1) / 1e3
    uniq = sum(uniq_b[k % len(host)] for k in range(warm, warm + n))
    h2d = sum(host[k % len(host)][0].numel() * 8 + host[k % len(host)][1].numel() * 4 for k in range(warm, warm + n))
    d2h = sum(host[k % len(host)][2].numel() * 4 for k in range(warm, warm + n))
    return t, uniq, h2d // n, d2h // n


def workload_e2e(batches, dim, step_fn, n, uniq_b, barrier=None):
    """End to end the way the reference's run_workload drives a step
    (workload.cpp:506-581), through the public rs_feeder API: the data
    loader's pinned token ids + sequence lengths go host -> device on a copy
    stream that runs ahead (two buffer sets); the step generates its
    gradients (pseudo_sparse_grad, a pure hash of (sample id, step),
    workload.cpp:348-355 -- on the device, inside the timed region), runs
    dedup -> lookup -> reduce -> update, and its embedding checksum
    (run_workload's emb_checksum) comes back device -> host.  step_fn(feeder,
    h_ids, h_lengths, step) issues one step."""
    import torch

    from paper_2505_12663_b200.feed import Feeder
    host = [(torch.from_numpy(ids.view(np.int64)).pin_memory(),
             torch.from_numpy(np.asarray(lengths, np.uint64).view(np.int64)).pin_memory()) for lengths, ids in batches]
    feeder = Feeder(max(h[0].numel() for h in host), max(h[1].numel() for h in host), dim)
    warm = 2 * len(host)  # every (batch, buffer set, scratch parity) graph captured before timing
    for k in range(warm):
        step_fn(feeder, *host[k % len(host)], k % len(host))
    torch.cuda.synchronize()
    if barrier:
        barrier()
    comp = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    h0 = time.perf_counter()
    for k in range(warm, warm + n):
        step_fn(feeder, *host[k % len(host)], k % len(host))
    global _E2E_HOST_MS
    _E2E_HOST_MS = (time.perf_counter() - h0) * 1e3 / n
    t1.record(comp)
    torch.cuda.synchronize()
    t = t0.elapsed_time(t1) / 1e3
    feeder.close()
    uniq = sum(uniq_b[k % len(host)] for k in range(warm, warm + n))
    h2d = sum(host[k % len(host)][0].numel() * 8 + host[k % len(host)][1].numel() * 8 for k in range(warm, warm + n))
    return t, uniq, h2d // n, 8


def host_batches(batches, dim, W):
    import torch
    host = []
    for b, (lengths, ids) in enumerate(batches):
        h_ids = torch.from_numpy(ids.view(np.int64)).pin_memory()
        g = W.pseudo_grads(torch.from_numpy(W.sample_of_tokens(lengths).view(np.int64)), b, dim).cpu().pin_memory()
        h_out = torch.empty((len(ids), dim), dtype=torch.float32).pin_memory()
        host.append((h_ids, g, h_out))
    return host


def e2e_pass(args, cfg, batches, step, P, W, rank):
    """Same metric through rs_step with host buffers (pipelined_e2e)."""
    n = max(200, args.steps)  # ~0.1 ms per step: enough steps (~20 ms) to average the host-fed pipeline
    uniq_b = [int(np.unique(ids).size) for _, ids in batches]
    t, uniq, h2d, d2h = workload_e2e(batches, cfg["dim"], lambda f, hi, hl, k: f.step(step, hi, hl, k), n, uniq_b)
    tf, uf, hf, df = pipelined_e2e(host_batches(batches, cfg["dim"], W), cfg["dim"],
                                   lambda i, g, o: step.step(i, g, o), n, uniq_b)
    return {"value": uniq / t, "unit": "unique-ids/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": t / n * 1e3, "host_issue_ms_per_step": _E2E_HOST_MS,
            "io": "H2D token ids + sequence lengths; gradients generated in-step on the device "
                  "(pseudo_sparse_grad per sample, as run_workload does); D2H the step's embedding checksum",
            "full_io": {"value": uf / tf, "h2d_bytes_per_step": hf, "d2h_bytes_per_step": df, "ms_per_step": tf / n * 1e3,
                        "io": "H2D ids + per-token f32 gradients, D2H every gathered f32 row (PCIe-bound)"}}


# ------------------------------------------------------------- CPU arm
def cpu_baseline(cfg, batches, budget_s=15.0):
    """The reference's own path (distributed_lookup on SimCluster(1, TwoStage) +
    GradAccumulator accumulate/apply, OpenMP rows; Adagrad rows via the frozen
    restatement) on the host cores, bounded sample of the same workload."""
    import ctypes as C

    from oracle import bind
    kind = "reference" if bind.ref_available() else "port"
    o = bind.Oracle("ref" if kind == "reference" else "oracle")
    dim, vocab = cfg["dim"], cfg["vocab"]
    keys = np.arange(vocab, dtype=np.uint64) + TAG1
    h = C.c_void_p()
    assert o.cluster_create(1, cfg["capacity"] // 2, dim, 1, 0.75, 1 << 16, 3, C.byref(h)) == 0
    shard = bind.Table(o, 0, dim, handle=o.cluster_shard(h, 0))
    row = np.zeros(dim, np.float32)
    for r in range(vocab):
        o.pseudo_sparse_grad(r, 0, row, dim)
        shard.insert(int(keys[r]), row)
    cores = o.omp_max_threads() if kind == "reference" else 1
    times, uniq, reps = [], 0, 0
    t_start = time.time()
    for b, (lengths, ids) in enumerate(batches * 100):
        grads = o.token_grads(lengths, b, dim)
        if kind == "reference":
            sec = o.c1_step(h, ids, grads.reshape(-1), len(ids), 1, 0.01, 1e-8, None)
        else:
            t0 = time.perf_counter()
            u, _ = o.stage1(ids)
            for k in u:
                o.table_ensure(shard.h, int(k))
            ia, sa = o.accumulate_np(ids, grads, dim)
            o.apply(shard.h, ia, sa.reshape(-1), len(ia), 1, 0.01, 0.9, 0.999, 1e-8)
            sec = time.perf_counter() - t0
        if b >= 1:
            times.append(sec)
            uniq += len(np.unique(ids))
        reps += 1
        if time.time() - t_start > budget_s and len(times) >= 2:
            break
    o.cluster_destroy(h)
    t = sum(times)
    import platform
    cpu = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    return {"value": uniq / t, "unit": "unique-ids/s", "cores": cores, "kind": kind,
            "sample": f"{len(times)} config-1 steps (after 1 warm-up) on the reference path "
                      f"(distributed_lookup W=1 two-stage + accumulate + apply), {cpu}, nproc={os.cpu_count()}",
            "ms_per_step": t / len(times) * 1e3}


def run_reference(args, cfg):
    """The reference arm: the reference's own CPU implementation of the path
    (oracle/_ref/librsref.so, compiled from the reference sources; else the C
    restatement) on this host's cores, on our arm's config / metric / batches
    (the reference's own generator, same seeds) and the same K/W step schedule.
    N = 1: ref_c1_step (distributed_lookup on SimCluster(1) + accumulate +
    apply); N > 1: ref_dist_step (distributed_lookup over N simulated workers,
    per-owner accumulate + apply, as run_workload, workload.cpp:506-581) on the
    N ranks' batches of each step.  Under torchrun only rank 0 runs.  Nothing
    of the product (librsgpu) is loaded in this process."""
    import ctypes as C
    rank, world, local = dist_env()
    if rank != 0:
        return
    # every host core (torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 is the only worker here)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    from oracle import bind
    kind = "reference" if bind.ref_available() else "port"
    o = bind.Oracle("ref" if kind == "reference" else "oracle")
    dim, vocab = cfg["dim"], cfg["vocab"]
    nb = n_batches(args.warmup)
    batches = []  # [b][r] = (ids, grads) of rank r's batch b
    for b in range(nb):
        per = []
        for r in range(world):
            lengths, ids = o.generate(batch_seed(cfg, r, b), cfg["seqs"], cfg["mean"], cfg["max_len"], cfg["sigma"],
                                      cfg["zipf"], [vocab])
            per.append((ids, o.token_grads(lengths, b, dim)))
        batches.append(per)
    h = C.c_void_p()
    assert o.cluster_create(world, max(cfg["capacity"] // (2 * world), 1 << 16), dim, 1, 0.75, 1 << 16, 3,
                            C.byref(h)) == 0
    keys = np.arange(vocab, dtype=np.uint64) + TAG1
    row = np.zeros(dim, np.float32)
    shards = [bind.Table(o, 0, dim, handle=o.cluster_shard(h, s)) for s in range(world)]
    for t in shards:
        t.owned = False
    for r in range(vocab):
        o.pseudo_sparse_grad(r, 0, row, dim)
        shards[int(o.shard_of(int(keys[r]), world)) if world > 1 else 0].insert(int(keys[r]), row)
    uniq_b = [sum(len(np.unique(ids)) for ids, _ in per) for per in batches]

    def one(b):
        per = batches[b]
        if world == 1 and kind == "reference":
            ids, g = per[0]
            return o.c1_step(h, ids, g.reshape(-1), len(ids), 1, 0.01, 1e-8, None)
        if kind == "reference":
            flat = np.ascontiguousarray(np.concatenate([ids for ids, _ in per]))
            cnt = np.array([len(ids) for ids, _ in per], np.uint64)
            g = np.ascontiguousarray(np.concatenate([g for _, g in per]).reshape(-1))
            return o.dist_step(h, flat, cnt, g, 1, 0.01, 1e-8)
        t0 = time.perf_counter()  # the C restatement: same sequence of reference operations
        flat = np.ascontiguousarray(np.concatenate([ids for ids, _ in per]))
        cnt = np.array([len(ids) for ids, _ in per], np.uint64)
        out = np.zeros(len(flat) * dim, np.float32)
        z = np.zeros(world * world, np.uint64)
        o.distributed_lookup(h, flat, cnt, out, z, z.copy(), np.zeros(world, np.uint64), np.zeros(2, np.uint64))
        g = np.concatenate([g for _, g in per])
        own = np.array([o.shard_of(int(k), world) for k in flat]) if world > 1 else np.zeros(len(flat), int)
        for s_ in range(world):
            sel = np.nonzero(own == s_)[0]
            if len(sel):
                ia, sa = o.accumulate_np(flat[sel], g[sel], dim)
                o.apply(o.cluster_shard(h, s_), ia, sa.reshape(-1), len(ia), 1, 0.01, 0.9, 0.999, 1e-8)
        return time.perf_counter() - t0

    for k in range(args.warmup):
        one(k % nb)
    times, uniq = [], 0
    for k in range(args.warmup, args.warmup + args.steps):
        times.append(one(k % nb))
        uniq += uniq_b[k % nb]
    o.cluster_destroy(h)
    t = sum(times)
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    cores = o.omp_max_threads() if kind == "reference" else 1
    value = uniq / t
    sample = (f"{args.steps} timed steps after {args.warmup} warm-up steps over the {nb} batches of every rank "
              f"({'ref_c1_step: distributed_lookup W=1' if world == 1 else f'ref_dist_step: distributed_lookup W={world} (single-threaded simulation)'}"
              f" + accumulate + apply, OpenMP rows), {cpu}, nproc={os.cpu_count()}")
    res = {"metric": "unique-ID lookups+updates/sec", "value": value, "unit": "unique-ids/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / len(times) * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f32 rows, f64 optimizer math, u64 ids",
           "data": "synthetic: the reference's generator (mt19937_64, truncated lognormal lengths, Zipf 1.1 ids), "
                   "pseudo_sparse_grad gradients",
           "config": bench_config(cfg, world, nb, world > 1),
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "unique-ids/s", "cores": cores, "kind": kind, "sample": sample},
           "e2e": {"value": value, "unit": "unique-ids/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def self_launch(args):
    """--gpus N without a torchrun environment: re-exec this command under
    torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1)."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="run the row-sharded step even at N=1")
    ap.add_argument("--config", default="c1", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE config (default: the headline c1; c4 = the sharded 100M-key table; "
                         "c5 = long-tail sequences balanced across the ranks)")
    ap.add_argument("--balance", default="lpt", choices=["lpt", "rr"], help="config 5 rank assignment")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)  # does not return
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}; "
              "n_gpus reports WORLD_SIZE", file=sys.stderr)
    if args.config == "c2" and args.impl == "ours":
        run_c2(args, C2)
    elif args.config == "c3" and args.impl == "ours":
        run_c3(args, C3)
    elif args.impl == "reference":
        if args.config != "c1":
            print(json.dumps({"impl": "reference", "unavailable": f"the reference arm is timed on config 1 only "
                              f"(--config {args.config} is a parity/extra config of this repo)"}))
            return
        run_reference(args, C1)
    elif args.config == "c5":
        run_sharded(args, C5)
    elif args.config == "c4" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded):
        run_sharded(args, C4)
    elif args.config == "c4":
        run_ours(args, C4)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.sharded:
        run_sharded(args, C1)
    else:
        run_ours(args, C1)


if __name__ == "__main__":
    main()
