# host-side cost of one Feeder.step call (the e2e path), idle GPU and back to back
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2505_12663_b200 as P
from paper_2505_12663_b200.feed import Feeder
torch.cuda.set_device(0)
rng = np.random.default_rng(1)
lengths = np.full(1024, 128, np.uint64)
n = int(lengths.sum())
ids = (rng.zipf(1.1, n) % (1 << 20)).astype(np.int64)
h_ids = torch.from_numpy(ids).pin_memory()
h_len = torch.from_numpy(lengths.view(np.int64)).pin_memory()
pr = P.AdagradParams(lr=0.01)
t = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=64, optimizer="adagrad", initial_rows=1 << 21))
sp = P.SparseStep(t, n, pr)
f = Feeder(n, 1024, 64)
for k in range(8):
    f.step(sp, h_ids, h_len, k)
torch.cuda.synchronize()
def timeit(name, fn, N=50):
    xs = []
    for _ in range(N):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); xs.append(time.perf_counter() - t0)
    xs.sort()
    print(f"{name:28s} median {xs[len(xs)//2]*1e6:8.1f} us  min {xs[0]*1e6:8.1f} us", flush=True)
timeit("Feeder.step (idle gpu)", lambda: f.step(sp, h_ids, h_len, 3))
g = torch.randn((n, 64), device="cuda"); out = torch.empty_like(g); d_ids = h_ids.cuda()
timeit("SparseStep.step", lambda: sp.step(d_ids, g, out))
for N in (200,):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); t0 = time.perf_counter()
    for k in range(N):
        f.step(sp, h_ids, h_len, k & 1)
    th = time.perf_counter() - t0; e1.record(); torch.cuda.synchronize()
    print(f"back-to-back N={N}: host {th/N*1e6:.1f} us/step, device {e0.elapsed_time(e1)/N*1e3:.1f} us/step", flush=True)
    torch.cuda.synchronize()
    e0.record(); t0 = time.perf_counter()
    for k in range(N):
        sp.step(d_ids, g, out)
    th = time.perf_counter() - t0; e1.record(); torch.cuda.synchronize()
    print(f"  plain step N={N}: host {th/N*1e6:.1f} us/step, device {e0.elapsed_time(e1)/N*1e3:.1f} us/step", flush=True)
f.close()
