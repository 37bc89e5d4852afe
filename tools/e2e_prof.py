# device time per step of the host-fed workload step vs the device-resident step (config 1)
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_12663_b200 as P
from paper_2505_12663_b200 import workload as W
from paper_2505_12663_b200.feed import Feeder
torch.cuda.set_device(0)
vocab, dim = 1 << 20, 64
t = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=dim, optimizer="adagrad", chunk_rows=1 << 16,
                               initial_rows=vocab + (1 << 20)))
raw = torch.arange(vocab, dtype=torch.int64, device="cuda")
t.insert(raw + (1 << 62), W.pseudo_grads(raw, 0, dim))
lengths, ids = W.generate(1, 1024, 128.0, 4096, 1.0, 1.1, [vocab])
T = len(ids)
h_ids = torch.from_numpy(ids.view(np.int64)).pin_memory()
h_len = torch.from_numpy(lengths.view(np.int64)).pin_memory()
d_ids = h_ids.cuda(); d_len = h_len.cuda()
g = torch.empty((T, dim), device="cuda"); out = torch.empty_like(g); s = torch.zeros((), dtype=torch.float64, device="cuda")
st = P.SparseStep(t, T, P.AdagradParams(lr=0.01))
f = Feeder(T, len(lengths), dim)
lib = P.lib(); cs = torch.cuda.current_stream().cuda_stream
def run(name, fn, N=40):
    for k in range(6): fn(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); h0 = time.perf_counter()
    for k in range(N): fn(k)
    h = (time.perf_counter() - h0) / N * 1e6
    e1.record(); torch.cuda.synchronize()
    print(f"{name:30s} device {e0.elapsed_time(e1) / N * 1e3:7.1f} us/step   host {h:7.1f} us/step")
run("step (device-resident)", lambda k: st.step(d_ids, g, out))
run("pseudo_grads_jagged", lambda k: W.pseudo_grads_jagged(d_len, k, dim, T, out=g))
run("checksum", lambda k: P._lib.check(lib.rs_checksum(out.data_ptr(), out.numel(), s.data_ptr(), cs), "c"))
run("grads + step + checksum", lambda k: (W.pseudo_grads_jagged(d_len, k, dim, T, out=g), st.step(d_ids, g, out),
                                          lib.rs_checksum(out.data_ptr(), out.numel(), s.data_ptr(), cs)))
run("feeder (H2D + all)", lambda k: f.step(st, h_ids, h_len, k))
