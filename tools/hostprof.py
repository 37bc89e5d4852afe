# host-side cost of one step call with an idle GPU (sync before each call)
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29601")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist, numpy as np
import paper_2505_12663_b200 as P
from paper_2505_12663_b200.dist import ShardedTable
from paper_2505_12663_b200 import _lib as L
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
n = 1 << 17
st = ShardedTable(P.TableConfig(capacity=1 << 22, embedding_dim=64, optimizer="adagrad", initial_rows=1 << 21), max_tokens=n)
ids = torch.randint(0, 1 << 18, (n,), device="cuda")
g = torch.randn((n, 64), device="cuda")
out = torch.empty_like(g)
pr = P.AdagradParams(lr=0.01)
t = P.EmbedTable(P.TableConfig(capacity=1 << 22, embedding_dim=64, optimizer="adagrad", initial_rows=1 << 21))
sp = P.SparseStep(t, n, pr)
for _ in range(6):
    st.step(ids, g, pr, out); sp.step(ids, g, out)
torch.cuda.synchronize()
lib = L.lib(); pc = pr.c(); s = torch.cuda.current_stream().cuda_stream
def timeit(name, fn, N=30):
    xs = []
    for _ in range(N):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); xs.append(time.perf_counter() - t0)
    xs.sort()
    print(f"{name:28s} median {xs[len(xs)//2]*1e6:8.1f} us  min {xs[0]*1e6:8.1f} us")
timeit("ShardedTable.step", lambda: st.step(ids, g, pr, out))
timeit("rs_dist_step raw", lambda: lib.rs_dist_step(st._c, st.shard.handle, ids.data_ptr(), n, g.data_ptr(), out.data_ptr(), C.byref(pc), s))
timeit("SparseStep.step", lambda: sp.step(ids, g, out))
timeit("rs_step raw", lambda: lib.rs_step(sp.ws.handle, t.handle, ids.data_ptr(), n, g.data_ptr(), out.data_ptr(), C.byref(pc), s))
fl = torch.empty(1 << 27, device="cuda")
timeit("flush.zero_", lambda: fl.zero_())
ev = torch.cuda.Event(enable_timing=True)
timeit("event.record", lambda: ev.record())
os.environ["RS_NO_GRAPH"] = "1"
st.close()
dist.destroy_process_group()
