# host-side cost of one sharded step call (W=1), per component
import os, sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29601")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist, numpy as np
import paper_2505_12663_b200 as P
from paper_2505_12663_b200.dist import ShardedTable
from paper_2505_12663_b200 import _lib as L
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
st = ShardedTable(P.TableConfig(capacity=1 << 20, embedding_dim=64, optimizer="adagrad"), max_tokens=1 << 17)
ids = torch.randint(0, 1 << 18, (1 << 17,), device="cuda")
g = torch.randn((1 << 17, 64), device="cuda")
out = torch.empty_like(g)
pr = P.AdagradParams(lr=0.01)
for _ in range(5): st.step(ids, g, pr, out)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N): st.step(ids, g, pr, out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("python step call us", (t1 - t0) / N * 1e6, "gpu-bound us", (t2 - t0) / N * 1e6)
lib = L.lib(); pc = pr.c(); s = torch.cuda.current_stream().cuda_stream
t0 = time.perf_counter()
for _ in range(N): lib.rs_dist_step(st._c, st.shard.handle, ids.data_ptr(), ids.numel(), g.data_ptr(), out.data_ptr(), C.byref(pc), s)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("raw ctypes call us", (t1 - t0) / N * 1e6)
t0 = time.perf_counter()
for _ in range(N): torch.cuda.current_stream().cuda_stream
print("current_stream us", (time.perf_counter() - t0) / N * 1e6)
t0 = time.perf_counter()
for _ in range(N): pr.c()
print("params.c us", (time.perf_counter() - t0) / N * 1e6)
st.close()
