"""Probe: NCCL P2P (to self, world size 1) and all-reduce on zero-copy views of
C-owned device memory (__cuda_array_interface__, as decomp.B200Domain hands
its buffers to Comm), eager and inside a CUDA-graph capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_1710_00882_b200.decomp import _Dev

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29581")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
owner = torch.arange(64, dtype=torch.float64, device="cuda")  # stands in for C-owned memory
src = torch.as_tensor(_Dev(owner.data_ptr(), (8, 3), "f8"), device="cuda")
dst_mem = torch.zeros(64, dtype=torch.float64, device="cuda")
dst = torch.as_tensor(_Dev(dst_mem.data_ptr() + 8 * 24, (8, 3), "f8"), device="cuda")
s = torch.cuda.Stream(); torch.cuda.set_stream(s)

def step():
    ops = [dist.P2POp(dist.isend, src, 0), dist.P2POp(dist.irecv, dst, 0)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    dist.all_reduce(dst_mem)

step(); torch.cuda.synchronize()
ok1 = torch.equal(dst_mem[24:48], owner[:24])
dst_mem.zero_(); owner.add_(1.0)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    step()
dst_mem.zero_(); torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
ok2 = torch.equal(dst_mem[24:48], owner[:24])
print({"eager_ok": bool(ok1), "graph_ok": bool(ok2)}, flush=True)
del g
os._exit(0)
