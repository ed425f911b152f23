"""Probe: can torch.distributed NCCL P2P (batch_isend_irecv, as decomp._exchange
uses) and all_reduce be captured in a CUDA graph on this image?  One rank
exchanging with itself (left = right = 0).
Usage: python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1
       --master-port 29555 tools/nccl_capture_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_1710_00882_b200 import decomp

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
a = torch.arange(30, dtype=torch.float64, device=dev).reshape(10, 3)
b = -a[:7].clone()
r = torch.ones(7, dtype=torch.float64, device=dev)
out = {}


def step():
    fl, fr = decomp._exchange((a, b), ((7, 3), (10, 3)), torch.float64, dev, 0, 0)
    s = fl.sum() + 2 * fr.sum()
    r.fill_(1.0)
    dist.all_reduce(r)
    return s, r


print("stage: eager", flush=True)
s, rr = step()
torch.cuda.synchronize()
print("stage: eager done", flush=True)
out["eager"] = [float(s), float(rr.sum())]
try:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    print("stage: capture", flush=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        sg, rg = step()
    print("stage: replay", flush=True)
    for _ in range(3):
        a.mul_(2.0); b.mul_(2.0)
        g.replay()
    torch.cuda.synchronize()
    out["graph"] = [float(sg), float(rg.sum())]
    out["graph_expected"] = [float(-a[:7].sum() * 0 + (b.sum() + 2 * a.sum())), 7.0]
    out["ok"] = abs(out["graph"][0] - out["graph_expected"][0]) < 1e-9
except Exception as e:  # noqa: BLE001
    out["graph_error"] = repr(e)[:400]
print(json.dumps(out), flush=True)
try:
    del g
except NameError:
    pass
torch.cuda.synchronize()
print("stage: destroy", flush=True)
dist.destroy_process_group()
print("stage: exit", flush=True)
