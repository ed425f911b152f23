"""Time the device-side list rebuild (tb_nlist_rebuild_device) vs the host-
synchronised build on BASELINE configs; DNL_NCU=1 does a single rebuild for
ncu launch lists."""
import ctypes
import json
import os
import time

import numpy as np
import torch

from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.kernels import compute
from paper_1710_00882_b200.neighbor import build_neighbor_list
from paper_1710_00882_b200.paramfile import builtin_params

ncu = os.environ.get("DNL_NCU") == "1"
out = {}
for cfg in [int(c) for c in os.environ.get("DNL_CONFIGS", "2,3,5").split(",")]:
    st, tn = structures.config(cfg)
    t = builtin_params(tn)

    class S:
        pass

    d = S()
    d.positions = torch.from_numpy(st.positions).cuda()
    d.species = torch.from_numpy(st.species.astype(np.int32)).cuda()
    d.box = st.box
    ctx = _native.default_context(0)
    ctx.set_table(t)
    nl = build_neighbor_list(d, t.r_cut, 0.3)
    compute(d, nl, t)
    reps = 1 if ncu else 20
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    nl.rebuild_on_device(d.positions, d.species)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        nl.rebuild_on_device(d.positions, d.species)
    torch.cuda.synchronize()
    dev_ms = (time.perf_counter() - t0) / reps * 1e3
    if ncu:
        continue
    t0 = time.perf_counter()
    for _ in range(reps):
        build_neighbor_list(d, t.r_cut, 0.3)
    torch.cuda.synchronize()
    host_ms = (time.perf_counter() - t0) / reps * 1e3
    out[cfg] = {"atoms": st.natoms, "device_rebuild_ms": dev_ms, "host_build_ms": host_ms}
    print(json.dumps({cfg: out[cfg]}), flush=True)
