"""A few device-side list rebuilds of one configuration (for ncu --set full)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_00882_b200 import _native, structures  # noqa: E402
from paper_1710_00882_b200.kernels import compute  # noqa: E402
from paper_1710_00882_b200.neighbor import build_neighbor_list  # noqa: E402
from paper_1710_00882_b200.paramfile import builtin_params  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st, tn = structures.config(cfg)
t = builtin_params(tn)


class D:
    pass


d = D()
d.positions = torch.from_numpy(st.positions).cuda()
d.species = torch.from_numpy(st.species.astype(np.int32)).cuda()
d.box = st.box
ctx = _native.default_context(0)
ctx.set_table(t)
nl = build_neighbor_list(d, t.r_cut, 0.3)
compute(d, nl, t)
for _ in range(3):
    nl.rebuild_on_device(d.positions, d.species)
torch.cuda.synchronize()
