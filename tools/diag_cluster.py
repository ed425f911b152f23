"""Diagnostics: a free cluster cut around atom 2150 of small config 4."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.system import SimulationBox
st, tn = structures.config(4, small=True)
t = B.builtin_params(tn)
c = st.positions[2150]
L = st.box.lengths
d = st.positions - c
d -= L * np.round(d / L)
sel = np.where((d * d).sum(1) < 6.5 ** 2)[0]
pos = d[sel] + 20.0
class Fr: pass
fr = Fr(); fr.positions = np.ascontiguousarray(pos); fr.species = np.zeros(len(sel), np.int64)
fr.box = SimulationBox([60, 60, 60], (False, False, False))
nl = B.build_neighbor_list(fr, t.r_cut, 0.3)
out = {"sel": sel, "pos": pos}
for prec in ("double", "single"):
    for sc in ("atomic", "gather"):
        r = B.compute(fr, nl, t, B.make_variant("B200", precision=prec, scatter=sc))
        out[prec + "_" + sc] = r.forces
np.savez("gpurun_out/diag_cluster.npz", **out)
print("ok", len(sel))
