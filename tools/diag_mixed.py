"""Dump GPU mixed/double forces for small config 4 (diagnostics)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
st, tn = structures.config(4, small=True)
t = B.builtin_params(tn)
nl = B.build_neighbor_list(st, t.r_cut, 0.3)
out = {}
for prec in ("double", "single"):
    r = B.compute(st, nl, t, B.make_variant("B200", precision=prec))
    out[prec] = r.forces
    out[prec + "_e"] = r.per_atom_energy
np.savez("gpurun_out/diag_mixed.npz", **out)
print("ok")
