import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1710_00882_b200 as B
from conftest import golden_clusters
from oracle import oracle as O
for k, (fr, table, row) in enumerate(golden_clusters()):
    nl = B.build_neighbor_list(fr, table.r_cut, 0.3)
    r = B.compute(fr, nl, table)
    df = np.abs(r.forces - row["forces"]).max()
    if df > 1e-9:
        bad = np.argmax(np.abs(r.forces - row["forces"]).max(1))
        print("cluster", k, "S", table.nspecies, "n", fr.positions.shape[0], "df", df, "bad atom", bad, "species", fr.species[bad])
        off, nb = nl.offsets, nl.neighbors
        pos = fr.positions
        for i in [bad]:
            for e in range(off[i], off[i+1]):
                j = nb[e]; d = np.linalg.norm(pos[j]-pos[i])
                print("  row", i, "->", j, "sp", fr.species[i], fr.species[j], "r", round(d,4))
        for i in range(len(pos)):
            if bad in nb[off[i]:off[i+1]]:
                print("  atom", i, "sp", fr.species[i], "has bad as nbr at r", round(np.linalg.norm(pos[bad]-pos[i]),4))
        break
