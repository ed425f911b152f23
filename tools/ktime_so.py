"""A/B kernel timing of alternative builds of the library (tb_profile CUDA
events around each Tersoff launch): python tools/ktime_so.py LIB.so [...]
Only the round-1 C-ABI subset is used, so older builds load too."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.paramfile import builtin_params

P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
cfgs = [int(c) for c in os.environ.get("KT_CONFIGS", "2,5").split(",")]
reps = int(os.environ.get("KT_REPS", "30"))
states = {c: structures.config(c) for c in cfgs}
out = {}
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    lib.tb_create.argtypes = [I, ctypes.POINTER(P)]
    lib.tb_set_params.argtypes = [P, I, P, P, P]
    lib.tb_set_stream.argtypes = [P, P]
    lib.tb_nlist_create.argtypes = [P, ctypes.POINTER(P)]
    lib.tb_build_neighbors.argtypes = [P, P, I64, P, P, P, D, D]
    lib.tb_compute_device.argtypes = [P, P, P, P, D, I, I, P, P, P, P]
    lib.tb_profile.argtypes = [P, I]
    lib.tb_profile_read.argtypes = [P, P, P]
    ctx = P(); assert lib.tb_create(0, ctypes.byref(ctx)) == 0
    s = torch.cuda.Stream(); torch.cuda.set_stream(s)
    lib.tb_set_stream(ctx, P(s.cuda_stream))
    res = {}
    for c, (st, tn) in states.items():
        t = builtin_params(tn)
        v = t.views("double")
        pair = np.ascontiguousarray(v["pair_matrix"]); trip = np.ascontiguousarray(v["trip_matrix"])
        lib.tb_set_params(ctx, t.nspecies, pair.ctypes.data, trip.ctypes.data, None)
        pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
        n = st.natoms
        f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); r = torch.zeros(8, dtype=torch.float64, device="cuda")
        nl = P(); lib.tb_nlist_create(ctx, ctypes.byref(nl))
        L = np.ascontiguousarray(st.box.lengths, dtype=np.float64); per = np.ones(3, np.int32)
        assert lib.tb_build_neighbors(ctx, nl, n, pos.data_ptr(), L.ctypes.data, per.ctypes.data, float(t.r_cut), 0.3) == 0
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        for prec in (0, 1):
            for _ in range(3):
                lib.tb_compute_device(ctx, nl, pos.data_ptr(), sp.data_ptr(), float(t.r_cut), prec, 0, f.data_ptr(), None, r.data_ptr(), None)
            torch.cuda.synchronize()
            lib.tb_profile(ctx, 1)
            for _ in range(reps):
                flush.zero_()
                lib.tb_compute_device(ctx, nl, pos.data_ptr(), sp.data_ptr(), float(t.r_cut), prec, 0, f.data_ptr(), None, r.data_ptr(), None)
            torch.cuda.synchronize()
            lib.tb_profile(ctx, 0)
            tot, cnt = ctypes.c_double(), ctypes.c_int64()
            lib.tb_profile_read(ctx, ctypes.byref(tot), ctypes.byref(cnt))
            res[f"c{c}_p{prec}_us"] = round(1e3 * tot.value / reps, 2)  # per evaluation (all Tersoff launches)
            res[f"c{c}_p{prec}_launches"] = cnt.value / reps
            res[f"c{c}_p{prec}_E"] = float(r[0])
        del pos, sp, f, flush
    out[os.path.basename(path)] = res
    print(json.dumps({os.path.basename(path): res}), flush=True)
json.dump(out, open(os.environ.get("KT_OUT", "gpurun_out/ktime.json"), "w"), indent=1)
