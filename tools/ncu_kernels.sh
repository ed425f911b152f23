#!/bin/bash
# ncu --set full of the Tersoff kernel (one launch after two warm-up
# evaluations, tools/kone.py) at the given configs, fp64 and mixed; raw CSV
# per capture + a JSON summary (tools/ncu_kernels_json.py).
# Usage (on the GPU box): bash tools/ncu_kernels.sh OUTDIR "2 3 4 5"
out=${1:-gpurun_out}
cfgs=${2:-"2 3 5"}
mkdir -p $out
for c in $cfgs; do for p in 0 1; do
  python tools/kone.py $c $p 0 1 > /dev/null 2>&1 || { echo "plain run failed: $c $p"; continue; }
  timeout 900 ncu --set full --clock-control none -k regex:k_tersoff_warp --launch-skip 2 -c 1 \
    -f -o /tmp/tk_c${c}_p${p} python tools/kone.py $c $p 0 3 > /dev/null 2>&1
  ncu -i /tmp/tk_c${c}_p${p}.ncu-rep --page raw --csv > $out/ncu_tk_c${c}_p${p}_raw.csv
done; done
python tools/ncu_kernels_json.py $out/ncu_kernels.json $out
