#!/bin/bash
# ncu --set full of the Tersoff kernel(s) of one evaluation (tools/kone.py; the
# atom-per-lane row kernel and/or the warp-chunk kernel) at the given configs,
# fp64 and mixed; raw CSV + source-level CSV per capture and a JSON summary of
# the dominant kernel (tools/ncu_kernels_json.py).
# Usage (on the GPU box): bash tools/ncu_kernels.sh OUTDIR "2 3 4 5"
out=${1:-gpurun_out}
cfgs=${2:-"2 3 5"}
mkdir -p $out
for c in $cfgs; do for p in 0 1; do
  python tools/kone.py $c $p 0 1 > /dev/null 2>&1 || { echo "plain run failed: $c $p"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tersoff_(row|warp)" -c 2 \
    -f -o /tmp/tk_c${c}_p${p} python tools/kone.py $c $p 0 1 > /dev/null 2>&1
  ncu -i /tmp/tk_c${c}_p${p}.ncu-rep --page raw --csv > $out/ncu_tk_c${c}_p${p}_raw.csv
  ncu -i /tmp/tk_c${c}_p${p}.ncu-rep --page source --csv --print-source sass > $out/ncu_tk_c${c}_p${p}_sass.csv 2>/dev/null
done; done
python tools/ncu_kernels_json.py $out/ncu_kernels.json $out
