#!/bin/bash
# ncu --set full of the Tersoff kernel at configs 2 / 3 / 5, fp64 and mixed
# (one launch each, after two warm-up evaluations), summarised to JSON.
# Usage (on the GPU box): bash tools/ncu_kernels.sh OUTDIR
out=${1:-gpurun_out}
for c in "2 0" "2 1" "3 0" "3 1" "5 0" "5 1"; do
  set -- $c
  python tools/kone.py $1 $2 0 1 > /dev/null 2>&1 || { echo "plain run failed: $c"; continue; }
  timeout 600 ncu --set full --clock-control none -k regex:k_tersoff_warp --launch-skip 2 -c 1 \
    -f -o /tmp/tk_c$1_p$2 python tools/kone.py $1 $2 0 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/tk_c$1_p$2.ncu-rep $out/ncu_tk_c$1_p$2.json > /dev/null
  ncu -i /tmp/tk_c$1_p$2.ncu-rep --page raw --csv > $out/ncu_tk_c$1_p$2_raw.csv
done
