#!/bin/bash
# Atomic-vs-gather scatter evidence (north_star (2)): event-timed graph steps
# and Tersoff-kernel times for both modes at configs 2/3/5 (fp64 + mixed),
# then an ncu launch list (duration + DRAM bytes per kernel) of one evaluation
# per mode.  Usage (GPU box): bash tools/scatter_ab.sh OUTDIR
out=${1:-gpurun_out}
mkdir -p $out
for s in 0 1; do
  CB_CONFIGS=2,3,5 CB_SCATTER=$s CB_MD=0 CB_OUT=$out/scatter_ab_s$s.json python tools/configs_bench.py > $out/scatter_ab_s$s.log 2>&1
done
for c in 2 3 5; do for p in 0 1; do for s in 0 1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --launch-skip 4 --csv --log-file $out/scatter_ncu_c${c}_p${p}_s${s}.csv \
    python tools/kone.py $c $p $s 3 > /dev/null 2>&1
done; done; done
