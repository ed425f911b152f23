# ncu source-level captures of the mixed kernel at configs 3 and 4 (and fp64 c4)
O=gpurun_out/r02_src; mkdir -p $O
for cp in "3 1" "4 1" "4 0"; do set -- $cp
  python tools/kone.py $1 $2 0 1 > /dev/null 2>&1 || continue
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tersoff_warp --launch-skip 2 -c 1 \
    -f -o /tmp/src_c$1_p$2 python tools/kone.py $1 $2 0 3 > /dev/null 2>&1
  ncu -i /tmp/src_c$1_p$2.ncu-rep --page source --csv --print-source cuda,sass > $O/src_c$1_p$2.csv 2>/dev/null
  ncu -i /tmp/src_c$1_p$2.ncu-rep --page raw --csv > $O/raw_c$1_p$2.csv
  python tools/ncu_src.py $O/src_c$1_p$2.csv 45 > $O/src_c$1_p$2.txt
done
ls -la $O
