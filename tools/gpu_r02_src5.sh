O=gpurun_out/r02_src5; mkdir -p $O
python tools/kone.py 5 0 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tersoff_warp --launch-skip 2 -c 1 \
    -f -o /tmp/src_c5_p0 python tools/kone.py 5 0 0 3 > /dev/null 2>&1
ncu -i /tmp/src_c5_p0.ncu-rep --page source --csv --print-source cuda,sass > $O/src_c5_p0.csv 2>/dev/null
ncu -i /tmp/src_c5_p0.ncu-rep --page raw --csv > $O/raw_c5_p0.csv
python tools/ncu_src.py $O/src_c5_p0.csv 50 > $O/src_c5_p0.txt
python tools/sass_summary.py $O/src_c5_p0.csv > $O/sass_c5_p0.txt 2>&1
