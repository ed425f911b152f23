O=gpurun_out/r02_row; mkdir -p $O
KT_CONFIGS=5 KT_OUT=$O/ktime11.json timeout 1200 python tools/ktime_so.py tools/ab/cur.so tools/ab/pf32_m3.so tools/ab/pf32_m4.so 2> $O/ktime.err; echo "ktime rc=$?"; tail -3 $O/ktime.err
