O=gpurun_out/r02_row; mkdir -p $O
KT_CONFIGS=5 KT_OUT=$O/ktime10.json timeout 1200 python tools/ktime_so.py tools/ab/cur.so tools/ab/outline.so 2> $O/ktime.err; echo "ktime rc=$?"; tail -3 $O/ktime.err
