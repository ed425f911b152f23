O=gpurun_out/r02_row; mkdir -p $O
KT_CONFIGS=5 KT_OUT=$O/ktime7.json timeout 1200 python tools/ktime_so.py tools/ab/row4_cur.so tools/ab/row7_sacc.so tools/ab/row7_sacc_recos.so 2> $O/ktime.err; echo "ktime rc=$?"; tail -3 $O/ktime.err
