O=gpurun_out/r02_row; mkdir -p $O
cp paper_1710_00882_b200/lib/libtersoff_b200.so /tmp/cur.so
KT_CONFIGS=5 KT_OUT=$O/ktime9.json timeout 1200 python tools/ktime_so.py /tmp/cur.so tools/ab/sst_m3.so tools/ab/sst_m4.so tools/ab/sst_m4_sacc.so 2> $O/ktime.err; echo "ktime rc=$?"; tail -3 $O/ktime.err
