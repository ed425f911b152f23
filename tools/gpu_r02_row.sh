O=gpurun_out/r02_row; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_md.py tests/test_gpu_stream.py tests/test_gpu_dnl.py tests/test_gpu_decomp.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -12 $O/pytest.txt
cp paper_1710_00882_b200/lib/libtersoff_b200.so /tmp/cur.so
KT_CONFIGS=2,4,5 KT_OUT=$O/ktime4.json timeout 1200 python tools/ktime_so.py tools/ab/base.so /tmp/cur.so 2> $O/ktime.err; echo "ktime rc=$?"; tail -3 $O/ktime.err
