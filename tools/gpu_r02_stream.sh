O=gpurun_out/r02_stream; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stream.py -q -p no:cacheprovider > $O/pytest_stream.txt 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_stream.txt
timeout 900 python tools/e2e_stream.py 5 0 131072 > $O/e2e_stream_c5.json 2> $O/e2e_stream_c5.err; echo "c5 rc=$?"; cat $O/e2e_stream_c5.json; tail -3 $O/e2e_stream_c5.err
timeout 900 python tools/e2e_stream.py 4 0 32768 > $O/e2e_stream_c4.json 2> $O/e2e_stream_c4.err; echo "c4 rc=$?"; cat $O/e2e_stream_c4.json; tail -3 $O/e2e_stream_c4.err
