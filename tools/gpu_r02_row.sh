O=gpurun_out/r02_row; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dnl.py tests/test_gpu_decomp.py tests/test_gpu_md.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "pair or neighbor or list or config" > $O/pytest_full.txt 2>&1; echo "pytest full rc=$?"; tail -3 $O/pytest_full.txt
bash tools/md_step_launches.sh 5 12 $O/md_step_c5.csv
grep -E "k_nl_atoms|k_nl_compact|k_fill_lanes" -A3 $O/md_step_c5.json | grep -E "tb::|us_mean"
