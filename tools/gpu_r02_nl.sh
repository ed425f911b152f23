for v in atoms cells; do
  if [ $v = cells ]; then export TB_NL_CELLS=1; else unset TB_NL_CELLS; fi
  echo "== $v"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_nl_$v.csv python tools/kone.py 5 0 0 1 > /dev/null 2>&1
  grep -E "k_nl_atoms|k_nl_cells" gpurun_out/r02_nl_$v.csv | head -2
done
unset TB_NL_CELLS
timeout 900 python -m pytest -q tests/test_gpu_parity.py tests/test_gpu_dnl.py tests/test_gpu_decomp.py -p no:cacheprovider 2>&1 | tail -2
MC_CONFIGS=3 MC_STEPS=200 MC_OUT=gpurun_out/r02_md3c.json python tools/md_configs.py 2>&1 | grep "{"
