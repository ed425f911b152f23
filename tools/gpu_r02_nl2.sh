for v in atoms cells; do
  if [ $v = cells ]; then export TB_NL_CELLS=1; else unset TB_NL_CELLS; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_nl2_$v.csv python tools/kone.py 2 0 0 1 > /dev/null 2>&1
  echo "== $v c2"; grep -E "k_nl_atoms|k_nl_cells" gpurun_out/r02_nl2_$v.csv | awk -F, '{print $NF}'
  MC_CONFIGS=2,5 MC_STEPS=200 MC_OUT=gpurun_out/r02_md25_$v.json python tools/md_configs.py 2>&1 | grep "{"
done
