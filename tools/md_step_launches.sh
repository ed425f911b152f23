# Launch list of a host-driven NVE run (tb_md_step per step) at a config: the
# kernels of a device list rebuild with their durations (the graph loop runs the
# same kernels inside conditional nodes, which ncu does not list).
# Usage: bash tools/md_step_launches.sh CONFIG STEPS OUT.csv
c=${1:-5}; n=${2:-12}; out=${3:-gpurun_out/md_step_launches.csv}
cat > /tmp/md_step_run.py <<PY
import os, sys
sys.path.insert(0, os.getcwd())
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.md import RunConfig, run_nve
st, tn = structures.config($c)
t = B.builtin_params(tn)
r = run_nve(st, t, RunConfig(dt=1.0, steps=$n, skin=0.3, rebuild_every=10, record_every=10,
                             variant=B.make_variant("B200")), loop="step")
print(r["loop"], r["rebuilds"])
PY
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out python /tmp/md_step_run.py > /dev/null 2>&1
python tools/ncu_launch_table.py $out > ${out%.csv}.json
