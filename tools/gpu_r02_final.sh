# Round-2 verification + measurement on one B200 (run from the repo root):
# GPU tests, smoke, the bench (default = config 5) and its reference arm, the
# two-rank functional run, per-config table, ncu launch list + --set full.
O=${OUT:-gpurun_out/r02_final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
BENCH_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 5 --warmup 3 --dd-md-steps 10 --e2e-steps 3 > $O/n2_gloo.json 2> $O/n2_gloo.err; echo "n2 rc=$?"
CB_CONFIGS=1,2,3,4,5 CB_STEPS=50 CB_OUT=$O/configs.json timeout 1200 python tools/configs_bench.py > $O/configs.log 2>&1; echo "configs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1800 bash tools/ncu_kernels.sh $O/ncu "2 3 4 5" > $O/ncu_kernels.log 2>&1; echo "ncu full rc=$?"
timeout 600 python tools/e2e_stream.py 5 0 131072 > $O/e2e_stream_c5.json 2> $O/e2e_stream.err; echo "e2e stream rc=$?"
timeout 900 python tools/md_loose_ab.py 5 200 30 0 2> $O/md_loose.err | grep "^{" > $O/md_loose_c5.jsonl; echo "md loose rc=$?"
timeout 600 python tools/row_crossover.py 20 32 40 50 64 2> $O/row_crossover.err | grep "^{" > $O/row_crossover.jsonl; echo "crossover rc=$?"
timeout 600 bash tools/md_step_launches.sh 5 12 $O/md_step_c5.csv; echo "md step launches rc=$?"
