# quick iteration: selected GPU tests (PYTEST_K), bench without the CPU leg, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
timeout 900 python -m pytest tests -m gpu -x -q -rf --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $W ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?"
grep -o '"ms_per_step": [0-9.]*\|"vmult_ms": [0-9.]*\|"vcycle_ms": [0-9.]*\|"asm_fine_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench.log; tail -2 gpurun_out/bench.err | cut -c1-300
if [ -n "$LAUNCHES" ]; then
python scripts/prof_kernels.py step $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv | head -20
fi
