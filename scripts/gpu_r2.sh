# round-2 evidence at HEAD: full GPU suite, smoke, default bench line (C5-128 + per-config),
# C5-128 step launch list, one ncu --set full capture of each dominant fine-level kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
fi
timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.log
if [ -z "$NO_PROF" ]; then
W=${WORKLOAD:-C5-128}
python scripts/prof_kernels.py step $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$W.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch.log 2>&1
echo "launches rc $?" >> gpurun_out/bench.log
python scripts/launch_summary.py gpurun_out/launches_$W.csv > gpurun_out/launch_summary_$W.txt 2>&1
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"${KREGEX:-st_brick_ws_kernel|fdm_strip_kernel|fdm_lines_kernel}" -c ${KCOUNT:-9} -f -o gpurun_out/prof_$W python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_full.log 2>&1
echo "full rc $?" >> gpurun_out/bench.log
fi
tail -4 gpurun_out/pytest_gpu.log 2>/dev/null; tail -1 gpurun_out/smoke.log 2>/dev/null; tail -c 3000 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
