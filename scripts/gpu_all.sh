# tests + smoke + bench + ncu (launch list, then one full capture per hot kernel)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 ${PYTEST_ARGS:--k "not full_size"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.log
if [ -z "$NO_PROF" ]; then
python scripts/prof_kernels.py step $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch.log 2>&1
echo "launches rc $?" >> gpurun_out/pytest_gpu.log
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_lines_kernel|st_apply_kernel" -c 1 -o gpurun_out/prof_st python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_st.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply" -c 1 -o gpurun_out/prof_asm python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_asm.log 2>&1
echo "full rc $?" >> gpurun_out/pytest_gpu.log
fi
tail -4 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
