# fast iteration: GPU tests (stop at first failure) + bench without the CPU leg
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rf --timeout 300 ${PYTEST_ARGS:--k "not full_size"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.log
tail -4 gpurun_out/pytest_gpu.log; grep -o '"ms_per_step": [0-9.]*\|"vmult_ms": [0-9.]*\|"vcycle_ms": [0-9.]*\|"asm_fine_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench.log; tail -2 gpurun_out/bench.err
