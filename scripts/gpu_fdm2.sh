cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multigrid.py -x -q -m gpu -k "fdm or asm_correction" > gpurun_out/pytest_fdm.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_fdm.log
timeout 300 python scripts/time_ops.py C5-128 --asm 2>&1 | tail -2
