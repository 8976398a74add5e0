cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_slab.py -x -q -m gpu -k "asm or fdm or smoother or vcycle" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_c3.log
timeout 600 python scripts/time_ops.py C3 C4 --asm 2>&1 | tail -2
