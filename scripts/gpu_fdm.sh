cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_slab.py -x -q -m gpu ${PTK} > gpurun_out/pytest_fdm.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_fdm.log
STMG_ROOT=$GRAFT_REPO_ROOT timeout 300 python scripts/time_ops.py C5-128 C4 C3 --asm --xfer 2>&1 | tail -4
