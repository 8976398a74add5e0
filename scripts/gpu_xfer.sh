cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transfer_large.py tests/test_gpu_multigrid.py -x -q -m gpu -k "transfer" > gpurun_out/pytest_xfer.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_xfer.log
timeout 600 python scripts/time_ops.py C5-128 --xfer 2>&1 | tail -2
