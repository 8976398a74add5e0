cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_slab.py -x -q -m gpu > gpurun_out/pytest_mr.log 2>&1; echo "pytest rc $?"; tail -30 gpurun_out/pytest_mr.log
