cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ref_binding.py tests/test_gpu_fullsize.py -q -m gpu -k "${PK:-binding or C2 or C3}" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests/test_gpu_multigrid.py -q -m gpu -k "gmres_solve" > gpurun_out/pytest_gm.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_gm.log
