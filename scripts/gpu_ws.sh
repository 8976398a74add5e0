# warp-specialised st_brick: parity tests of the operator + timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/time_ops.py ${WL:-C5-64 C5-128} > gpurun_out/time_ops.log 2>&1; echo "time rc $?"; cat gpurun_out/time_ops.log | tail -5
timeout 900 python -m pytest tests/test_gpu_operator.py -x -q -m gpu -k "brick or config_vmult or every_field" > gpurun_out/pytest_brick.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_brick.log
