cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py -x -q -m gpu -k "${PT:-brick or config_vmult}" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_iter.log
timeout 600 python scripts/time_ops.py ${TW:-C5-128 C4 C5-64} ${TA} 2>&1 | tail -8
if [ -n "$PROF" ]; then
python scripts/prof_kernels.py kernels ${W:-C5-128} > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"${K:-st_brick_kernel}" -c 1 -o gpurun_out/prof_iter python scripts/prof_kernels.py kernels ${W:-C5-128} > gpurun_out/ncu_iter.log 2>&1; echo "ncu rc $?"
fi
