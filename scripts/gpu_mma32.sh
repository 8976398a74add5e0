# 27-dof tensor-core smoother: parity tests, C3 V-cycle sweep, one ncu capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_slab.py -m gpu -q -rf --timeout 600 -x > gpurun_out/pytest_mg.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_mg.log
timeout 400 python scripts/sweep.py C3n > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo "sweep rc $?" >> gpurun_out/sweep_c3.err
timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply_mma32" -c 1 -o gpurun_out/prof_mma32 python scripts/prof_kernels.py kernels C3 > gpurun_out/ncu_mma32.log 2>&1
echo "ncu rc $?"
tail -4 gpurun_out/pytest_mg.log; cut -c 1-600 gpurun_out/sweep_c3.jsonl; tail -2 gpurun_out/sweep_c3.err
