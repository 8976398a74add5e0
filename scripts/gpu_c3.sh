# exact-cell smoothers: parity tests, C3 default (tensor cores) vs STMG_ASM27=warp (DFMA), launch list, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigrid.py -m gpu -q -rf --timeout 600 -k "27dof or q2_exact or 2d_q4 or (asm_correction and C3)" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_c3.log
STMG_ASM27=warp timeout 600 python scripts/sweep.py C3n > gpurun_out/sweep_c3_warp.jsonl 2> gpurun_out/sweep_c3_warp.err
timeout 600 python scripts/sweep.py C3n > gpurun_out/sweep_c3_mma.jsonl 2> gpurun_out/sweep_c3_mma.err

python scripts/prof_kernels.py step C3 > gpurun_out/prof_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c3.csv python scripts/prof_kernels.py step C3 > gpurun_out/ncu_launch_c3.log 2>&1
echo "launches rc $?" >> gpurun_out/pytest_c3.log
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply_mma32" -c 1 -o gpurun_out/prof_mma32 python scripts/prof_kernels.py kernels C3 > gpurun_out/ncu_mma32.log 2>&1
echo "full rc $?" >> gpurun_out/pytest_c3.log
tail -5 gpurun_out/pytest_c3.log; for f in gpurun_out/sweep_c3_warp.jsonl gpurun_out/sweep_c3_mma.jsonl gpurun_out/sweep_c4.jsonl; do echo $f; cut -c 1-700 $f; done; tail -3 gpurun_out/sweep_c3_mma.err
