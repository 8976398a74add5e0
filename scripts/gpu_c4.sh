# exact-cell tensor-core smoothers (27 / 125 dofs): parity tests, C4 default vs STMG_ASM125=dfma, launch list, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multigrid.py tests/test_gpu_slab.py -m gpu -q -rf --timeout 600 -k "asm or vcycle or gmres or smoother" > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_c4.log
timeout 900 python scripts/sweep.py C4n > gpurun_out/sweep_c4_mma.jsonl 2> gpurun_out/sweep_c4_mma.err
STMG_ASM125=dfma timeout 900 python scripts/sweep.py C4n > gpurun_out/sweep_c4_dfma.jsonl 2> gpurun_out/sweep_c4_dfma.err
python scripts/prof_kernels.py step C4 > gpurun_out/prof_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c4.csv python scripts/prof_kernels.py step C4 > gpurun_out/ncu_launch_c4.log 2>&1
echo "launches rc $?" >> gpurun_out/pytest_c4.log
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply_large_mma" -c 1 -o gpurun_out/prof_large_mma python scripts/prof_kernels.py kernels C4 > gpurun_out/ncu_large.log 2>&1
echo "full rc $?" >> gpurun_out/pytest_c4.log
tail -5 gpurun_out/pytest_c4.log; cat gpurun_out/sweep_c4_mma.jsonl gpurun_out/sweep_c4_dfma.jsonl | cut -c 1-600; tail -3 gpurun_out/sweep_c4_mma.err
