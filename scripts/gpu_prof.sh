cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
python scripts/prof_kernels.py step $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch.log 2>&1
echo "launches rc $?"
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_apply_kernel|asm_apply_kernel" -c 2 -o gpurun_out/prof_full python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_full.log 2>&1
echo "full rc $?"
tail -5 gpurun_out/ncu_full.log
