# exact-cell tensor-core smoothers (C3 27-dof, C4 125-dof): step launch lists and one ncu --set full capture each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for W in C3 C4; do
  python scripts/prof_kernels.py step $W > gpurun_out/prof_$W.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$W.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch_$W.log 2>&1
  echo "$W launches rc $?"
done
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply_mma32" -c 1 -o gpurun_out/prof_mma32 python scripts/prof_kernels.py kernels C3 > gpurun_out/ncu_mma32.log 2>&1
echo "mma32 rc $?"
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply_large_mma" -c 1 -o gpurun_out/prof_large_mma python scripts/prof_kernels.py kernels C4 > gpurun_out/ncu_large.log 2>&1
echo "large_mma rc $?"
