# plain run of the kernel driver, then one ncu --set full capture per hot kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_apply_kernel" -c 1 -o gpurun_out/prof_st python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_st.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"asm_apply" -c 1 -o gpurun_out/prof_asm python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_asm.log 2>&1
echo "prof rc $?"
