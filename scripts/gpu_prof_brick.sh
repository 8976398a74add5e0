cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${W:-C5-128}
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"${K:-st_brick_kernel}" -c 1 -o gpurun_out/prof_brick_$W python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_brick.log 2>&1; echo "ncu rc $?"
