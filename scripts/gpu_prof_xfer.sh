cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:xyz_restrict_kernel -c 1 -f -o gpurun_out/prof_restrict python scripts/prof_kernels.py step C5-128 > gpurun_out/ncu_r.log 2>&1; echo "rc $?"
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:xyz_prolong_kernel -s 1 -c 1 -f -o gpurun_out/prof_prolong python scripts/prof_kernels.py step C5-128 > gpurun_out/ncu_p.log 2>&1; echo "rc $?"
