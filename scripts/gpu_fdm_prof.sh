cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/fdm_launches.csv python scripts/prof_kernels.py kernels C5-128 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/fdm_launches.csv | head -12
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:fdm_strip_kernel -c 1 -f -o gpurun_out/prof_fdm_strip python scripts/prof_kernels.py kernels C5-128 > gpurun_out/ncu_fdm_strip.log 2>&1; echo "ncu rc $?"
