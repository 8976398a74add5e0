cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/k_launches.csv python scripts/prof_kernels.py ${MODE:-kernels} ${W:-C5-128} > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/k_launches.csv | head -${HEADN:-12}
