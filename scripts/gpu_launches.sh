cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${W:-C5-128}
python scripts/prof_kernels.py step $W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$W.csv python scripts/prof_kernels.py step $W > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$W.csv | head -30
