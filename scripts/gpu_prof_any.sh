# ncu full capture of kernels matching KREGEX in `prof_kernels.py kernels W`
# (one launch each), plus the launch list of a bench step (LAUNCH_W)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for W in ${PROF_W:-C5-128}; do
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"${KREGEX:-fdm_lines}" -c ${NCU_C:-1} -o gpurun_out/prof_${TAG:-k}_$W python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_${TAG:-k}_$W.log 2>&1
echo "ncu $W rc $?"
done
if [ -n "$LAUNCH_W" ]; then
python scripts/prof_kernels.py step $LAUNCH_W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$LAUNCH_W.csv python scripts/prof_kernels.py step $LAUNCH_W > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$LAUNCH_W.csv | head -25
fi
