# Cartesian vmult: ncu full capture (C3, C5-128) and the C5 sweeps, one process per config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for W in ${PROF_W:-C3 C5-128}; do
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_cart_kernel" -c 1 -o gpurun_out/prof_cart_$W python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_cart_$W.log 2>&1
echo "ncu $W rc $?"
done
for W in ${SWEEP:-C5-128 C5-256v}; do
timeout 900 python scripts/sweep.py $W >> gpurun_out/sweep_c5.jsonl 2>> gpurun_out/sweep_c5.err; echo "sweep $W rc $?"
done
if [ -n "$LAUNCH_W" ]; then
python scripts/prof_kernels.py step $LAUNCH_W > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$LAUNCH_W.csv python scripts/prof_kernels.py step $LAUNCH_W > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$LAUNCH_W.csv | head -25
fi
cut -c1-300 gpurun_out/sweep_c5.jsonl; tail -3 gpurun_out/sweep_c5.err
