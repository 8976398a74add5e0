cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${W:-C5-128}
python scripts/prof_kernels.py ${PM:-kernels} $W > gpurun_out/prof_plain.log 2>&1 || { echo plain failed; tail -20 gpurun_out/prof_plain.log; exit 1; }
for K in ${KS:-st_brick_kernel fdm_lines_kernel}; do
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$K" -c 1 -f -o gpurun_out/prof_${K}_$W python scripts/prof_kernels.py ${PM:-kernels} $W > gpurun_out/ncu_$K.log 2>&1; echo "ncu $K rc $?"
done
