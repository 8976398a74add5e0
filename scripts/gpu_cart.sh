# Cartesian element-matrix vmult: parity (PYTEST_FILES) and the per-config
# sweep, one process per config (SWEEP); QUAD=1 also sweeps STMG_VMULT=quad
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest ${PYTEST_FILES:-tests/test_gpu_operator.py tests/test_gpu_multigrid.py tests/test_gpu_slab.py tests/test_gpu_wide.py} -m gpu -x -q -rf --timeout 600 -k "not full_size" > gpurun_out/pytest_cart.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_cart.log
tail -3 gpurun_out/pytest_cart.log
rm -f gpurun_out/sweep_cart.jsonl gpurun_out/sweep_quad.jsonl
for W in ${SWEEP:-C3 C4 C5-128}; do
timeout 900 python scripts/sweep.py $W >> gpurun_out/sweep_cart.jsonl 2>> gpurun_out/sweep_cart.err; echo "sweep $W rc $?"
if [ -n "$QUAD" ]; then STMG_VMULT=quad timeout 900 python scripts/sweep.py $W >> gpurun_out/sweep_quad.jsonl 2>> gpurun_out/sweep_quad.err; fi
done
cat gpurun_out/sweep_cart.jsonl | cut -c1-330; tail -3 gpurun_out/sweep_cart.err
if [ -n "$PROF_W" ]; then
for W in $PROF_W; do
python scripts/prof_kernels.py kernels $W > gpurun_out/prof_plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_cart_kernel" -c 1 -o gpurun_out/prof_cart_$W python scripts/prof_kernels.py kernels $W > gpurun_out/ncu_cart_$W.log 2>&1
echo "ncu $W rc $?"
done
fi
