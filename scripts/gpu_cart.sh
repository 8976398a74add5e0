# Cartesian element-matrix vmult: parity (operator, multigrid, slab tests) and
# the per-config sweep with both kernels (STMG_VMULT=quad = quadrature form)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_operator.py tests/test_gpu_multigrid.py tests/test_gpu_slab.py tests/test_gpu_wide.py -m gpu -x -q -rf --timeout 600 -k "not full_size" > gpurun_out/pytest_cart.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_cart.log
tail -3 gpurun_out/pytest_cart.log
timeout 900 python scripts/sweep.py ${SWEEP:-C3 C4 C5-128} > gpurun_out/sweep_cart.jsonl 2> gpurun_out/sweep_cart.err; echo "sweep rc $?"
STMG_VMULT=quad timeout 900 python scripts/sweep.py ${SWEEP:-C3 C4 C5-128} > gpurun_out/sweep_quad.jsonl 2> gpurun_out/sweep_quad.err; echo "sweep quad rc $?"
cat gpurun_out/sweep_cart.jsonl gpurun_out/sweep_quad.jsonl | cut -c1-400; tail -3 gpurun_out/sweep_cart.err
