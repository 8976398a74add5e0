cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 ${BARGS} > gpurun_out/bench2.log 2> gpurun_out/bench2.err; echo "bench rc $?"
tail -5 gpurun_out/bench2.err
timeout 600 python bench.py --partitioned --steps 3 --warmup 3 > gpurun_out/bench_part.log 2> gpurun_out/bench_part.err; echo "bench part rc $?"
tail -3 gpurun_out/bench_part.err; cut -c1-600 gpurun_out/bench_part.log
