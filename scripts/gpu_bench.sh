cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.log
tail -c 4000 gpurun_out/bench.log; tail -20 gpurun_out/bench.err
