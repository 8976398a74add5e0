# round-2 baseline at HEAD: C5-128 bench line, step launch list, ncu full of the two dominant kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 600 python bench.py --workload C5-128 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "bench rc $?"
python scripts/prof_kernels.py step C5-128 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C5-128.csv python scripts/prof_kernels.py step C5-128 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_C5-128.csv | head -25
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"st_cart_kernel|fdm_lines_kernel" -c 2 -o gpurun_out/prof_c5_base python scripts/prof_kernels.py kernels C5-128 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
