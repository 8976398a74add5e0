cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operator.py -x -q -m gpu -k "brick or config_vmult or every_field or full_size" > gpurun_out/pytest_brick.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_brick.log
timeout 600 python bench.py --workload C5-128 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_c5.log').read().strip().splitlines()[-1]);k=d['kernels']
print('step',d['ms_per_step'],'vmult',k['vmult_ms'],'vcycle',k['vcycle_ms'],'solve',d['solve'])"
