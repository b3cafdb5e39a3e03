set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm --format=csv
mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2a/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a/bench_20_5.json 2> gpurun_out/r2a/bench_20_5.err; echo rc=$?
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2a/bench_200_10.json 2> gpurun_out/r2a/bench_200_10.err; echo rc=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a/bench_20_5b.json 2>&1; echo rc=$?
cat gpurun_out/r2a/*.json | python -c "
import sys,json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['us_per_step'], d['roofline']['launch_us'], d['roofline']['bytes_per_launch'], d['details']['kv_pool_pages'], d['details']['ws_pages_mean'], d['select_roofline']['call_us'])
"
