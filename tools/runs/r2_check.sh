# Round-2 checkpoint: full GPU suite, then the bench at the driver's K/W and at 200 steps.
mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2c/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r2c/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c/bench_20_5.json 2> gpurun_out/r2c/bench_20_5.err; echo rc=$?
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2c/bench_200_10.json 2> gpurun_out/r2c/bench_200_10.err; echo rc=$?
tail -3 gpurun_out/r2c/bench_20_5.err
for f in gpurun_out/r2c/bench_*.json; do python -c "
import sys,json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']; print('$f', round(d['us_per_step'],1), round(r['launch_us'],2), round(r['frac'],3), r.get('tiles_per_launch'), r.get('unique_tiles_per_launch'), round(d['details']['ws_pages_mean'],2), round(d['select_roofline']['call_us'],1), json.dumps(d.get('variants')))
"; done
