mkdir -p gpurun_out/r2d
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d/bench_20_5.json 2> gpurun_out/r2d/bench_20_5.err; echo rc=$?
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2d/bench_200_10.json 2> gpurun_out/r2d/bench_200_10.err; echo rc=$?
tail -3 gpurun_out/r2d/bench_20_5.err
for f in gpurun_out/r2d/bench_*.json; do python -c "
import sys,json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']; print('$f', round(d['us_per_step'],1), round(r['launch_us'],2), round(r['frac'],3), r['tiles_per_launch'], r['unique_tiles_per_launch'], round(d['details']['ws_pages_mean'],2), round(d['select_roofline']['call_us'],1), json.dumps(d.get('variants')))
"; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2d/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2d/pytest.log
