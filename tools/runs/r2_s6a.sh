# session-6 start: fresh container rebuild -> GPU suite + default bench (driver flags) + cfg2/cfg5
mkdir -p gpurun_out/s6a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6a/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/s6a/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/s6a/bench_cfg3_20_5.json 2> gpurun_out/s6a/bench_cfg3.err; echo rc=$?
for cfg in cfg2 cfg5; do
timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s6a/bench_$cfg.json 2> gpurun_out/s6a/bench_$cfg.err; echo $cfg rc=$?
done
for f in gpurun_out/s6a/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']; print('$f', round(d['us_per_step'],1), 'K4', round(r['launch_us'],2), round(r['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1), round(d['select_roofline']['frac'],3), 'e2e', round(d['e2e']['value']))
"; done
