# session-6 closing check on the committed tree: GPU suite, smoke, bench at the driver's flags and default
mkdir -p gpurun_out/s6q
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6q/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s6q/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6q/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/s6q/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s6q/bench_cfg3_s20_w5.json 2> gpurun_out/s6q/bench_s20.err; echo "bench s20 rc=$?"
timeout 900 python bench.py > gpurun_out/s6q/bench_cfg3_default.json 2> gpurun_out/s6q/bench_default.err; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s6q/bench_reference.json 2> gpurun_out/s6q/bench_reference.err; echo "reference rc=$?"
for f in gpurun_out/s6q/bench_cfg3_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']
print('$f', round(d['us_per_step'],1), 'tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'K4', round(r['launch_us'],2), round(r['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1), d['scaling'], d['gpu_launches'], d['clocks'])
"; done
tail -c 400 gpurun_out/s6q/bench_reference.json
