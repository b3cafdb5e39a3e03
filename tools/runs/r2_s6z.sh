# session-6 final: GPU suite, smoke, default + driver-flag bench, every config, launch list, ncu of the tc scan levels (after the small-cascade and entropy changes)
mkdir -p gpurun_out/s6z/allcfg
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6z/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/s6z/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6z/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/s6z/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s6z/bench_cfg3_s20_w5.json 2> gpurun_out/s6z/bench_s20.err; echo "bench s20 rc=$?"
timeout 900 python bench.py > gpurun_out/s6z/bench_cfg3_default.json 2> gpurun_out/s6z/bench_default.err; echo "bench default rc=$?"
for cfg in cfg1 cfg2 cfg4 cfg5; do
  timeout 900 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s6z/allcfg/bench_$cfg.json 2> gpurun_out/s6z/allcfg/bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 400 --csv --log-file gpurun_out/s6z/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > /dev/null 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/s6z/launches_cfg3.csv "python bench.py --steps 3 --warmup 3 --headline-only (launches 5000..5400)" > gpurun_out/s6z/launch_summary_cfg3.txt 2>&1; head -14 gpurun_out/s6z/launch_summary_cfg3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_tc_kernel -s 5 -c 3 -o gpurun_out/s6z/prof_tc python tools/select_tc_probe.py --dtypes f16tc --reps 1 > /dev/null 2>&1; echo "ncu tc rc=$?"
for f in gpurun_out/s6z/bench_cfg3_*.json gpurun_out/s6z/allcfg/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']; v=d.get('variants',{})
print('$f', round(d['us_per_step'],1), 'tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'K4', round(r['launch_us'],2), round(r['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1), round(d['select_roofline']['frac'],3), 'dyn', round(v.get('dynamic',{}).get('us_per_step',0),1), d['clocks'])
"; done
