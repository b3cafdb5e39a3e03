# every config with the round-2 defaults (40 steps; variants included)
mkdir -p gpurun_out/allcfg
for cfg in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/allcfg/bench_$cfg.json 2> gpurun_out/allcfg/bench_$cfg.err
  python -c "
import json
d=json.loads(open('gpurun_out/allcfg/bench_$cfg.json').read().strip().splitlines()[-1])
v=d.get('variants',{})
print('$cfg', d['details']['summary_dtype'], round(d['us_per_step'],1), 'tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'K4', round(d['roofline']['launch_us'],2), round(d['roofline']['frac'],3), 'step frac', round(d['step_roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1), 'dyn', round(v.get('dynamic',{}).get('us_per_step',0),1))"
done
