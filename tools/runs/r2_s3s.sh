# summary dtype per config: f32 vs f16tc (headline step, 40 steps)
mkdir -p gpurun_out/s3s
for cfg in cfg1 cfg2 cfg4 cfg5; do for dt in f32 f16tc; do
  timeout 400 python bench.py --config $cfg --summary-dtype $dt --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3s/bench_${cfg}_$dt.json 2> gpurun_out/s3s/bench_${cfg}_$dt.err
  python -c "
import json
d=json.loads(open('gpurun_out/s3s/bench_${cfg}_$dt.json').read().strip().splitlines()[-1])
print('$cfg $dt', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1), 'frac', round(d['step_roofline']['frac'],3))" 2>&1 | tail -1
done; done
