# K4 consumer A/B per config: mma.sync (CHESS_ATTN_TC=0) vs tcgen05 everywhere (=2)
mkdir -p gpurun_out/s3k
for cfg in cfg3 cfg5 cfg4 cfg2; do for tc in 0 2; do
  CHESS_ATTN_TC=$tc timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3k/bench_${cfg}_tc$tc.json 2> gpurun_out/s3k/bench_${cfg}_tc$tc.err
  python -c "
import json
d=json.loads(open('gpurun_out/s3k/bench_${cfg}_tc$tc.json').read().strip().splitlines()[-1])
print('$cfg tc=$tc', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'frac', round(d['roofline']['frac'],3))
" 2>&1 | tail -1
done; done
