# new default (tc scan grid 96 when concurrent) at cfg3 + f32 scan grid sweep at cfg4 / cfg5
mkdir -p gpurun_out/s3y
for rep in 1 2; do timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3y/bench_cfg3_default_r$rep.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s3y/bench_cfg3_default_r$rep.json').read().strip().splitlines()[-1])
print('cfg3 default rep $rep', round(d['us_per_step'],1))"; done
for cfg in cfg4 cfg5 cfg2; do for g in 148 120 96; do
  CHESS_SELECT_GRID=$g timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3y/bench_${cfg}_g$g.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/s3y/bench_${cfg}_g$g.json').read().strip().splitlines()[-1])
print('$cfg f32 grid $g', round(d['us_per_step'],1))"
done; done
