# selection grid in the concurrent cfg3 step (f16tc): 3 runs each, interleaved
mkdir -p gpurun_out/s3x
for rep in 1 2; do for g in 112 104 96 88 72 64; do
  CHESS_SELECT_GRID=$g timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3x/bench_g${g}_r$rep.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/s3x/bench_g${g}_r$rep.json').read().strip().splitlines()[-1])
print('rep $rep grid $g', round(d['us_per_step'],1))"
done; done
