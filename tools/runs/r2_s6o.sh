# does the entropy kernel's grid delay the first decode layer in the two-stream step? (cfg2 / cfg3 timelines + bench)
mkdir -p gpurun_out/s6o
for sp in 0 4 16; do
  CHESS_ENT_SPLITS=$sp timeout 300 python tools/step_timeline.py --config cfg2 --summary-dtype f32 --steps 2 > gpurun_out/s6o/cfg2_sp$sp.txt 2>&1
  echo "== cfg2 splits=$sp"; awk '/# step 1/{f=1} f' gpurun_out/s6o/cfg2_sp$sp.txt | head -6
  CHESS_ENT_SPLITS=$sp timeout 300 python bench.py --config cfg2 --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6o/bench_cfg2_sp$sp.json 2>/dev/null
  CHESS_ENT_SPLITS=$sp timeout 300 python bench.py --steps 40 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6o/bench_cfg3_sp$sp.json 2>/dev/null
  python -c "
import json
for c in ('cfg2','cfg3'):
    d=json.loads(open('gpurun_out/s6o/bench_'+c+'_sp$sp.json').read().strip().splitlines()[-1]); print(c, 'splits $sp', round(d['us_per_step'],1))
"
done
