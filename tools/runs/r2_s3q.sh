# selection grid size A/B in the concurrent step (f16tc)
mkdir -p gpurun_out/s3q
for g in 148 120 96 74; do CHESS_SELECT_GRID=$g timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3q/bench_g$g.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s3q/bench_g$g.json').read().strip().splitlines()[-1])
print('grid $g', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1))"; done
