# K4 co-residency A/B: per-CTA smem capped at 112 KB (CHESS_ATTN_SMEM_KB) so layer l+1's CTA fits beside layer l's
mkdir -p gpurun_out/s5a
for lib in "" smem112; do for cfg in cfg3 cfg5 cfg2 cfg4; do
  if [ -n "$lib" ]; then export CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_$lib.so; else unset CHESS_B200_LIB; fi
  timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s5a/b.json 2>gpurun_out/s5a/err_${lib}_$cfg.txt; python -c "
import json
d=json.loads(open('gpurun_out/s5a/b.json').read().strip().splitlines()[-1])
print('lib=${lib:-default} $cfg', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), round(d['roofline']['frac'],3))"; done; done
