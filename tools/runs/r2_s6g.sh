# env-only A/Bs at cfg3: forced stream-K K4 at 1 vs 2 CTAs per SM; selection grid next to the decode after the tail rewrite
mkdir -p gpurun_out/s6g
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6g/$name.json 2> gpurun_out/s6g/$name.err; python -c "
import json
d=json.loads(open('gpurun_out/s6g/$name.json').read().strip().splitlines()[-1])
print('$name', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1))"; }
run base CHESS_X=0
run streamk_cps1 CHESS_ATTN_MODE=7 CHESS_ATTN_CPS=1
run streamk_cps2 CHESS_ATTN_MODE=7 CHESS_ATTN_CPS=2
run selgrid72 CHESS_SELECT_GRID=72
run selgrid120 CHESS_SELECT_GRID=120
run base2 CHESS_X=0
