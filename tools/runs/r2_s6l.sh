# cfg5 K4 mode A/B after the round-2 K4 changes: cluster (default) vs piece mode (global merges) at 1 and 2 CTAs/SM
mkdir -p gpurun_out/s6l
run() { name=$1; shift; env "$@" timeout 300 python bench.py --config cfg5 --steps 30 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6l/$name.json 2> gpurun_out/s6l/$name.err; python -c "
import json
d=json.loads(open('gpurun_out/s6l/$name.json').read().strip().splitlines()[-1])
print('$name', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
run cluster CHESS_X=0
run piece_cps1 CHESS_ATTN_CLUSTER=0
run piece_cps2 CHESS_ATTN_CLUSTER=0 CHESS_ATTN_CPS=2
run piece_cps1_pf8 CHESS_ATTN_CLUSTER=0 CHESS_ATTN_NEXTPF=8
run cluster2 CHESS_X=0
