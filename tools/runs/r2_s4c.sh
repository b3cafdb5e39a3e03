mkdir -p gpurun_out/s4c
for cfg in "0 0" "8 0" "8 6000" "8 9000" "16 6000"; do set -- $cfg; CHESS_ATTN_HELPER=$1 CHESS_ATTN_HELPER_NS=$2 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s4c/b.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s4c/b.json').read().strip().splitlines()[-1])
print('helper $1 delay $2', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
