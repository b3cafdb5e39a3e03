# K4 per-layer timeline at batch 1 (cfg2 shape) on the trace build
mkdir -p gpurun_out/s6s
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/attn_micro.py --batch 1 --ws 16 --pool-gib 8 > gpurun_out/s6s/b1_trace.json 2>&1; echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s6s/b1_trace.json').read().strip().splitlines()[-1])
for k in ('random',):
    v=d[k]; print(k, v['us'], v.get('graph_us'))
    for a,b in v.get('trace_us',{}).items(): print('  ',a,b)
"
