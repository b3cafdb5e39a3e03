mkdir -p gpurun_out/s3h
for tc in 1 0; do CHESS_ATTN_TC=$tc timeout 300 python tools/attn_micro.py --batch 16 --ws 46 --pool-gib 40 > gpurun_out/s3h/micro_tc$tc.json 2>&1; echo "tc=$tc rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/s3h/micro_tc$tc.json').read().strip().splitlines()[-1])
print({k:(round(v['us'],2), round(v['graph_us'],2)) for k,v in d.items() if isinstance(v,dict)})"; done
