mkdir -p gpurun_out/s6e
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6e/probe_trace.json 2> gpurun_out/s6e/probe_trace.err; echo trace rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s6e/probe_trace.json').read().strip().splitlines()[-1])
print('trace us', d['us_per_pass'])
for k,v in d['trace'].items(): print(k, json.dumps({x:y for x,y in v.items() if x.startswith('rescore')}))
"
