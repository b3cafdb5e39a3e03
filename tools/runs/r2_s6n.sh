mkdir -p gpurun_out/s6n
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6n/probe_trace.json 2> gpurun_out/s6n/probe_trace.err; echo trace rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s6n/probe_trace.json').read().strip().splitlines()[-1])
for k,v in d['trace'].items(): print(k, 'won', v.get('rescore_tail_won'), 'phases', v.get('rescore_tail_phases_us'), 'finish', v.get('rescore_finish_us'), 'end', v.get('rescore_tail_end'))
"
