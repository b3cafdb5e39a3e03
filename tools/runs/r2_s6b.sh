# tc selection tail breakdown (trace build) + timing after batching the tail's partial loads
mkdir -p gpurun_out/s6b
timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6b/probe_prod.json 2> gpurun_out/s6b/probe_prod.err; echo probe rc=$?
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6b/probe_trace.json 2> gpurun_out/s6b/probe_trace.err; echo trace rc=$?
timeout 300 python bench.py --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6b/bench_cfg3.json 2> gpurun_out/s6b/bench_cfg3.err; echo bench rc=$?
CHESS_ATTN_MODE=7 timeout 300 python bench.py --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6b/bench_cfg3_streamk.json 2> gpurun_out/s6b/bench_cfg3_streamk.err; echo streamk rc=$?
cat gpurun_out/s6b/probe_prod.json
python -c "
import json
d=json.loads(open('gpurun_out/s6b/probe_trace.json').read().strip().splitlines()[-1])
print('trace us', d['us_per_pass'])
for k,v in d['trace'].items(): print(k, json.dumps(v))
"
for f in gpurun_out/s6b/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']; print('$f', round(d['us_per_step'],1), 'K4', round(r['launch_us'],2), round(r['frac'],3), 'sel', round(d['select_roofline']['call_us'],1))
"; done
