mkdir -p gpurun_out/s6m
timeout 900 python -m pytest tests/test_gpu_select_tc.py tests/test_gpu_engine_oracle.py -m gpu -q -x > gpurun_out/s6m/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s6m/pytest.log
timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6m/probe_prod.json 2> gpurun_out/s6m/probe_prod.err; echo probe rc=$?
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s6m/probe_trace.json 2> gpurun_out/s6m/probe_trace.err; echo trace rc=$?
timeout 300 python bench.py --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6m/bench_cfg3.json 2> gpurun_out/s6m/bench_cfg3.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s6m/probe_prod.json').read().strip().splitlines()[-1]); print('prod us', d['us_per_pass'], d['rescored_rows_per_pass'])
d=json.loads(open('gpurun_out/s6m/probe_trace.json').read().strip().splitlines()[-1])
print('trace us', d['us_per_pass'])
for k,v in d['trace'].items(): print(k, 'tail', v['tail_us'], v['tail_phases_us'], 'resc', v.get('rescore_entry'), v.get('rescore_tail_won'), v.get('rescore_tail_end'))
d=json.loads(open('gpurun_out/s6m/bench_cfg3.json').read().strip().splitlines()[-1])
print('bench', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1), round(d['select_roofline']['frac'],3))
"
