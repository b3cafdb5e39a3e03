mkdir -p gpurun_out/s6j
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_acceptance.py tests/test_gpu_engine_oracle.py tests/test_gpu_pagesel.py -m gpu -q -x > gpurun_out/s6j/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/s6j/pytest.log
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_micro.py --batch 1 --pages 256 --dim 1024 > gpurun_out/s6j/small_trace.json 2>&1; echo rc=$?
timeout 300 python tools/select_micro.py --batch 1 --pages 256 --dim 1024 > gpurun_out/s6j/small_prod.json 2>&1; echo rc=$?
timeout 300 python bench.py --config cfg1 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s6j/bench_cfg1.json 2> gpurun_out/s6j/bench_cfg1.err; echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s6j/small_trace.json').read().strip().splitlines()[-1]); print(d['us'], d.get('small_phases_us'), d.get('small_total_us'))
d=json.loads(open('gpurun_out/s6j/small_prod.json').read().strip().splitlines()[-1]); print('prod', d['us'])
d=json.loads(open('gpurun_out/s6j/bench_cfg1.json').read().strip().splitlines()[-1]); print('cfg1', round(d['us_per_step'],1), d['select_roofline']['call_us'], d['variants']['dynamic']['us_per_step'])
"
