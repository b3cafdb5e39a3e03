mkdir -p gpurun_out/s3u
timeout 1500 python -m pytest tests/test_gpu_select.py tests/test_gpu_pagesel.py tests/test_gpu_engine_oracle.py tests/test_gpu_acceptance.py -x -q > gpurun_out/s3u/pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s3u/pytest.log
for cfg in cfg1; do timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3u/bench_$cfg.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s3u/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1))"; done
