# tensor-core scan v2 (rows as N): parity, probe, bench
mkdir -p gpurun_out/s3l
timeout 900 python -m pytest tests/test_gpu_select_tc.py tests/test_gpu_engine_oracle.py -x -q -k "tc or f16tc" > gpurun_out/s3l/pytest_tc.log 2>&1; echo "tc tests rc=$?"; tail -3 gpurun_out/s3l/pytest_tc.log
timeout 600 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s3l/probe.json 2> gpurun_out/s3l/probe.err; echo probe rc=$?; head -c 300 gpurun_out/s3l/probe.json; echo
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3l/bench.json 2> gpurun_out/s3l/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s3l/bench.err
python -c "
import json
d=json.loads(open('gpurun_out/s3l/bench.json').read().strip().splitlines()[-1])
print(round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', d['select_roofline'])
"
