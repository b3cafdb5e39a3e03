# tc K4 with separate K / V producer warps: parity, cfg3 bench; M=64 TMEM probe
mkdir -p gpurun_out/s3g
timeout 60 ./tools/tc_attn_probe > gpurun_out/s3g/probe.txt 2>&1; head -3 gpurun_out/s3g/probe.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode or attention_paths" > gpurun_out/s3g/pytest_attn.log 2>&1; echo "attn tests rc=$?"; tail -3 gpurun_out/s3g/pytest_attn.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3g/bench_tc.json 2> gpurun_out/s3g/bench_tc.err; echo "bench tc rc=$?"; tail -3 gpurun_out/s3g/bench_tc.err
python -c "
import json
d=json.loads(open('gpurun_out/s3g/bench_tc.json').read().strip().splitlines()[-1])
print('tc', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'frac', round(d['roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1))
"
