# session 3 first GPU call: whole GPU suite, tensor-core scan parity, cfg3 bench f32 vs f16tc
mkdir -p gpurun_out/s3a
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3a/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -8 gpurun_out/s3a/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s3a/bench_f32.json 2> gpurun_out/s3a/bench_f32.err; echo "bench f32 rc=$?"; tail -3 gpurun_out/s3a/bench_f32.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --summary-dtype f16tc > gpurun_out/s3a/bench_f16tc.json 2> gpurun_out/s3a/bench_f16tc.err; echo "bench f16tc rc=$?"; tail -3 gpurun_out/s3a/bench_f16tc.err
for f in f32 f16tc; do python -c "
import json,sys
d=json.loads(open('gpurun_out/s3a/bench_$f.json').read().strip().splitlines()[-1])
print('$f', d['us_per_step'], d['select_roofline'], d['roofline']['launch_us'], d['variants'])
" 2>&1 | tail -3; done
timeout 600 python tools/select_tc_probe.py --dtypes f32 f16tc > gpurun_out/s3a/probe.json 2> gpurun_out/s3a/probe.err; echo probe rc=$?; cat gpurun_out/s3a/probe.json; tail -3 gpurun_out/s3a/probe.err
