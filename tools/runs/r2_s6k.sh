mkdir -p gpurun_out/s6k
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_oracle.py tests/test_gpu_engine.py -m gpu -q -x > gpurun_out/s6k/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s6k/pytest.log
timeout 300 python bench.py --config cfg1 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s6k/bench_cfg1.json 2> gpurun_out/s6k/bench_cfg1.err; echo rc=$?
timeout 300 python bench.py --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6k/bench_cfg3.json 2> gpurun_out/s6k/bench_cfg3.err; echo rc=$?
timeout 300 python tools/step_timeline.py --config cfg1 --summary-dtype f32 --steps 2 > gpurun_out/s6k/cfg1_timeline.txt 2>&1
grep -A8 "# step 1" gpurun_out/s6k/cfg1_timeline.txt
python -c "
import json
d=json.loads(open('gpurun_out/s6k/bench_cfg1.json').read().strip().splitlines()[-1]); print('cfg1', round(d['us_per_step'],1), d['select_roofline']['call_us'], d['variants']['dynamic']['us_per_step'])
d=json.loads(open('gpurun_out/s6k/bench_cfg3.json').read().strip().splitlines()[-1]); print('cfg3', round(d['us_per_step'],1))
"
