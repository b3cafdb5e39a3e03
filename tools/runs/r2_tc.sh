# tensor-core selection: parity tests, then the cfg3 bench with f16tc summaries
mkdir -p gpurun_out/r2tc
timeout 900 python -m pytest tests/test_gpu_select_tc.py -x -q -s > gpurun_out/r2tc/pytest_tc.log 2>&1; echo "tc tests rc=$?"; tail -15 gpurun_out/r2tc/pytest_tc.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --summary-dtype f16tc > gpurun_out/r2tc/bench_f16tc.json 2> gpurun_out/r2tc/bench_f16tc.err; echo "bench rc=$?"; tail -3 gpurun_out/r2tc/bench_f16tc.err
python -c "
import json
d=json.loads(open('gpurun_out/r2tc/bench_f16tc.json').read().strip().splitlines()[-1])
print(d['us_per_step'], d['select_roofline'], d['roofline']['launch_us'], d['variants']['select_every_step'])
" 2>&1 | tail -3
