# full GPU suite + smoke after the append/entropy/graph changes
mkdir -p gpurun_out/s5o
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/s5o/pytest_gpu.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s5o/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s5o/bench_s20.json 2>gpurun_out/s5o/bench_s20.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s5o/bench_s20.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['us_per_step'],1), d['e2e']['value'], d['gpu_launches'], d['roofline']['frac'], d['step_roofline']['frac'], d.get('select_marginal'), d['clocks'], d['variants']['dynamic']['us_per_step'])"
