# closing check after the cluster-cap knob (k_attn.cu rebuilt, default unchanged)
mkdir -p gpurun_out/s6t
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s6t/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/s6t/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6t/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/s6t/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s6t/bench_cfg3_s20_w5.json 2> gpurun_out/s6t/bench_s20.err; echo "bench s20 rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/s6t/bench_cfg3_s20_w5.json').read().strip().splitlines()[-1])
print(round(d['us_per_step'],1), round(d['value']), round(d['e2e']['value']), round(d['roofline']['launch_us'],2), d['clocks'])"
