# full GPU suite + smoke + default bench + multi-rank launch path on one GPU (plumbing, not a scaling number)
mkdir -p gpurun_out/s3v
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3v/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/s3v/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s3v/bench_default_s20.json 2> gpurun_out/s3v/bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/s3v/bench_default_s20.json').read().strip().splitlines()[-1])
print(d['value'], d['us_per_step'], d['e2e'], d['roofline']['frac'], d['step_roofline']['frac'], d['clocks'])"
CHESS_BENCH_ONE_DEVICE=1 timeout 600 python bench.py --gpus 2 --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/s3v/bench_cfg4_2ranks_one_device.json 2> gpurun_out/s3v/bench_2r.err; echo "2-rank rc=$?"; tail -c 400 gpurun_out/s3v/bench_cfg4_2ranks_one_device.json; tail -3 gpurun_out/s3v/bench_2r.err
