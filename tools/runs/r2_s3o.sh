mkdir -p gpurun_out/s3o
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode" > gpurun_out/s3o/pytest_attn.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/s3o/pytest_attn.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3o/racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"; tail -2 gpurun_out/s3o/racecheck_smoke.log; grep -oE "in [a-z_]+\.(cu|cuh):[0-9]+" gpurun_out/s3o/racecheck_smoke.log | sort | uniq -c | sort -rn | head -5
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest -x -q tests/test_gpu_kernels.py -k "sparse_decode_vs_fp64" > gpurun_out/s3o/racecheck_attn.log 2>&1; echo "racecheck attn rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/s3o/racecheck_attn.log | tail -3; grep -oE "in [a-z_]+\.(cu|cuh):[0-9]+" gpurun_out/s3o/racecheck_attn.log | sort | uniq -c | sort -rn | head -5
for cfg in cfg3 cfg4 cfg5; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3o/bench_$cfg.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s3o/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
