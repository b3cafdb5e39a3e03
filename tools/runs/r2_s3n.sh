# K4 piece-state handoff on mbarriers: parity, racecheck (smoke + stream-K case), cfg3/cfg4 bench
mkdir -p gpurun_out/s3n
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode" > gpurun_out/s3n/pytest_attn.log 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/s3n/pytest_attn.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3n/racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"; tail -3 gpurun_out/s3n/racecheck_smoke.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest -x -q tests/test_gpu_kernels.py -k "sparse_decode_vs_fp64 and (case4 or case3 or case2)" > gpurun_out/s3n/racecheck_attn.log 2>&1; echo "racecheck attn rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed|Error" gpurun_out/s3n/racecheck_attn.log | sort | uniq -c | head
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3n/synccheck_smoke.log 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/s3n/synccheck_smoke.log
for cfg in cfg3 cfg4; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3n/bench_$cfg.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s3n/bench_$cfg.json').read().strip().splitlines()[-1])
print('$cfg', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
