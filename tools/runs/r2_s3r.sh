# fused rescoring: parity (tc tests, engine-vs-oracle f16tc, pagesel/acceptance), probe, bench A/B
mkdir -p gpurun_out/s3r
timeout 1200 python -m pytest tests/test_gpu_select_tc.py tests/test_gpu_engine_oracle.py -x -q -k "tc or f16tc" > gpurun_out/s3r/pytest_tc.log 2>&1; echo "tc tests rc=$?"; tail -2 gpurun_out/s3r/pytest_tc.log
timeout 600 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s3r/probe.json 2> gpurun_out/s3r/probe.err; echo probe rc=$?; head -c 250 gpurun_out/s3r/probe.json; echo; tail -2 gpurun_out/s3r/probe.err
CHESS_TC_FUSE=0 timeout 600 python tools/select_tc_probe.py --dtypes f16tc > gpurun_out/s3r/probe_nofuse.json 2>/dev/null; head -c 120 gpurun_out/s3r/probe_nofuse.json; echo
for f in 1 0; do CHESS_TC_FUSE=$f timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3r/bench_fuse$f.json 2>gpurun_out/s3r/bench_fuse$f.err; python -c "
import json
d=json.loads(open('gpurun_out/s3r/bench_fuse$f.json').read().strip().splitlines()[-1])
print('fuse $f', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'sel', round(d['select_roofline']['call_us'],1))"; done
