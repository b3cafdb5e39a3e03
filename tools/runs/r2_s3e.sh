# tensor-core K4: parity (default + both forced consumers), then cfg3 bench
mkdir -p gpurun_out/s3e
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode or attention_paths" > gpurun_out/s3e/pytest_attn.log 2>&1; echo "attn tests rc=$?"; tail -30 gpurun_out/s3e/pytest_attn.log | grep -v "^$" | tail -25
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3e/bench_tc.json 2> gpurun_out/s3e/bench_tc.err; echo "bench tc rc=$?"; tail -3 gpurun_out/s3e/bench_tc.err
CHESS_ATTN_TC=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s3e/bench_mma.json 2> gpurun_out/s3e/bench_mma.err; echo "bench mma rc=$?"
for f in tc mma; do python -c "
import json
d=json.loads(open('gpurun_out/s3e/bench_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2), 'frac', round(d['roofline']['frac'],3), 'sel', round(d['select_roofline']['call_us'],1))
" 2>&1 | tail -2; done
