# K4 tail stealing: parity (forced), stress, bench sweep
mkdir -p gpurun_out/s4a
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode or attention_paths" > gpurun_out/s4a/pytest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s4a/pytest.log
CHESS_ATTN_STEAL=8 timeout 300 python tools/stress_tc_attn.py 100 2>&1 | tail -1
for st in 0 4 8 12; do CHESS_ATTN_STEAL=$st timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s4a/bench_steal$st.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s4a/bench_steal$st.json').read().strip().splitlines()[-1])
print('steal $st', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
