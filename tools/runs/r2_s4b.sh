mkdir -p gpurun_out/s4b
timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention_paths" > gpurun_out/s4b/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s4b/pytest.log
for cfg in "0 2" "4 2" "8 4" "8 8" "16 8"; do set -- $cfg; CHESS_ATTN_STEAL=$1 CHESS_ATTN_STEAL_CHUNK=$2 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/s4b/b.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s4b/b.json').read().strip().splitlines()[-1])
print('steal $1 chunk $2', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
