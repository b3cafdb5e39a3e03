mkdir -p gpurun_out/xc2
CHESS_ATTN_XC2=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sparse_decode_vs_fp64" > gpurun_out/xc2/pytest.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/xc2/pytest.log
for x in 0 1; do for cfg in cfg3 cfg5; do CHESS_ATTN_XC2=$x timeout 300 python bench.py --config $cfg --steps 60 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/xc2/b.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/xc2/b.json').read().strip().splitlines()[-1])
print('xc2 $x $cfg', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done; done
