# K4 cluster cap 8 (compile-time inbox for 7 peers) at b=1 (cfg1, cfg2) vs the default cap 4
mkdir -p gpurun_out/s6r
L8=$PWD/paper_2602_20732_b200/libchess_b200_cl8.so
for cfg in cfg2 cfg1; do
  timeout 300 python bench.py --config $cfg --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6r/${cfg}_cl4.json 2>/dev/null
  CHESS_B200_LIB=$L8 timeout 300 python bench.py --config $cfg --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6r/${cfg}_cl8.json 2>gpurun_out/s6r/${cfg}_cl8.err
  CHESS_B200_LIB=$L8 CHESS_ATTN_CLMAX=4 timeout 300 python bench.py --config $cfg --steps 60 --warmup 5 --headline-only --no-cpu-baseline > gpurun_out/s6r/${cfg}_cl8lib_cap4.json 2>/dev/null
  for v in cl4 cl8 cl8lib_cap4; do python -c "
import json
d=json.loads(open('gpurun_out/s6r/${cfg}_$v.json').read().strip().splitlines()[-1])
print('$cfg $v', round(d['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))" 2>&1 | tail -1; done
done
CHESS_B200_LIB=$L8 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "attention or attn or decode" > gpurun_out/s6r/pytest_cl8.log 2>&1; echo "pytest cl8 rc=$?"; tail -n 1 gpurun_out/s6r/pytest_cl8.log
