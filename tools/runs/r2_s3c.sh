# tensor-core scan ring-granularity sweep (stage K blocks / TMEM windows), probe at cfg3
mkdir -p gpurun_out/s3c
for v in default kb2 kb2a16 kb1a16; do
  if [ $v = default ]; then lib=paper_2602_20732_b200/libchess_b200.so; else lib=paper_2602_20732_b200/libchess_b200_$v.so; fi
  CHESS_B200_LIB=$PWD/$lib timeout 300 python tools/select_tc_probe.py --dtypes f16tc --reps 10 > gpurun_out/s3c/probe_$v.json 2> gpurun_out/s3c/probe_$v.err
  echo "$v rc=$? $(head -c 200 gpurun_out/s3c/probe_$v.json)"
done
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_kb1a16.so timeout 600 python -m pytest tests/test_gpu_select_tc.py -x -q > gpurun_out/s3c/tc_tests_kb1.log 2>&1; echo "kb1 tc tests rc=$?"; tail -2 gpurun_out/s3c/tc_tests_kb1.log
