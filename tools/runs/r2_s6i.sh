mkdir -p gpurun_out/s6i
CHESS_B200_LIB=$PWD/paper_2602_20732_b200/libchess_b200_trace.so timeout 300 python tools/select_micro.py --batch 1 --pages 256 --dim 1024 > gpurun_out/s6i/small_trace.json 2>&1; echo rc=$?
timeout 300 python tools/select_micro.py --batch 1 --pages 256 --dim 1024 > gpurun_out/s6i/small_prod.json 2>&1; echo rc=$?
tail -n 1 gpurun_out/s6i/small_trace.json; tail -n 1 gpurun_out/s6i/small_prod.json | cut -c1-200
