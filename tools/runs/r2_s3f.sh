# ncu full capture of one tensor-core K4 launch and one mma.sync K4 launch at cfg3 (bench state)
mkdir -p gpurun_out/s3f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_decode_tc_kernel -s 200 -c 1 -o gpurun_out/s3f/prof_k4tc python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/s3f/ncu1.log 2>&1; echo ncu1 rc=$?; tail -2 gpurun_out/s3f/ncu1.log
CHESS_ATTN_TC=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_decode_kernel -s 200 -c 1 -o gpurun_out/s3f/prof_k4mma python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/s3f/ncu2.log 2>&1; echo ncu2 rc=$?; tail -2 gpurun_out/s3f/ncu2.log
