mkdir -p gpurun_out/s3t
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_small -s 20 -c 1 -o gpurun_out/s3t/prof_small python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/s3t/ncu.log 2>&1; echo rc=$?; tail -2 gpurun_out/s3t/ncu.log
