# warm-cache serialised launch list of the cfg3 headline step (ncu --cache-control none): per-kernel durations
mkdir -p gpurun_out/s5b
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --cache-control none --clock-control none -s 5000 -c 400 --csv --log-file gpurun_out/s5b/launches_warm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > /dev/null 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/s5b/launches_warm.csv "warm (cache-control none)" > gpurun_out/s5b/summary.txt 2>&1; cat gpurun_out/s5b/summary.txt
