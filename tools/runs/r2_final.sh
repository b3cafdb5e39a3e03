# round-2 evidence: default bench (driver flags and 200 steps), launch list of the default bench, ncu of K4 + the page-level tc scan at the bench state
mkdir -p gpurun_out/final
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_cfg3_s20_w5.json 2> gpurun_out/final/bench_s20.err; echo "bench s20 rc=$?"
timeout 900 python bench.py > gpurun_out/final/bench_cfg3_default.json 2> gpurun_out/final/bench_default.err; echo "bench default rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 400 --csv --log-file gpurun_out/final/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > /dev/null 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/final/launches_cfg3.csv "python bench.py --steps 3 --warmup 3 --headline-only (launches 5000..5400)" > gpurun_out/final/launch_summary_cfg3.txt 2>&1; head -25 gpurun_out/final/launch_summary_cfg3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_decode_kernel -s 200 -c 1 -o gpurun_out/final/prof_k4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > /dev/null 2>&1; echo "ncu k4 rc=$?"
for f in s20_w5 default; do python -c "
import json
d=json.loads(open('gpurun_out/final/bench_cfg3_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['us_per_step'],1), d['e2e']['value'], round(d['roofline']['launch_us'],2), round(d['roofline']['frac'],3), round(d['step_roofline']['frac'],3), d['clocks'], d['variants']['dynamic']['us_per_step'] if 'variants' in d else '')"; done
