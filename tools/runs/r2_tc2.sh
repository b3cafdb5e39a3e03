mkdir -p gpurun_out/r2tc2
timeout 600 python tools/select_tc_probe.py --dtypes f32 f16tc > gpurun_out/r2tc2/probe.json 2> gpurun_out/r2tc2/probe.err; echo rc=$?; cat gpurun_out/r2tc2/probe.json; tail -3 gpurun_out/r2tc2/probe.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|anchor|scan" -c 40 --csv --log-file gpurun_out/r2tc2/launches_f16tc.csv python tools/select_tc_probe.py --dtypes f16tc --reps 1 > /dev/null 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/r2tc2/launches_f16tc.csv 2>&1 | tail -30
python - <<'PY'
import csv, re
rows=[r for r in csv.reader(open('gpurun_out/r2tc2/launches_f16tc.csv')) if r]
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:h+1+40]:
    print(re.sub(r'\(.*','',r[ki]).replace('(anonymous namespace)::','')[:60], r[vi])
PY
