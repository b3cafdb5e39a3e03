mkdir -p gpurun_out/s3m
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_tc_kernel -c 3 -o gpurun_out/s3m/prof_tc2 python tools/select_tc_probe.py --dtypes f16tc --reps 1 > gpurun_out/s3m/ncu.log 2>&1; echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|anchor|scan" -c 14 --csv --log-file gpurun_out/s3m/launches.csv python tools/select_tc_probe.py --dtypes f16tc --reps 1 > /dev/null 2>&1; echo ncu2 rc=$?
python - <<'PY'
import csv, re
rows=[r for r in csv.reader(open('gpurun_out/s3m/launches.csv')) if r]
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:]:
    print(re.sub(r'\(.*','',r[ki]).replace('(anonymous namespace)::','')[:60], r[vi])
PY
