# tensor-core selection profile: launch list + full capture of the three select_tc_kernel launches
mkdir -p gpurun_out/s3b
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3b/launches_f16tc.csv python tools/select_tc_probe.py --dtypes f16tc --reps 1 > /dev/null 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/s3b/launches_f16tc.csv 2>&1 | tail -20
python - <<'PY'
import csv, re
rows=[r for r in csv.reader(open('gpurun_out/s3b/launches_f16tc.csv')) if r]
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
ki,vi=H.index('Kernel Name'),H.index('Metric Value')
for r in rows[h+1:h+1+60]:
    print(re.sub(r'\(.*','',r[ki]).replace('(anonymous namespace)::','')[:60], r[vi])
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_tc_kernel -c 3 -o gpurun_out/s3b/prof_tc python tools/select_tc_probe.py --dtypes f16tc --reps 1 > gpurun_out/s3b/ncu_full.log 2>&1; echo ncu2 rc=$?; tail -3 gpurun_out/s3b/ncu_full.log
