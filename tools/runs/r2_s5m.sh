mkdir -p gpurun_out/s5m
for c in cfg2 cfg5; do
timeout 300 python tools/step_timeline.py --config $c --policy every_step --steps 3 > gpurun_out/s5m/$c.txt 2>&1; echo $c; sed -n '/# step 2/,+12p' gpurun_out/s5m/$c.txt; tail -1 gpurun_out/s5m/$c.txt
timeout 300 python tools/step_timeline.py --config $c --policy every_step --steps 3 --sequential > gpurun_out/s5m/${c}_seq.txt 2>&1; echo $c seq; sed -n '/# step 2/,+4p' gpurun_out/s5m/${c}_seq.txt; tail -1 gpurun_out/s5m/${c}_seq.txt
done
