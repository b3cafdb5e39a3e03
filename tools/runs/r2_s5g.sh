# append triggers its dependent K4 launch early (griddepcontrol.launch_dependents): tests, timeline, benches
mkdir -p gpurun_out/s5g
timeout 1200 python -m pytest tests -x -q -m gpu -k "engine or model or append or pool or kernels or headshard or p2p" 2>&1 | tail -3
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5g/every_step.txt 2>&1; sed -n '/# step 2/,+6p' gpurun_out/s5g/every_step.txt; tail -1 gpurun_out/s5g/every_step.txt
timeout 300 python tools/step_timeline.py --config cfg3 --policy "fixed(1000000)" --steps 3 > gpurun_out/s5g/attn_only.txt 2>&1; sed -n '/# step 2/,+4p' gpurun_out/s5g/attn_only.txt; tail -1 gpurun_out/s5g/attn_only.txt
for cfg in cfg3 cfg5 cfg4 cfg2 cfg1; do timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s5g/b_${cfg}.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s5g/b_${cfg}.json').read().strip().splitlines()[-1])
v=d['variants']
print('$cfg', round(d['us_per_step'],1), 'dyn', round(v['dynamic']['us_per_step'],1), 'attn_only', round(v['attn_only']['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done
