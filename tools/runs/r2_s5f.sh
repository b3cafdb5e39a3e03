# concurrent step: first decode layer issued before the side-stream work (CHESS_FIRST_LAYER_FIRST A/B)
mkdir -p gpurun_out/s5f
for c in 1 0; do
CHESS_FIRST_LAYER_FIRST=$c timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5f/every_step_$c.txt 2>&1; echo first=$c; sed -n '/# step 2/,+8p' gpurun_out/s5f/every_step_$c.txt; tail -1 gpurun_out/s5f/every_step_$c.txt
done
for c in 1 0; do for cfg in cfg3 cfg5 cfg4 cfg2; do CHESS_FIRST_LAYER_FIRST=$c timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s5f/b_${cfg}_$c.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s5f/b_${cfg}_$c.json').read().strip().splitlines()[-1])
v=d['variants']
print('first=$c $cfg', round(d['us_per_step'],1), 'dyn', round(v['dynamic']['us_per_step'],1), 'attn_only', round(v['attn_only']['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done; done
