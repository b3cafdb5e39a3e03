# fork point of the concurrent step (CHESS_FORK_AFTER_LAYERS): timeline + benches
mkdir -p gpurun_out/s5i
for n in 0 1 2; do
CHESS_FORK_AFTER_LAYERS=$n timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5i/every_step_$n.txt 2>&1; echo fork_after=$n; sed -n '/# step 2/,+6p' gpurun_out/s5i/every_step_$n.txt; tail -1 gpurun_out/s5i/every_step_$n.txt
done
for n in 0 1 2; do for cfg in cfg3 cfg5 cfg4; do CHESS_FORK_AFTER_LAYERS=$n timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s5i/b_${cfg}_$n.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s5i/b_${cfg}_$n.json').read().strip().splitlines()[-1])
v=d['variants']
print('fork_after=$n $cfg', round(d['us_per_step'],1), 'dyn', round(v['dynamic']['us_per_step'],1), 'attn_only', round(v['attn_only']['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done; done
