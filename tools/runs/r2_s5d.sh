# append loads in one round trip + entropy one CTA per SM: tests, step timeline, bench A/B
mkdir -p gpurun_out/s5d
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pagesel.py tests/test_gpu_engine_oracle.py tests/test_gpu_pool.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5d/every_step.txt 2>&1; sed -n '/# step 2/,+8p' gpurun_out/s5d/every_step.txt; tail -1 gpurun_out/s5d/every_step.txt
timeout 300 python tools/step_timeline.py --config cfg3 --policy "fixed(1000000)" --steps 3 > gpurun_out/s5d/attn_only.txt 2>&1; sed -n '/# step 2/,+5p' gpurun_out/s5d/attn_only.txt; tail -1 gpurun_out/s5d/attn_only.txt
for e in 1 2; do for cfg in cfg3 cfg2; do CHESS_ENT_PER_SM=$e timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/s5d/b_${cfg}_$e.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/s5d/b_${cfg}_$e.json').read().strip().splitlines()[-1])
v=d['variants']
print('ent_per_sm=$e $cfg', round(d['us_per_step'],1), 'dyn', round(v['dynamic']['us_per_step'],1), 'attn_only', round(v['attn_only']['us_per_step'],1), 'K4', round(d['roofline']['launch_us'],2))"; done; done
