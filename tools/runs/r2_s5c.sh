# per-kernel timeline of captured cfg3 steps (CUPTI via torch.profiler): headline and attention-only
mkdir -p gpurun_out/s5c
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 --json gpurun_out/s5c/every_step.json > gpurun_out/s5c/every_step.txt 2>&1; echo rc=$?
timeout 300 python tools/step_timeline.py --config cfg3 --policy "fixed(1000000)" --steps 3 --json gpurun_out/s5c/attn_only.json > gpurun_out/s5c/attn_only.txt 2>&1; echo rc=$?
tail -3 gpurun_out/s5c/every_step.txt; tail -3 gpurun_out/s5c/attn_only.txt
