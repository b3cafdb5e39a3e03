# cfg1 / cfg2 step timelines (where the small-batch step goes)
mkdir -p gpurun_out/s6h
timeout 300 python tools/step_timeline.py --config cfg1 --summary-dtype f32 --steps 2 > gpurun_out/s6h/cfg1_every_step.txt 2>&1; echo rc=$?
timeout 300 python tools/step_timeline.py --config cfg2 --summary-dtype f32 --steps 2 > gpurun_out/s6h/cfg2_every_step.txt 2>&1; echo rc=$?
grep -v Warning gpurun_out/s6h/cfg1_every_step.txt | grep -v warn | tail -20
