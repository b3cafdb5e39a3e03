mkdir -p gpurun_out/s5k
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 1 --dot gpurun_out/s5k/conc.dot > /dev/null 2>&1; echo rc=$?
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 1 --sequential --dot gpurun_out/s5k/seq.dot > /dev/null 2>&1; echo rc=$?
ls -la gpurun_out/s5k
