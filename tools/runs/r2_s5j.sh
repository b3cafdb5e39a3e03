# graph edge census + timeline: concurrent vs sequential every_step
mkdir -p gpurun_out/s5j
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5j/conc.txt 2>&1; head -3 gpurun_out/s5j/conc.txt | cut -c1-1500; sed -n '/# step 2/,+3p' gpurun_out/s5j/conc.txt
timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 --sequential > gpurun_out/s5j/seq.txt 2>&1; head -3 gpurun_out/s5j/seq.txt | cut -c1-1500; sed -n '/# step 2/,+3p' gpurun_out/s5j/seq.txt; tail -1 gpurun_out/s5j/seq.txt
