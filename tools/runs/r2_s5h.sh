# append -> first decode layer gap: sequential step (policy never) vs concurrent
mkdir -p gpurun_out/s5h
timeout 300 python tools/step_timeline.py --config cfg3 --policy never --steps 3 > gpurun_out/s5h/never.txt 2>&1; sed -n '/# step 2/,+4p' gpurun_out/s5h/never.txt; tail -1 gpurun_out/s5h/never.txt
CHESS_ATTN_MODE=8 timeout 300 python tools/step_timeline.py --config cfg3 --policy never --steps 3 > gpurun_out/s5h/never_mode8.txt 2>&1; sed -n '/# step 2/,+4p' gpurun_out/s5h/never_mode8.txt
