mkdir -p gpurun_out/s5l
for v in "0 0" "1 0" "0 1" "1 1"; do set -- $v
CHESS_SIDE_LAST=$1 CHESS_FORK_AFTER_LAYERS=$2 timeout 300 python tools/step_timeline.py --config cfg3 --policy every_step --steps 3 > gpurun_out/s5l/t_$1_$2.txt 2>&1; echo side_last=$1 fork_after=$2; sed -n '/# step 2/,+3p' gpurun_out/s5l/t_$1_$2.txt; tail -1 gpurun_out/s5l/t_$1_$2.txt
done
