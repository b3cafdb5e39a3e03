mkdir -p gpurun_out/s5n
for c in cfg3 cfg2; do for p in 1 0; do for f in 0 1; do
CHESS_ATTN_PDL_FIRST=$p CHESS_FORK_AFTER_LAYERS=$f timeout 300 python tools/step_timeline.py --config $c --policy every_step --steps 3 > gpurun_out/s5n/${c}_$p$f.txt 2>&1; echo $c pdl_first=$p fork_after=$f; sed -n '/# step 2/,+3p' gpurun_out/s5n/${c}_$p$f.txt | tail -3; tail -1 gpurun_out/s5n/${c}_$p$f.txt
done; done; done
