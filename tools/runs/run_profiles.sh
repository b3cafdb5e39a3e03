#!/bin/bash
# On the GPU box: kernel launch list of one bench run + full ncu captures of
# the two dominant kernels (K4 sparse decode, K2/K3 select scan) inside the
# real cfg3 bench (graph-replayed, pool >> L2).  Outputs into gpurun_out/$1.
set -u
OUT=gpurun_out/${1:-prof}
mkdir -p $OUT
KREGEX='regex:sparse_decode|select_scan|append_kernel|seal_kernel|entropy|build_ws|flush_ws|reset_kernel'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KREGEX" --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline \
  > $OUT/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_decode -s 200 -c 1 \
  -o $OUT/attn python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > $OUT/attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_scan -s 12 -c 3 \
  -o $OUT/select python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > $OUT/select.log 2>&1
ls -la $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:entropy_kernel|append_kernel|seal_kernel' -s 30 -c 3 \
  -o $OUT/small python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > $OUT/small.log 2>&1
ls -la $OUT
