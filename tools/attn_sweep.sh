#!/bin/bash
# K4 micro sweep over the config shapes.  Env A/B knobs: CHESS_ATTN_MODE
# (1 loads only, 2 math only, 7 force stream-K, 8 no PDL wait),
# CHESS_ATTN_CLUSTER=0 (no cluster-merge mode); TRACE=1 uses the
# debug-timeline library (libchess_b200_trace.so).
OUT=gpurun_out/${1:-attn_sweep}
MODES=${MODES:-0}
CLUSTERS=${CLUSTERS:-"1 0"}
mkdir -p $OUT
[ -n "$TRACE" ] && export CHESS_B200_LIB=paper_2602_20732_b200/libchess_b200_trace.so
run() { echo "== mode=${CHESS_ATTN_MODE:-0} cluster=${CHESS_ATTN_CLUSTER:-1} trace=${TRACE:-0} $*"; timeout 120 python tools/attn_micro.py "$@"; }
{
for cl in $CLUSTERS; do
for m in $MODES; do
  export CHESS_ATTN_MODE=$m CHESS_ATTN_CLUSTER=$cl
  [ -z "$SMALL" ] && run --batch 16 --ws 45 --q-heads 32
  run --batch 8 --ws 45 --q-heads 64
  run --batch 1 --ws 16 --q-heads 32
  run --batch 4 --ws 45 --q-heads 32
done
done
} > $OUT/sweep.txt 2>&1
