export CHESS_B200_LIB=paper_2602_20732_b200/libchess_b200_x2.so
for m in 7 0; do
export CHESS_ATTN_MODE=$m
for args in "--batch 16 --ws 45 --q-heads 32" "--batch 8 --ws 45 --q-heads 64" "--batch 4 --ws 45 --q-heads 32" "--batch 16 --ws 24 --q-heads 32"; do
  echo "== x2 mode=$m $args"; timeout 120 python tools/attn_micro.py $args
done
done
unset CHESS_B200_LIB
export CHESS_ATTN_MODE=0
for args in "--batch 4 --ws 45 --q-heads 32" "--batch 16 --ws 24 --q-heads 32"; do
  echo "== x1 $args"; timeout 120 python tools/attn_micro.py $args
done
