for lib in libchess_b200.so libchess_b200_x2.so; do
  export CHESS_B200_LIB=paper_2602_20732_b200/$lib
  for args in "--batch 16 --ws 45 --q-heads 32" "--batch 8 --ws 45 --q-heads 64" "--batch 1 --ws 16 --q-heads 32" "--batch 128 --ws 16 --q-heads 32" "--batch 32 --ws 45 --q-heads 32"; do
    echo "== $lib $args"; timeout 120 python tools/attn_micro.py $args
  done
done
