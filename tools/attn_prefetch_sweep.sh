for pf in 0 16 32 56; do
  export CHESS_ATTN_PREFETCH=$pf
  echo "== prefetch=$pf b16"; timeout 120 python tools/attn_micro.py --batch 16 --ws 45 --q-heads 32
  echo "== prefetch=$pf b8 hq64"; timeout 120 python tools/attn_micro.py --batch 8 --ws 45 --q-heads 64
  echo "== prefetch=$pf b128 ws16"; timeout 120 python tools/attn_micro.py --batch 128 --ws 16 --q-heads 32
done
