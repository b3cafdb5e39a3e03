# is the ~9 us wait before the first decode layer an SM shared-memory carveout switch after the append?
mkdir -p gpurun_out/s6p
for cv in 0 1; do
  CHESS_APPEND_CARVE=$cv timeout 300 python tools/step_timeline.py --config cfg3 --steps 2 > gpurun_out/s6p/cfg3_cv$cv.txt 2>&1
  echo "== cfg3 carve=$cv"; awk '/# step 1/{f=1} f' gpurun_out/s6p/cfg3_cv$cv.txt | head -5
  CHESS_APPEND_CARVE=$cv timeout 300 python tools/step_timeline.py --config cfg2 --summary-dtype f32 --steps 2 > gpurun_out/s6p/cfg2_cv$cv.txt 2>&1
  echo "== cfg2 carve=$cv"; awk '/# step 1/{f=1} f' gpurun_out/s6p/cfg2_cv$cv.txt | head -5
done
