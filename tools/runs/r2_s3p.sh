# checkpoint: whole GPU suite + smoke + default bench (cfg3, f16tc)
mkdir -p gpurun_out/s3p
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3p/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/s3p/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3p/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s3p/smoke.log
timeout 600 python bench.py > gpurun_out/s3p/bench_default.json 2> gpurun_out/s3p/bench_default.err; echo "bench rc=$?"; tail -c 600 gpurun_out/s3p/bench_default.json
