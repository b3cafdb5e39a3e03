mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_engine_oracle.py tests/test_gpu_acceptance.py "tests/test_gpu_select.py::test_select_at_bench_cfg3_state" -q -x > gpurun_out/r2b/new.log 2>&1; echo "new rc=$?"; tail -5 gpurun_out/r2b/new.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b/all.log 2>&1; echo "all rc=$?"; tail -8 gpurun_out/r2b/all.log
