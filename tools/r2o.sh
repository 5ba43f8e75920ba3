timeout 1200 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_concurrency.py -q --timeout 900 > gpurun_out/r2o_tests.log 2>&1
bash tools/sanitize.sh
