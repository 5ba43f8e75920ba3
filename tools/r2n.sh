timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2n_variants_cfg3.txt 2>&1
timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2n_variants_cfg2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -q --timeout 900 -x > gpurun_out/r2n_tests.log 2>&1
