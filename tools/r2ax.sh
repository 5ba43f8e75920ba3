# host-I/O decompress pipeline depth 4 / 8 / 16: e2e on cfg3 and cfg2; host-path tests on the new default
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ax_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py -q --timeout 600 > gpurun_out/r2ax_tests.log 2>&1
timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2ax_var_cfg3.txt 2>&1
timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2ax_var_cfg2.txt 2>&1
