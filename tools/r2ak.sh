# k_quant_flags chunk-escape marking in the store path (A) or after the row loop (B): bench cfg3/cfg2 + escape parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ak_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/r2ak_tests.log 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2ak_var_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2ak_var_cfg2.txt 2>&1
