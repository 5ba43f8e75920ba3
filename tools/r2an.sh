# slab escapes fix (tests) + k_tiles flag words in shared memory (LOPC_TILE_FSMEM) for 4 CTAs/SM: parity on the variant, variant bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2an_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_parity.py -q --timeout 600 > gpurun_out/r2an_tests.log 2>&1
LOPC_LIB=$PWD/variants/liblopc_fs1.so timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/r2an_tests_fs1.log 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2an_var_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2an_var_cfg2.txt 2>&1
