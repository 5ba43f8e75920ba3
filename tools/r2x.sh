# k_tiles L1 prefetch of the next tile: parity tests, cfg3/cfg2 variant bench (PF on / off)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_engine.py tests/test_gpu_concurrency.py -q --timeout 600 -x > gpurun_out/r2x_tests.log 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2x_variants_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2x_variants_cfg2.txt 2>&1
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2x_phase_cfg3.txt 2>&1
