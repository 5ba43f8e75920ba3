# subbin-role CTAs 6: GPU parity/engine/slab tests, cfg5 variant check, default bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2au_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_slab.py tests/test_gpu_noa.py tests/test_gpu_concurrency.py -q --timeout 900 > gpurun_out/r2au_tests.log 2>&1
timeout 900 python tools/variant_bench.py cfg5 > gpurun_out/r2au_var_cfg5.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_r2au.json 2> gpurun_out/bench_r2au.err
