# decoder: both payloads' upper RZE levels decoded at once (two warps, one barrier): tests + bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aq_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_slab.py tests/test_gpu_noa.py -q --timeout 900 -x > gpurun_out/r2aq_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2aq_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2aq_bench_cfg2.json 2>&1
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2aq_bench_cfg5.json 2>&1
