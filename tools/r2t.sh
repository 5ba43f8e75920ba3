python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_concurrency.py tests/test_gpu_noa.py -q --timeout 900 -x > gpurun_out/r2t_tests.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_bench_cfg3.json 2>&1
bash tools/profile_round.sh r2t5 cfg5
