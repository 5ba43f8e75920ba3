python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_slab.py -q --timeout 900 -x > gpurun_out/r2r_tests.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2r_bench_cfg2.json 2>&1
timeout 1200 python tools/oracle_timing.py cfg1 cfg4 cfg2 --reps 3 > gpurun_out/r2r_oracle_timing.jsonl 2> gpurun_out/r2r_oracle_timing.err
