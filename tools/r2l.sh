python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_engine.py -q --timeout 900 -x > gpurun_out/r2l_tests.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_bench_cfg3.json 2> gpurun_out/r2l_bench_cfg3.err
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2l_phase_cfg3.txt 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/r2l_phase_cfg2.txt 2>&1
