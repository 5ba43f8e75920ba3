# quick GPU cycle: parity + slab tests, a short bench, per-phase cycles
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_engine.py -q --timeout 600 -x > gpurun_out/quick_tests.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/phase.txt 2>&1
