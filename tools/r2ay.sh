# final HEAD: smoke, full GPU suite, default bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2ay_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=5 > gpurun_out/r2ay_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r2ay.json 2> gpurun_out/bench_r2ay.err
