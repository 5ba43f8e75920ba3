# f64 x prefetch in the bin role: f64 parity (random fields, engines, cfg5 8-slab crop) + cfg5 bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2ba_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -x > gpurun_out/r2ba_tests.log 2>&1
timeout 600 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2ba_cfg5.json 2>&1
