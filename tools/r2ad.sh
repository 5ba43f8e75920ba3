# slab mode on the tile engine: slab / engine / parity tests, cfg2 slab bench at N=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ad_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_engines.py tests/test_gpu_parity.py -q --timeout 900 -x > gpurun_out/r2ad_tests.log 2>&1
timeout 300 python bench.py --config cfg2 --slab --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ad_bench_slab_cfg2.json 2>&1
timeout 300 python bench.py --config cfg3 --slab --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ad_bench_slab_cfg3.json 2>&1
