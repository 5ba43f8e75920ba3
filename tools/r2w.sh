# balanced g=4/8 RZE data phase: parity tests, cfg3/cfg2 bench, phase cycles; k_tiles occupancy variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_engine.py -q --timeout 600 -x > gpurun_out/r2w_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2w_bench_cfg2.json 2>&1
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2w_phase_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2w_variants.txt 2>&1
