# One GPU iteration: build, the parity / concurrency / engine / slab tests,
# a short cfg3 bench and the per-pass repair timeline (cfg3, cfg2).
TAG=${1:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_engine.py tests/test_gpu_slab.py -q --timeout 900 -x > gpurun_out/${TAG}_tests.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench_cfg3.err
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/${TAG}_phase_cfg3.txt 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/${TAG}_phase_cfg2.txt 2>&1
