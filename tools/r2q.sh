python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_concurrency.py -q --timeout 900 -x > gpurun_out/r2q_tests.log 2>&1
for d in 1 2; do LOPC_DECODER=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_bench_dec$d.json 2>&1; done
LOPC_DECODER=1 timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_bench_cfg2_dec1.json 2>&1
LOPC_DECODER=2 timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_bench_cfg2_dec2.json 2>&1
