# hybrid engine (tile pass 1, then point worklist on a short tail): engine/parity tests, benches per engine
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2af_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_slab.py -q --timeout 900 -x > gpurun_out/r2af_tests.log 2>&1
for c in cfg2 cfg4 cfg3 cfg1; do
  for e in 0 3 2; do
    timeout 300 python bench.py --config $c --engine $e --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r2af_bench_${c}_e$e.json 2>&1
  done
done
