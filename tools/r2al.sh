# k_quant_flags row-loop unroll variants; slab mode on the planes-mode encoder (tests + slab bench)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2al_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_parity.py tests/test_gpu_cfg5.py::test_cfg5_eight_slabs_crop -q --timeout 900 -x > gpurun_out/r2al_tests.log 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2al_var_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2al_var_cfg2.txt 2>&1
timeout 300 python bench.py --config cfg3 --slab --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2al_bench_slab_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --slab --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2al_bench_slab_cfg2.json 2>&1
