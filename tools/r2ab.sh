# encoder: x loads before the plane gather (bins role), ballot prefixes in level_up_warp; decoder line profile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ab_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -x > gpurun_out/r2ab_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ab_bench_cfg2.json 2>&1
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2ab_phase_cfg3.txt 2>&1
bash tools/ncu_kernel.sh r2ab_dec k_decode1 cfg3 1
