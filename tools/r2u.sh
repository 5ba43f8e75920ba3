# Re-entry check of HEAD: build, smoke, full GPU suite, bench cfg3 + cfg2, phase timeline.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2u_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -x --durations=10 > gpurun_out/r2u_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench_cfg3.json 2> gpurun_out/r2u_bench_cfg3.err
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_bench_cfg2.json 2> gpurun_out/r2u_bench_cfg2.err
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2u_phase_cfg3.txt 2>&1
