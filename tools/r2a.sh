python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_cfg3.json 2> gpurun_out/r2a_bench_cfg3.err
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2a_phase_cfg3.txt 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/r2a_phase_cfg2.txt 2>&1
