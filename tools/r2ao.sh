# randomised GPU-vs-oracle stress (plain, host I/O, slab mode; escapes)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ao_build.log 2>&1
timeout 1500 python tools/stress.py 400 1 > gpurun_out/r2ao_stress.log 2>&1
