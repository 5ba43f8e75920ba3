# final evidence (final code): smoke, full GPU suite, stress, then tools/r2final.sh (benches, reference arm, every config, slab, ncu, phases)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=10 > gpurun_out/r2h_tests.log 2>&1
timeout 900 python tools/stress.py 200 2 > gpurun_out/r2h_stress.log 2>&1
bash tools/r2final.sh r2h
