# final evidence: full GPU suite, then tools/r2final.sh (benches, reference arm, every config, slab, ncu, phases)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2g_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=10 > gpurun_out/r2g_tests.log 2>&1
bash tools/r2final.sh r2g
