# full GPU suite (cfg5 included) + compute-sanitizer (memcheck/racecheck/synccheck) incl. slab mode and corrupt streams
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2ae_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=10 > gpurun_out/r2ae_tests.log 2>&1
bash tools/sanitize.sh
