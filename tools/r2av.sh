# final code: full GPU suite + stress
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2av_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -x --durations=5 > gpurun_out/r2av_tests.log 2>&1
timeout 900 python tools/stress.py 200 3 > gpurun_out/r2av_stress.log 2>&1
