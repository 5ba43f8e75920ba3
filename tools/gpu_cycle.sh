timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --cpu-budget 3 > gpurun_out/bench.log 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/phase.txt 2>&1
