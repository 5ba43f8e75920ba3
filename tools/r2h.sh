bash tools/gpu_iter.sh r2h
timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2h_variants_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2h_variants_cfg2.txt 2>&1
