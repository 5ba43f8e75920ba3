timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2m_variants_cfg3.txt 2>&1
bash tools/ncu_kernel.sh r2m_tiles k_tiles cfg3 1
