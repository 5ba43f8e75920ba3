bash tools/gpu_iter.sh r2g
bash tools/ncu_kernel.sh r2g_tiles k_tiles cfg3 1
bash tools/ncu_kernel.sh r2g_qf k_quant_flags cfg3 1
bash tools/ncu_kernel.sh r2g_dec k_decode cfg3 1
