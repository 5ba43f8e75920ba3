bash tools/gpu_iter.sh r2f
bash tools/ncu_kernel.sh r2f_tiles k_tiles cfg3 1
bash tools/ncu_kernel.sh r2f_enc1 "k_encode" cfg3 2
