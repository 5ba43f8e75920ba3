python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
bash tools/ncu_kernel.sh r2v_dec k_decode1 cfg3 1
bash tools/ncu_kernel.sh r2v_tiles k_tiles cfg3 1
bash tools/ncu_kernel.sh r2v_qf k_quant_flags cfg3 1
