# f64 k_quant_flags CTAs per SM 3 vs 4 (cfg5)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2bb_build.log 2>&1
timeout 900 python tools/variant_bench.py cfg5 > gpurun_out/r2bb_var_cfg5.txt 2>&1
