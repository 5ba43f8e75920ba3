# occupancy re-tune after the r2 changes: subbin-role / bin-role / k_quant_flags CTAs per SM
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2at_build.log 2>&1
timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2at_var_cfg3.txt 2>&1
timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2at_var_cfg2.txt 2>&1
