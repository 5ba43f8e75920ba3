# bin-role x prefetch into L2 at CTA start (LOPC_ENC_PF)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2az_build.log 2>&1
timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2az_var_cfg3.txt 2>&1
timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2az_var_cfg2.txt 2>&1
timeout 900 python tools/variant_bench.py cfg5 > gpurun_out/r2az_var_cfg5.txt 2>&1
