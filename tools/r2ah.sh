# decoder payload prefetch variants (none / L1 / L2): cfg3 + cfg2 + cfg5 crop bench, decode DRAM bytes
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ah_build.log 2>&1
timeout 600 python tools/variant_bench.py cfg3 > gpurun_out/r2ah_var_cfg3.txt 2>&1
timeout 600 python tools/variant_bench.py cfg2 > gpurun_out/r2ah_var_cfg2.txt 2>&1
for v in pf0 pf1 pf2; do
  LOPC_LIB=$PWD/variants/liblopc_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_decode1 -s 1 -c 1 --csv python tools/prof_step.py cfg3 > gpurun_out/r2ah_dec_$v.csv 2>&1
done
