timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2s_variants_cfg3.txt 2>&1
timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2s_variants_cfg2.txt 2>&1
LOPC_ENC_SERIAL=1 timeout 900 python tools/variant_bench.py cfg3 > gpurun_out/r2s_variants_cfg3_serial.txt 2>&1
LOPC_ENC_SERIAL=1 timeout 900 python tools/variant_bench.py cfg2 > gpurun_out/r2s_variants_cfg2_serial.txt 2>&1
