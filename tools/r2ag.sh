# per-chunk escape bits (k_quant_flags -> subbin encoder): parity/engine/noa tests, bench cfg3/cfg2, encoder traffic
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ag_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_noa.py tests/test_gpu_check.py -q --timeout 900 -x > gpurun_out/r2ag_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ag_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ag_bench_cfg2.json 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_encode -s 2 -c 2 --csv python tools/prof_step.py cfg3 > gpurun_out/r2ag_enc_traffic.csv 2>&1
