# f64 (cfg5 crop) line profiles of the codec kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ai_build.log 2>&1
bash tools/ncu_kernel.sh r2ai_dec k_decode1 cfg5 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_encode -s 2 -c 2 \
  -o gpurun_out/r2ai_enc python tools/prof_step.py cfg5 > gpurun_out/r2ai_enc_ncu.log 2>&1
ncu -i gpurun_out/r2ai_enc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2ai_enc_cudasass.csv 2>/dev/null
ncu -i gpurun_out/r2ai_enc.ncu-rep --page details --csv > gpurun_out/r2ai_enc_details.csv 2>/dev/null
rm -f gpurun_out/r2ai_enc.ncu-rep
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2ai_bench_cfg5.json 2>&1
