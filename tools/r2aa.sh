python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aa_build.log 2>&1
bash tools/ncu_kernel.sh r2aa_dec k_decode1 cfg3 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_encode -s 2 -c 2 \
  -o gpurun_out/r2aa_enc python tools/prof_step.py cfg3 > gpurun_out/r2aa_enc_ncu.log 2>&1
ncu -i gpurun_out/r2aa_enc.ncu-rep --page source --csv > gpurun_out/r2aa_enc_source.csv 2>/dev/null
ncu -i gpurun_out/r2aa_enc.ncu-rep --page details --csv > gpurun_out/r2aa_enc_details.csv 2>/dev/null
ncu -i gpurun_out/r2aa_enc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2aa_enc_cudasass.csv 2>/dev/null
rm -f gpurun_out/r2aa_enc.ncu-rep
