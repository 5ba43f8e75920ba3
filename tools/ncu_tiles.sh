# ncu --set full of one k_tiles launch (cfg3) + the source page
TAG=${1:-tiles}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tiles" -s 2 -c 1 \
  -o gpurun_out/${TAG} python tools/prof_step.py cfg3 > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
