# ncu --set full of one launch of kernel regex $2 on config $3 (skip $4 launches), source + details CSV
TAG=$1; K=$2; CFG=${3:-cfg3}; SKIP=${4:-1}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -s $SKIP -c 1 \
  -o gpurun_out/${TAG} python tools/prof_step.py $CFG > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_cudasass.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
