# Build liblopc variants (launch-bound / occupancy experiments) into variants/
set -e
mkdir -p variants
SRC=paper_2603_26968_b200/csrc/lopc_api.cu
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -shared"
for v in "$@"; do  # v = name:DEFINES (comma separated)
  name=${v%%:*}; defs=${v#*:}
  D=""; for d in ${defs//,/ }; do D="$D -D$d"; done
  nvcc $F $D -o variants/liblopc_$name.so $SRC &
done
wait
