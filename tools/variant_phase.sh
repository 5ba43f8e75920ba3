# per-variant sweep pass timeline (tools/phase_prof.py) for the configs given
for so in variants/liblopc_*.so; do
  for c in "$@"; do
    echo "== $(basename $so) $c"; LOPC_LIB=$PWD/$so timeout 300 python tools/phase_prof.py $c | grep "sweep"
  done
done
