for m in 1 0 2 1 0 2; do LOPC_OVERLAP=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode $m', round(d['compress_GBps'],1), d['step_ms']['compress'])"; done
