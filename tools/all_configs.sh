# One bench line per config (N=1) and the slab-mode path at N=1, into gpurun_out/
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 4 > gpurun_out/bench_all_$c.json 2> gpurun_out/bench_all_$c.err
done
timeout 600 torchrun --standalone --nproc-per-node 1 bench.py --slab --config cfg2 --steps 5 --warmup 3 > gpurun_out/bench_all_slab_cfg2.json 2> gpurun_out/bench_all_slab_cfg2.err
