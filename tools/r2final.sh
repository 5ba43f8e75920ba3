# Round-2 final evidence (no GPU suite: see r2ae): smoke, default bench (cfg3,
# CPU baselines), reference arm, every config, slab path under torchrun, ncu
# captures + launch lists of cfg3 and cfg2, phase timelines.
TAG=${1:-r2f}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/smi_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2>&1
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-budget 4 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 600 torchrun --standalone --nproc-per-node 1 bench.py --slab --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_slab_cfg2.json 2> gpurun_out/bench_${TAG}_slab_cfg2.err
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/phase_${TAG}_cfg3.txt 2>&1
timeout 200 python tools/phase_prof.py cfg2 > gpurun_out/phase_${TAG}_cfg2.txt 2>&1
bash tools/profile_round.sh ${TAG} cfg3
bash tools/profile_round.sh ${TAG}c2 cfg2
