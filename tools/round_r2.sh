# Round-2 evidence run: full GPU suite (slow cfg5 slab test included), the
# default bench (cfg3, with the CPU baselines), the reference arm, the ncu
# captures of cfg3 and the sanitizer summary is separate (tools/sanitize.sh).
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 2000 -x --durations=15 > gpurun_out/gpu_tests_${TAG}.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/smi_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1
bash tools/profile_round.sh ${TAG} cfg3
