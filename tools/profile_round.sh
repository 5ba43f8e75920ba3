# One ncu --set full capture of every kernel of one compress+decompress step
# of a config (after a warm-up step), plus the per-launch duration list of a
# short bench run.  Outputs land in gpurun_out/ (scratch); summaries are
# copied to profiles/ by tools/ncu_summary.py TAG --config CFG.
set -x
TAG=${1:-r2}
CFG=${2:-cfg3}
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"k_quant_flags|k_tiles|k_sweep|k_encode|k_chunk_scan|k_place|k_decode" -s 8 -c 8 \
  -o gpurun_out/full_${TAG} python tools/prof_step.py ${CFG} > gpurun_out/full_${TAG}.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  -k regex:"k_quant_flags|k_tiles|k_sweep|k_encode|k_chunk_scan|k_place|k_decode|k_planes" \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --config ${CFG} --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/launches_${TAG}.log 2>&1
