# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_rt.py
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1
for t in memcheck racecheck synccheck; do
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_rt.py > gpurun_out/san_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$t.log
done
