# debug: concurrent upper-level decode, default vs printf build, repeated
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2as_build.log 2>&1
for v in nodbg dbg nodbg; do
  echo "== $v" >> gpurun_out/r2as_tests.log
  LOPC_LIB=$PWD/variants/liblopc_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -s 2>&1 | grep -E 'DBG|passed|failed|FAILED' | head -20 >> gpurun_out/r2as_tests.log
done
