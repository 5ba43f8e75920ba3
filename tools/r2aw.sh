# bisect the concurrent upper-level decode: LOPC_EARLY 0 (sequential), 1 (subbins' early), 2 (bins' early), 3 (both)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aw_build.log 2>&1
for v in e0 e1 e2 e3; do
  echo "== $v" >> gpurun_out/r2aw_tests.log
  LOPC_LIB=$PWD/variants/liblopc_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -1 >> gpurun_out/r2aw_tests.log
done
