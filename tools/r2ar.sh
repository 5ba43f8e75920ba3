# debug: concurrent upper-level decode, which check fails on the ragged 2D ties case
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ar_build.log 2>&1
LOPC_LIB=$PWD/variants/liblopc_dbg.so timeout 600 python -m pytest tests/test_gpu_parity.py -k "random_fields" -x -q -s > gpurun_out/r2ar_tests.log 2>&1
