# slab escapes test (both engines, f32/f64) + slab file
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2am_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_slab.py -q --timeout 600 > gpurun_out/r2am_tests.log 2>&1
