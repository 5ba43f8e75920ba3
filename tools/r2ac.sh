# rze_dec: every warp decodes the upper bitmap levels (no barrier on warp 0); rze_enc: every warp counts |K1|, |K2|
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ac_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -k "not test_cfg5" -q --timeout 900 -x > gpurun_out/r2ac_tests.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ac_bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ac_bench_cfg2.json 2>&1
timeout 200 python tools/phase_prof.py cfg3 > gpurun_out/r2ac_phase_cfg3.txt 2>&1
