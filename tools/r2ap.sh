# NEXT f3 refresh on the final code: error-bound sweep x cfg1-4 (+ engine ablation)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ap_build.log 2>&1
timeout 2400 python tools/eb_sweep.py > gpurun_out/r2ap_eb.log 2>&1
cp results/eb_sweep.json gpurun_out/eb_sweep_r2.json
