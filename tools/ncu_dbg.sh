python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dbg_build.log 2>&1
ls -la paper_2603_26968_b200/*.so >> gpurun_out/dbg_build.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg_launches.csv python tools/prof_step.py cfg2 > gpurun_out/dbg.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"tiles" -c 1 -o gpurun_out/dbg_tiles python tools/prof_step.py cfg2 >> gpurun_out/dbg.log 2>&1
ncu -i gpurun_out/dbg_tiles.ncu-rep --page source --csv > gpurun_out/dbg_tiles_source.csv 2>&1
ncu -i gpurun_out/dbg_tiles.ncu-rep --page details --csv > gpurun_out/dbg_tiles_details.csv 2>&1
