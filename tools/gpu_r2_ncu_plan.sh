mkdir -p gpurun_out
timeout 900 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none -k regex:plan_big -c 1 -o gpurun_out/plan_src python tools/cfg5_plan.py > gpurun_out/ncu_plan.log 2>&1
ncu -i gpurun_out/plan_src.ncu-rep --page source --csv --print-source sass > gpurun_out/plan_sass.csv 2>&1
ls -la gpurun_out/plan_sass.csv
