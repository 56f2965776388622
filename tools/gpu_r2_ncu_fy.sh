# ncu --set full + SASS source page of the CTA-wide shuffle kernels
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:cursor_shuffle|component_order' -s 2 -c 2 -o gpurun_out/fy_src python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_fy.log 2>&1
ncu -i gpurun_out/fy_src.ncu-rep --page source --csv --print-source sass > gpurun_out/fy_sass.csv 2>&1
ncu -i gpurun_out/fy_src.ncu-rep --page raw --csv > gpurun_out/fy_raw.csv 2>&1
ls -la gpurun_out/fy_*
