mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_u16 -s 2 -c 1 -o gpurun_out/scan_src python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1
ncu -i gpurun_out/scan_src.ncu-rep --page source --csv --print-source sass > gpurun_out/scan_sass.csv 2>&1
ncu -i gpurun_out/scan_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/scan_cuda.csv 2>&1
ls -la gpurun_out/scan_*; tail -3 gpurun_out/ncu_scan.log
