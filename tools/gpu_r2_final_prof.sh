# final round-2 profiles: the scan kernel (ncu --set full + source page) and
# the bench step's launch list (per-launch durations)
mkdir -p gpurun_out
bash tools/gpu_r2_ncu_scan.sh
ncu -i gpurun_out/scan_src.ncu-rep --page raw --csv > gpurun_out/scan_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
ls -la gpurun_out/launches.csv gpurun_out/scan_raw.csv
