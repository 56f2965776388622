timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_t8.json 2> gpurun_out/bench_t8.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_fast_kernel -s 2 -c 1 -o gpurun_out/scan1_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan1.log 2>&1
ls -la gpurun_out
