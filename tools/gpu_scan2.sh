timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_scan2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scan2.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_u16.json 2> gpurun_out/bench_u16.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 --layout columns > gpurun_out/bench_cols.json 2> gpurun_out/bench_cols.err
for o in 4 6; do MX_FAST1_OCC=$o timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_u16_occ$o.json 2>/dev/null; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_fast_kernel -s 2 -c 1 -o gpurun_out/scan2_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan2.log 2>&1
tail -3 gpurun_out/pytest_scan2.txt
