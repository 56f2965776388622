timeout 600 python -m pytest tests/test_gpu_scan_u16.py tests/test_gpu_stage12.py -x -q > gpurun_out/pytest_u16.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_u16.txt
timeout 300 python tools/trace_step.py > gpurun_out/trace.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_u16 -s 2 -c 1 -o gpurun_out/scan_u16_r2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_u16.log 2>&1
tail -n 3 gpurun_out/pytest_u16.txt; tail -n 40 gpurun_out/trace.txt
