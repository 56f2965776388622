timeout 600 python -m pytest tests/test_gpu_scan_u16.py -x -q > gpurun_out/pytest_u16.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_u16.txt
timeout 300 python tools/trace_step.py > gpurun_out/trace.txt 2>&1
timeout 300 python tools/trace_step.py --cprofile > gpurun_out/trace_cprofile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -n 3 gpurun_out/pytest_u16.txt; tail -n 20 gpurun_out/trace.txt
