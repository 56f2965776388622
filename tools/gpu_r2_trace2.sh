# stage12 parity, bench, CUPTI step timeline, host split, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage12.py -x -q > gpurun_out/fy_t1.txt 2>&1; echo "rc=$?" >> gpurun_out/fy_t1.txt
timeout 600 python bench.py --no-cpu-baseline --no-extras > gpurun_out/fy_bench.json 2> gpurun_out/fy_bench.err
timeout 600 python tools/trace_step.py > gpurun_out/trace2.txt 2>&1
MX_HOST_TIMING=1 timeout 600 python tools/host_split.py > gpurun_out/host_split.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fy_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/fy_ncu.log 2>&1
tail -n 2 gpurun_out/fy_t1.txt
