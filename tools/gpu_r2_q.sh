# quick check: stage-1/2 parity, full-size cfg2 parity, bench, host split, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_scale.py tests/test_gpu_rows.py tests/test_gpu_scan_u16.py -x -q > gpurun_out/q_t1.txt 2>&1; echo "rc=$?" >> gpurun_out/q_t1.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -x -q -k cfg2 > gpurun_out/q_t2.txt 2>&1; echo "rc=$?" >> gpurun_out/q_t2.txt
timeout 600 python bench.py --no-cpu-baseline --no-extras > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
MX_HOST_TIMING=1 timeout 600 python tools/host_split.py > gpurun_out/q_host.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1
tail -n 2 gpurun_out/q_t1.txt gpurun_out/q_t2.txt
