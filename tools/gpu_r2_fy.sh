# CTA-wide Fisher-Yates: cursor / component-order parity, full-size jobs, bench, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage12.py -x -q > gpurun_out/fy_t1.txt 2>&1; echo "rc=$?" >> gpurun_out/fy_t1.txt
timeout 1200 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_shard.py tests/test_gpu_partition.py -x -q > gpurun_out/fy_t2.txt 2>&1; echo "rc=$?" >> gpurun_out/fy_t2.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/fy_bench.json 2> gpurun_out/fy_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fy_launches.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/fy_ncu.log 2>&1
tail -2 gpurun_out/fy_t1.txt gpurun_out/fy_t2.txt; head -c 300 gpurun_out/fy_bench.json
