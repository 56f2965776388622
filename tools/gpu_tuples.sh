set -x
timeout 900 python -m pytest tests/test_gpu_stage12.py -x -q -k "tuples or device_tuple" > gpurun_out/pytest_tuples.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tuples.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tuples.json 2> gpurun_out/bench_tuples.err
MX_SCAN_SEGS=4 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tuples_s4.json 2> gpurun_out/bench_tuples_s4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_tuples.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/pytest_tuples.txt
