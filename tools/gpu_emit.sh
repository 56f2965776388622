timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_ew2.json 2> gpurun_out/bench_ew2.err
MX_EMIT_DIRECT=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_ew1.json 2> gpurun_out/bench_ew1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ew.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ew.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt
