timeout 1800 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
tail -n 30 gpurun_out/pytest_gpu.txt
head -c 3000 gpurun_out/bench.json
tail -n 5 gpurun_out/bench.err
