timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for r in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_sc_$r.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_sc.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_sc.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt
