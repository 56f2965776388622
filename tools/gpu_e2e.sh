timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
timeout 300 python -m pytest tests/test_gpu_bench.py -x -q > gpurun_out/pytest_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_bench.txt
tail -2 gpurun_out/pytest_bench.txt
