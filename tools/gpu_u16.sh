timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_bench.py -x -q > gpurun_out/pytest_u16.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_u16.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_u16.json 2> gpurun_out/bench_u16.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 --layout columns > gpurun_out/bench_cols.json 2> gpurun_out/bench_cols.err
tail -3 gpurun_out/pytest_u16.txt
