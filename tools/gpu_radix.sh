timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_rs2.json 2> gpurun_out/bench_rs2.err
MX_RADIX=direct timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_rs1.json 2> gpurun_out/bench_rs1.err
tail -2 gpurun_out/pytest_gpu.txt
