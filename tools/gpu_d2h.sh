timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_d2h.json 2> gpurun_out/bench_d2h.err
timeout 300 python tools/trace_step.py > gpurun_out/trace.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
