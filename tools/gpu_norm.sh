timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_np_$r.json 2>/dev/null
MX_NORM_NOPACK=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_nn_$r.json 2>/dev/null
done
tail -2 gpurun_out/pytest_gpu.txt
