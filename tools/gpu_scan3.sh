timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 --layout columns > gpurun_out/bench_s3c.json 2> gpurun_out/bench_s3c.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_fast_kernel -s 2 -c 1 -o gpurun_out/scan3_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_scan3.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt
