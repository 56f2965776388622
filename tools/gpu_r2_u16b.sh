timeout 900 python -m pytest tests/test_gpu_scan_u16.py tests/test_gpu_stage12.py tests/test_gpu_rows.py -x -q > gpurun_out/pytest_s12.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_s12.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -x -q -k "cfg2" > gpurun_out/pytest_scale.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_scale.txt
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_u16.json 2> gpurun_out/bench_u16.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_u16 -s 2 -c 1 -o gpurun_out/scan_u16b python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_u16.log 2>&1
for f in gpurun_out/pytest_s12.txt gpurun_out/pytest_scale.txt; do tail -n 3 $f; done
head -c 1200 gpurun_out/bench_u16.json
