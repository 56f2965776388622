for o in 4 6 8; do MX_FAST1_OCC=$o timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_occ$o.json 2> gpurun_out/bench_occ$o.err; done
MX_SCAN=fast1_off timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_occoff.json 2> gpurun_out/bench_occoff.err
timeout 300 python -m pytest tests/test_gpu_stage12.py -x -q -k "tuples" > gpurun_out/pytest_tuples.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tuples.txt
MX_FAST1_OCC=4 timeout 300 python -m pytest tests/test_gpu_stage12.py -x -q -k "tuples" >> gpurun_out/pytest_tuples.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tuples.txt
tail -2 gpurun_out/pytest_tuples.txt
