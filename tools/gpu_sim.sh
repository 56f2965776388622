MX_SCAN_SEGS=4 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err
MX_SCAN_SEGS=4 timeout 600 python -m pytest tests/test_gpu_stage12.py -x -q -k "tuples" > gpurun_out/pytest_s4.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_s4.txt
timeout 900 python tools/shard_sim.py --world 8 > gpurun_out/shard_sim_w8_tuples.json 2> gpurun_out/shard_sim.err
tail -2 gpurun_out/pytest_s4.txt
