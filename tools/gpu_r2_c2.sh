timeout 600 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_rows.py tests/test_gpu_scan_u16.py -x -q > gpurun_out/pytest_c.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_c.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
timeout 300 python tools/host_split.py > gpurun_out/host_split.txt 2>&1
timeout 300 python tools/trace_step.py --cprofile > gpurun_out/cprofile.txt 2>&1
timeout 300 python tools/trace_step.py > gpurun_out/trace_c.txt 2>&1
tail -n 3 gpurun_out/pytest_c.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_c.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
tail -n 3 gpurun_out/bench_c.err
cat gpurun_out/host_split.txt | tail -2
grep span gpurun_out/trace_c.txt
