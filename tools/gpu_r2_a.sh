timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_planner.py tests/test_gpu_dropin.py tests/test_gpu_json.py tests/test_gpu_scan_u16.py -x -q > gpurun_out/pytest_a.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_a.txt
timeout 600 python -m pytest tests/test_gpu_parity_scale.py -x -q -k "cfg2_full" > gpurun_out/pytest_a2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_a2.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
timeout 300 python tools/trace_step.py > gpurun_out/trace_a.txt 2>&1
tail -n 3 gpurun_out/pytest_a.txt gpurun_out/pytest_a2.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_a.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'])"
tail -n 3 gpurun_out/bench_a.err
grep span gpurun_out/trace_a.txt
