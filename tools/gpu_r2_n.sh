timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_scale.py tests/test_gpu_json.py tests/test_gpu_planner.py tests/test_gpu_dropin.py tests/test_gpu_parity_scale.py -x -q > gpurun_out/pytest_n.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 --no-extras > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err
timeout 300 python tools/trace_step.py > gpurun_out/trace_n.txt 2>&1
tail -n 3 gpurun_out/pytest_n.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_n.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
grep span gpurun_out/trace_n.txt
