timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_scale.py tests/test_gpu_json.py tests/test_gpu_planner.py -x -q > gpurun_out/pytest_f.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_f.txt
timeout 600 python -m pytest tests/test_gpu_parity_scale.py -x -q -k "cfg2" > gpurun_out/pytest_f2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_f2.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
timeout 300 python tools/trace_step.py > gpurun_out/trace_f.txt 2>&1
tail -n 3 gpurun_out/pytest_f.txt gpurun_out/pytest_f2.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_f.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
tail -n 3 gpurun_out/bench_f.err
grep span gpurun_out/trace_f.txt
