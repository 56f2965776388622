timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_scan_u16.py tests/test_gpu_rows.py tests/test_gpu_scale.py -x -q > gpurun_out/pytest_h.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_h.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -x -q -k "cfg2 or cfg5 or cfg3" > gpurun_out/pytest_h2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_h2.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
timeout 300 python tools/trace_step.py > gpurun_out/trace_h.txt 2>&1
tail -n 3 gpurun_out/pytest_h.txt gpurun_out/pytest_h2.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_h.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['more']['north_star_1b']['ms_per_job'])"
tail -n 3 gpurun_out/bench_h.err
grep span gpurun_out/trace_h.txt
