timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 300 python tools/trace_step.py > gpurun_out/trace_b.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_b.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.txt
tail -n 5 gpurun_out/pytest_b.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_b.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
tail -n 3 gpurun_out/bench_b.err
grep span gpurun_out/trace_b.txt
