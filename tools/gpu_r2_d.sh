timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
timeout 300 python tools/host_split.py > gpurun_out/host_split_d.txt 2>&1
timeout 300 python tools/trace_step.py > gpurun_out/trace_d.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_d.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_d.txt
tail -n 3 gpurun_out/pytest_d.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_d.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
tail -n 3 gpurun_out/bench_d.err
tail -1 gpurun_out/host_split_d.txt
grep span gpurun_out/trace_d.txt
