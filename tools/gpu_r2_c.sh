timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
tail -n 25 gpurun_out/pytest_gpu.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_c.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms']); print(json.dumps(d.get('more'), indent=0)[:2500])"
tail -n 5 gpurun_out/bench_c.err
