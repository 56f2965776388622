timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_l.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms']); print(json.dumps(d['more']['registration'], indent=1))"
tail -n 5 gpurun_out/bench_l.err
