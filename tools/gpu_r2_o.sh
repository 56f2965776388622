timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_o.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_o.txt
MX_HOST_TIMING=1 timeout 300 python tools/host_split.py > gpurun_out/host_o.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err
tail -n 3 gpurun_out/pytest_o.txt; tail -n 23 gpurun_out/host_o.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_o.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['more']['north_star_1b']['ms_per_job'], d['more']['columns_layout']['ms_per_step'])"
tail -n 3 gpurun_out/bench_o.err
