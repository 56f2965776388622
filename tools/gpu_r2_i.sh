timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "beyond" > gpurun_out/pytest_i.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_i.txt
MX_PLAN_STATS=1 timeout 600 python tools/cfg5_plan.py > gpurun_out/cfg5_plan.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
tail -n 3 gpurun_out/pytest_i.txt
tail -n 20 gpurun_out/cfg5_plan.txt | cut -c1-300
python -c "
import json;d=json.loads(open('gpurun_out/bench_i.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'])"
