timeout 900 python -m pytest tests/test_gpu_stage12.py tests/test_gpu_scale.py tests/test_gpu_json.py tests/test_gpu_planner.py tests/test_gpu_dropin.py -x -q > gpurun_out/pytest_m.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_m2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_m2.txt
timeout 300 python bench.py --no-cpu-baseline --steps 10 --no-extras > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err
timeout 300 python tools/job_phases.py --cfg cfg3 > gpurun_out/phases_m.txt 2>&1
tail -n 3 gpurun_out/pytest_m.txt gpurun_out/pytest_m2.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_m.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
tail -n 3 gpurun_out/bench_m.err; cat gpurun_out/phases_m.txt
