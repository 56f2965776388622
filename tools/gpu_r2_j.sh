timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_json.py -x -q > gpurun_out/pytest_j.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_j.txt
tail -n 15 gpurun_out/pytest_j.txt
