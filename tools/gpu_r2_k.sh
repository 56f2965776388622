timeout 900 python -m pytest tests/test_gpu_register.py -x -q > gpurun_out/pytest_k.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.txt
tail -n 40 gpurun_out/pytest_k.txt
