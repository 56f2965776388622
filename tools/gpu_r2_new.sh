timeout 600 python -m pytest tests/test_gpu_rows.py -x -q > gpurun_out/pytest_rows.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_rows.txt
timeout 1200 python -m pytest tests/test_gpu_reference_suite.py -q > gpurun_out/pytest_refsuite.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_refsuite.txt
timeout 1800 python -m pytest tests/test_gpu_parity_scale.py -q --durations=0 > gpurun_out/pytest_scale.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_scale.txt
tail -3 gpurun_out/pytest_rows.txt gpurun_out/pytest_refsuite.txt gpurun_out/pytest_scale.txt
