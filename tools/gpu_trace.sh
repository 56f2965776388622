timeout 300 python tools/trace_step.py > gpurun_out/trace.txt 2>&1
timeout 300 python tools/trace_step.py --cprofile > gpurun_out/cprofile.txt 2>&1
