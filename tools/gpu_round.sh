#!/bin/bash
# One GPU-box pass: smoke, GPU parity tests, bench (both arms), ncu launch list
# and a full ncu capture of the stage-1 scan kernel. Outputs in gpurun_out/.
set -x
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $O/cpu.txt
python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
[ -n "$SKIP_NCU" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-scan_fast_kernel} -s 1 -c 1 \
  -o $O/prof_top python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/prof_top.log 2>&1
echo done
