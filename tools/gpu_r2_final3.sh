# round-2 final evidence: full GPU suite, smoke, bench lines (ours + reference arm),
# launch list of one bench run, ncu --set full of the scan and cursor kernels
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/final/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:scan_u16_kernel|cursor_shuffle|key_mt_seed|component_order' -s 8 -c 4 -o gpurun_out/final/kernels_full python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/final/ncu_full.log 2>&1
ncu -i gpurun_out/final/kernels_full.ncu-rep --page raw --csv > gpurun_out/final/kernels_raw.csv 2>&1
rm -f gpurun_out/final/kernels_full.ncu-rep
tail -3 gpurun_out/final/pytest_gpu.txt; tail -1 gpurun_out/final/smoke.txt; head -c 300 gpurun_out/final/bench.json
