# round-2 profile pass: bench line, launch list, ncu --set full of the step's kernels
timeout 900 python bench.py --steps 10 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/r2_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:scan_u16|radix_downsweep2|plan_fused|cursor_shuffle|component_order|emit_write_staged|normalize_warp|compact_warp|emit_count|gs_apply|key_seed|chunk_seed' -s 40 -c 16 -o gpurun_out/r2_kernels python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r2_ncu_full.log 2>&1
timeout 300 python tools/trace_step.py > gpurun_out/r2_trace.txt 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'))"
tail -3 gpurun_out/r2_ncu_full.log
