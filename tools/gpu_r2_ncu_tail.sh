timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:plan_kernel|cursor_shuffle|radix_downsweep2|emit_write_staged|normalize_warp|component_order|build_segments|match_fill|compact_warp' -s 30 -c 12 -o gpurun_out/tail_r2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tail.log 2>&1
tail -3 gpurun_out/ncu_tail.log
