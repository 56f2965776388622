timeout 900 ncu --set full --clock-control none -k regex:"radix_downsweep2|emit_write_staged_kernel|cursor_shuffle_kernel|plan_kernel|normalize_warp_kernel" -s 5 -c 5 -o gpurun_out/kernels_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_more.log 2>&1
ls -la gpurun_out/kernels_full.ncu-rep
