mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cursor_shuffle -s 2 -c 1 -o gpurun_out/shuf_src python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_shuf.log 2>&1
ncu -i gpurun_out/shuf_src.ncu-rep --page source --csv --print-source sass > gpurun_out/shuf_sass.csv 2>&1
ncu -i gpurun_out/shuf_src.ncu-rep --page raw --csv > gpurun_out/shuf_raw.csv 2>&1
ls -la gpurun_out/shuf_*
