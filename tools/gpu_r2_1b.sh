# launch list of one 1B-sample job (strong scaling at N=1)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mx:: -c 120 --csv --log-file gpurun_out/l1b.csv python bench.py --scaling strong --steps 1 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/l1b.log 2>&1
timeout 600 python bench.py --scaling strong --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/b1b.json 2> gpurun_out/b1b.err
head -c 400 gpurun_out/b1b.json
