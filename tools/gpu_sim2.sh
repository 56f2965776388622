for w in 2 4 8; do timeout 900 python tools/shard_sim.py --world $w > gpurun_out/shard_sim_w${w}_final.json 2> gpurun_out/shard_sim_w${w}.err; done
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_n1.json 2>/dev/null
