for cfg in "8 1.25" "4 2.5" "2 5"; do
  set -- $cfg
  timeout 900 python tools/shard_sim.py --world $1 --scale $2 > gpurun_out/sim_strong_w$1.json 2> gpurun_out/sim_strong_w$1.err
  tail -c 1500 gpurun_out/sim_strong_w$1.json; echo
done
