mkdir -p gpurun_out
for cfg in "8 1.25" "4 2.5" "2 5" "1 10"; do
  set -- $cfg
  timeout 900 python tools/partition_sim.py --world $1 --scale $2 > gpurun_out/psim_w$1.json 2> gpurun_out/psim_w$1.err
  cat gpurun_out/psim_w$1.json; tail -3 gpurun_out/psim_w$1.err; echo
done
