for b in 1184 592 296 2368; do
  MX_EF_BLOCKS=$b timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_g$b.json 2> /dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/bench_g$b.json').read().strip().splitlines()[-1])
print($b, d['ms_per_step'], d['phases_ms']['emit'])"
done
MX_EMIT_OLD=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_gold.json 2> /dev/null
python -c "
import json;d=json.loads(open('gpurun_out/bench_gold.json').read().strip().splitlines()[-1])
print('old', d['ms_per_step'], d['phases_ms']['emit'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:place_fused --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -3
