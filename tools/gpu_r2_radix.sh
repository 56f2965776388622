ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"radix_downsweep" --csv --log-file gpurun_out/lr.csv python bench.py --scaling strong --steps 2 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2>&1
python - <<PY
import csv, io
txt=open("gpurun_out/lr.csv").read()
lines=[l for l in txt.splitlines() if l.startswith(chr(34))]
rows=list(csv.reader(io.StringIO(chr(10).join(lines))))
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
print("downsweeps 1B:", [r[vi] for r in rows[1:]][-4:])
PY
python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phases_ms']['radix_sort'])"
