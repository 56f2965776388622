for e in "X=1" "MX_RADIX=direct" "MX_RADIX_ITEMS=16" "MX_EMIT_DIRECT=1" "MX_NORM_NOPACK=1" "X=2"; do
  echo "$e $(env $e timeout 300 python tools/bench_configs.py --only cfg1 2>/dev/null | head -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["cfg1_R1"]["gpu_ms_per_job"])')" >> gpurun_out/cfg1ab.txt
done
cat gpurun_out/cfg1ab.txt
