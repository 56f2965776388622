"""GPU timeline of one bench step via torch.profiler (CUPTI): every kernel /
memcpy / memset with start and duration, plus the idle gaps between them on
the device -- where host overhead and synchronisations cost time.

    python tools/trace_step.py [--scale 1.0] > gpurun_out/trace.txt
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2502_19790_b200 import synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--layout", default="tuples", choices=["tuples", "columns"])
    ap.add_argument("--cprofile", action="store_true", help="host Python profile of 20 steps instead")
    ap.add_argument("--cfg1r1", action="store_true", help="trace the iid cfg1 job instead of cfg2")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    if args.cfg1r1:  # iid 1M-sample cfg1 (long chunks, ~1000 ranges each)
        from paper_2502_19790_b200 import DeviceCatalog

        dcat = DeviceCatalog(synth.expand_numpy(synth.config("cfg1", layout_r=1)))
        spec = synth.cfg1_mixtures()["disjoint"]
    else:
        rt = bench.make_workload(0, args.scale)
        meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
        cols, table = bench.layout_columns(rt, bench.device_columns(rt, dev), args.layout)
        spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
        dcat = bench.device_catalog(meta, cols, table)
    for _ in range(3):
        bench.run_step(dcat, spec)
    torch.cuda.synchronize()
    if args.cprofile:
        import cProfile
        import pstats

        pr = cProfile.Profile()
        pr.enable()
        for _ in range(20):
            bench.run_step(dcat, spec)
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(30)
        return
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        idx, gen, batch = bench.run_step(dcat, spec)
        torch.cuda.synchronize()
    prof.export_chrome_trace(args.out)
    ev = json.load(open(args.out))["traceEvents"]
    gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    gpu.sort(key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    end = t0
    busy = 0.0
    print(f"{'start_us':>9} {'dur_us':>8} {'gap_us':>8}  name")
    for e in gpu:
        gap = e["ts"] - end
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} {gap:8.1f}  {e['cat'][:6]} {e['name'][:70]}")
        busy += e["dur"]
        end = max(end, e["ts"] + e["dur"])
    span = end - t0
    print(f"span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")
    # host-side API calls that block (syncs) in the same window
    cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
    agg = {}
    for e in cpu:
        a = agg.setdefault(e["name"], [0, 0.0])
        a[0] += 1
        a[1] += e["dur"]
    for k, (n, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
        print(f"runtime {k[:40]:40s} n={n:4d} total_us={d:9.1f}")
    print("host runtime calls >= 15 us (start relative to the first GPU op):")
    for e in sorted(cpu, key=lambda e: e["ts"]):
        if e["dur"] >= 15:
            print(f"  {e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['name']}")


if __name__ == "__main__":
    main()
