"""Per-rank device cost of the file-sharded pipeline at N ranks, on ONE GPU.

Builds the N ranks' local indexes (bench workload, 100M samples each at
--scale 1), then replays every rank's hybrid build, generator, plan and the
root merge sequentially, timing each with CUDA events. Collectives are
replaced by in-memory concatenation (their NVLink cost is estimated from the
bytes printed). Usage: python tools/shard_sim.py --world 8 [--scale 1.0]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, _lib, build_index_from_catalog, synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402
from paper_2502_19790_b200.parallel import hybrid_index  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b), (time.perf_counter() - t0) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--ranks", default="0", help="comma list of ranks to time (all are run)")
    ap.add_argument("--layout", default="tuples", choices=["tuples", "columns"])
    ap.add_argument("--trace", action="store_true", help="CUPTI kernel summary of rank 0's hybrid+gen+plan")
    args = ap.parse_args()
    W = args.world
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    L = _lib.lib()
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    locs = []
    for q in range(W):
        rt = bench.make_workload(q, args.scale)
        meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
        cols, table = bench.layout_columns(rt, bench.device_columns(rt, dev), args.layout)
        dcat = bench.device_catalog(meta, cols, table)
        idx, ms, _ = timed(lambda: build_index_from_catalog(dcat, []))
        nf = len(rt.file_sizes)
        rows = torch.empty((max(idx.n_blocks, 1), 4), dtype=torch.int32, device=dev)
        _lib.check(L.mx_index_block_table(idx.handle, q * nf, rows.data_ptr(), C.c_void_p(_lib.stream_ptr())))
        packed = np.zeros(idx.n_keys, np.uint32)
        _lib.check(L.mx_index_packed_keys(idx.handle, _lib.ptr(packed)))
        if dcat.columns is not None:  # free the code columns
            dcat.columns = {p: c[:0] for p, c in dcat.columns.items()}
        else:
            dcat.tuple_codes = dcat.tuple_codes[:0]
        del cols
        locs.append(dict(idx=idx, dcat=dcat, rows=rows[: idx.n_blocks], packed=packed, nf=nf, stage1_ms=ms))
        torch.cuda.empty_cache()
    counts = [len(x["rows"]) for x in locs]
    cap = max(counts)
    tables = torch.zeros((W, cap, 4), dtype=torch.int32, device=dev)
    for q, x in enumerate(locs):
        tables[q, : counts[q]] = x["rows"]
    gkeys = np.unique(np.concatenate([x["packed"] for x in locs])).astype(np.uint32)
    nf = locs[0]["nf"]
    file_ds, file_ids = np.zeros(W * nf, np.int32), np.arange(1, W * nf + 1, dtype=np.int64)
    report = {"world": W, "layout": args.layout, "samples_per_rank": int(locs[0]["idx"].n_samples), "block_rows": counts,
              "table_allgather_bytes": int(W * cap * 16), "stage1_ms": [round(x["stage1_ms"], 3) for x in locs]}
    timed_ranks = {int(r) for r in args.ranks.split(",")}
    results = []
    per_rank = {}
    prof = None
    # warm-up (first-call costs: side stream, pool growth) on rank 0, untimed
    x = locs[0]
    hyb = hybrid_index(x["idx"], x["dcat"], tables, counts, gkeys, 0, file_ds, file_ids, W, 0)
    del hyb.shard
    gen = ChunkGenerator(hyb, bench.CFG["job_seed"])
    gen.plan_batch(spec, 1 << 40)
    del gen, hyb
    torch.cuda.synchronize()
    for r, x in enumerate(locs):
        if args.trace and r == 0:
            from torch.profiler import ProfilerActivity, profile

            prof = profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU])
            prof.__enter__()
        L.mx_profile_reset()
        L.mx_profile_enable(1)
        hyb, t_h, _ = timed(lambda: hybrid_index(x["idx"], x["dcat"], tables, counts, gkeys, r * nf, file_ds,
                                                  file_ids, W, r))
        del hyb.shard  # no collectives here: keep the local result
        gen, t_g, _ = timed(lambda: ChunkGenerator(hyb, bench.CFG["job_seed"]))
        batch, t_p, _ = timed(lambda: gen.plan_batch(spec, 1 << 40))
        L.mx_profile_enable(0)
        phases = {p: round(_lib.profile_read(p)[0], 4) for p in ("index_scans", "cursor_layout", "cursor_shuffle",
                                                                 "plan", "emit")}
        n, rr = batch.n_chunks, batch.n_ranges
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        cols4 = torch.empty((4, max(rr, 1)), dtype=torch.int32, device=dev)
        _lib.check(L.mx_gen_result_export(gen._h, off.data_ptr(), *(cols4[f].data_ptr() for f in range(4)),
                                          C.c_void_p(_lib.stream_ptr())))
        results.append((off, cols4[:, :rr], rr))
        if prof is not None and r == 0:
            torch.cuda.synchronize()
            prof.__exit__(None, None, None)
            agg = {}
            for e in prof.events():
                if e.device_type.name == "CUDA":
                    a = agg.setdefault(e.name[:60], [0, 0.0])
                    a[0] += 1
                    a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            for k, (n_, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
                print(f"  {us:9.1f} us  x{n_:3d}  {k}", file=sys.stderr)
            prof.export_chrome_trace("/tmp/sim_trace.json")
            ev = json.load(open("/tmp/sim_trace.json"))["traceEvents"]
            gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
                         key=lambda e: e["ts"])
            end = gpu[0]["ts"]
            t0 = end
            for e in gpu:
                gap = e["ts"] - end
                if gap > 20:
                    print(f"  gap {gap:8.1f} us before {e['name'][:60]} at {e['ts'] - t0:9.1f}", file=sys.stderr)
                end = max(end, e["ts"] + e["dur"])
            cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime" and e["dur"] > 30]
            for e in sorted(cpu, key=lambda e: e["ts"]):
                print(f"  host {e['name'][:30]} {e['dur']:8.1f} us at {e['ts'] - t0:9.1f}", file=sys.stderr)
            prof = None
        if r in timed_ranks:
            per_rank[r] = {"hybrid_intervals": hyb.n_intervals, "hybrid_ms": round(t_h, 3),
                           "gen_create_ms": round(t_g, 3), "plan_emit_ms": round(t_p, 3), "phases_ms": phases,
                           "chunks": n, "local_pieces": rr}
        del gen, hyb, batch
    report["ranks"] = per_rank
    # root merge of the N local CSRs
    n = results[0][0].numel() - 1
    capr = max(max(x[2] for x in results), 1)
    offs = torch.stack([x[0] for x in results]).contiguous()
    g4 = torch.zeros((4, W, capr), dtype=torch.int32, device=dev)
    for q, (_, c4, rr) in enumerate(results):
        g4[:, q, :rr] = c4
    total = sum(x[2] for x in results)
    out_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.empty((4, max(total, 1)), dtype=torch.int32, device=dev)

    def merge():
        _lib.check(L.mx_chunks_merge(W, n, capr, offs.data_ptr(), *(g4[f].data_ptr() for f in range(4)),
                                     out_off.data_ptr(), *(out[f].data_ptr() for f in range(4)),
                                     C.c_void_p(_lib.stream_ptr())))

    merge()
    _, t_m, _ = timed(merge)
    if args.trace:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as pm:
            merge()
            torch.cuda.synchronize()
        for e in pm.key_averages():
            if e.device_type.name == "CUDA":
                t = getattr(e, "device_time_total", 0) or getattr(e, "cuda_time_total", 0)
                print(f"  merge: {t:9.1f} us  {e.key[:60]}", file=sys.stderr)
    report.update(merge_ms=round(t_m, 3), global_pieces=int(total), pieces_allgather_bytes=int(W * capr * 16),
                  global_chunks=int(n))
    print(json.dumps(report))


if __name__ == "__main__":
    main()
