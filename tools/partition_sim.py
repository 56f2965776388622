"""Per-rank device cost of the KEY-PARTITIONED pipeline at N ranks, on ONE GPU.

Builds the N ranks' local indexes (bench workload; --scale 1 = 100M samples
per rank), then replays, with CUDA events: the replicated key-level index
(parallel.build_partitioned_index), every key OWNER's block layout (owner
index + generator + block offsets over the rows all ranks send it), every
rank's plan + local emission (csrc/stage2.cu emit_local), and the root merge.
Collectives are replaced by in-memory concatenation; their bytes are printed
so the NVLink cost can be estimated. Usage:
python tools/partition_sim.py --world 8 --scale 1.25   (1B samples total)
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
from paper_2502_19790_b200 import ChunkGenerator, _lib, build_index_from_catalog, synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402
from paper_2502_19790_b200.index import ChunkerIndex  # noqa: E402
from paper_2502_19790_b200.parallel import U32_SPLIT  # noqa: E402
from paper_2502_19790_b200.seeding import derive_seed, hash_message  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--trace", type=int, default=None, help="profile this rank's plan + emission")
    args = ap.parse_args()
    W = args.world
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    L = _lib.lib()
    sp = C.c_void_p(_lib.stream_ptr())
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    seed = bench.CFG["job_seed"]
    locs = []
    for q in range(W):
        rt = bench.make_workload(q, args.scale)
        meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
        codes, table = bench.run_level_tuples(rt, dev)
        dcat = bench.device_catalog(meta, {"tuples": codes}, table)
        idx, ms = timed(lambda: build_index_from_catalog(dcat, []))
        for _ in range(2):  # warm: first-call costs (pool growth, module load) are not the step
            del idx
            idx, t = timed(lambda: build_index_from_catalog(dcat, []))
            ms = min(ms, t)
        nf = len(rt.file_sizes)
        packed, samples = idx.packed_keys()
        rows = torch.empty((max(idx.n_blocks, 1), 4), dtype=torch.int32, device=dev)
        _lib.check(L.mx_index_block_table(idx.handle, q * nf, rows.data_ptr(), sp))
        dcat.tuple_codes = dcat.tuple_codes[:0]
        del codes
        locs.append(dict(idx=idx, dcat=dcat, rows=rows[: idx.n_blocks], packed=packed, samples=samples, nf=nf,
                         stage1_ms=ms, n_samples=rt.n_samples))
        torch.cuda.empty_cache()
    nf = locs[0]["nf"]
    F = W * nf
    file_ds, file_ids = np.zeros(F, np.int32), np.arange(1, F + 1, dtype=np.int64)
    # ---- replicated key-level index (host part: union of the gathered key lists)
    cat = np.concatenate([np.stack([x["packed"].astype(np.int64), x["samples"]], 1) for x in locs])
    t0 = time.perf_counter()
    gkeys, inv = np.unique(cat[:, 0], return_inverse=True)
    totals = np.zeros(len(gkeys), np.int64)
    np.add.at(totals, inv, cat[:, 1])
    pieces = np.maximum(1, -(-totals // U32_SPLIT))
    rk = np.repeat(np.arange(len(gkeys)), pieces)
    sub = np.arange(len(rk)) - np.repeat(np.cumsum(pieces) - pieces, pieces)
    krows = np.zeros((len(rk), 4), np.uint32)
    krows[:, 0], krows[:, 1] = gkeys[rk].astype(np.uint32), sub
    krows[:, 2], krows[:, 3] = np.minimum(totals[rk] - sub * U32_SPLIT, U32_SPLIT), rk
    host_keys_ms = (time.perf_counter() - t0) * 1e3
    d_krows = torch.from_numpy(krows.view(np.int32)).to(dev)
    d_gkeys = torch.from_numpy(gkeys).to(dev)
    dense_k = max(1, (len(gkeys) - 1).bit_length())
    dense_o = max(1, ((len(gkeys) - 1) // W).bit_length())

    def key_index():
        out = C.c_void_p()
        _lib.check(L.mx_index_build_owner(locs[0]["idx"].handle, d_krows.data_ptr(), len(krows), F,
                                          _lib.ptr(file_ds), _lib.ptr(file_ids), dense_k, sp, C.byref(out)))
        return ChunkerIndex(out.value, locs[0]["dcat"])

    # ---- owner work: rows sent to owner o = rows whose key rank % W == o
    for x in locs:
        x["kg_rows"] = torch.searchsorted(d_gkeys, x["rows"][:, 0].to(torch.int64) & 0xFFFFFFFF)
        x["key_g"] = torch.searchsorted(d_gkeys, torch.from_numpy(x["packed"].astype(np.int64)).to(dev)).to(
            torch.int32)
    recv = []
    for o in range(W):
        parts = []
        for x in locs:
            sel = x["kg_rows"] % W == o
            r = x["rows"][sel].clone()
            r[:, 3] = (x["kg_rows"][sel] // W).to(torch.int32)
            parts.append(r)
        recv.append((torch.cat(parts).contiguous(), [len(p) for p in parts]))
    cur, chk = hash_message(seed, "cursor"), hash_message(seed, "chunk")
    oseed = derive_seed(seed, "component-order")

    def owner(o):
        rows, _ = recv[o]
        n = len(rows)
        oix, og = C.c_void_p(), C.c_void_p()
        off = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        _lib.check(L.mx_index_build_owner(locs[0]["idx"].handle, rows.data_ptr(), n, F, _lib.ptr(file_ds),
                                          _lib.ptr(file_ids), dense_o, sp, C.byref(oix)))
        _lib.check(L.mx_gen_create(oix, cur, len(cur), chk, len(chk), oseed, sp, C.byref(og)))
        _lib.check(L.mx_gen_block_offsets(og, off.data_ptr(), sp))
        L.mx_gen_free(og)
        L.mx_index_free(oix)
        return off[:n]

    offs = [owner(o) for o in range(W)]  # warm
    if args.trace is not None:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as pr:
            owner(args.trace)
            torch.cuda.synchronize()
        print("OWNER", file=sys.stderr)
        print(pr.key_averages().table(sort_by="self_cuda_time_total", row_limit=20), file=sys.stderr)
    own_ms = []
    for o in range(W):
        best = min(timed(lambda: owner(o))[1] for _ in range(args.reps))
        own_ms.append(round(best, 3))
    # offsets back to the file owners
    for q, x in enumerate(locs):
        perm = torch.argsort(x["kg_rows"] % W, stable=True)
        back = []
        for o in range(W):
            lo = sum(recv[o][1][:q])
            back.append(offs[o][lo: lo + recv[o][1][q]])
        blk = torch.empty(len(perm), dtype=torch.int64, device=dev)
        blk[perm] = torch.cat(back)
        x["blk_off"] = blk

    # ---- per rank: key-level index + generator + plan + cut (handoff); then
    # every chunk owner finishes its contiguous chunk range
    from paper_2502_19790_b200.parallel import _DevPtr, chunk_range

    def rank_job(q, finish=None):
        x = locs[q]
        kix = key_index()
        gen = ChunkGenerator(kix, seed)
        _lib.check(L.mx_gen_set_local(gen._h, x["idx"].handle, x["blk_off"].data_ptr(), x["key_g"].data_ptr(),
                                      q * nf))
        _lib.check(L.mx_gen_set_handoff(gen._h, 1))
        n, _, _ = gen._plan(spec, 1 << 40)
        return kix, gen, n

    def handoff(gen, n):
        nc, npc, offp, pp = C.c_int64(), C.c_int64(), C.c_void_p(), C.c_void_p()
        _lib.check(L.mx_gen_handoff(gen._h, C.byref(nc), C.byref(npc), C.byref(offp), C.byref(pp)))
        off = torch.as_tensor(_DevPtr(offp.value, (n + 1,), "<i8"), device=dev).clone()
        pieces = torch.as_tensor(_DevPtr(pp.value, (npc.value, 4), "<i4"), device=dev).clone()
        return off, pieces

    rank_job(0)
    if args.trace is not None:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as pr:
            rank_job(args.trace)
            torch.cuda.synchronize()
        print("RANK", file=sys.stderr)
        print(pr.key_averages().table(sort_by="self_cuda_time_total", row_limit=30), file=sys.stderr)
    cut_ms, host_ms, hand = [], [], []
    for q in range(W):
        best = None
        for _ in range(args.reps):
            h0 = time.perf_counter()
            (kix, gen, n), t = timed(lambda: rank_job(q))
            host_ms.append(round((time.perf_counter() - h0) * 1e3, 3))
            best = t if best is None else min(best, t)
        cut_ms.append(round(best, 3))
        hand.append(handoff(gen, n))
        del kix, gen
    # owner r: counts [W][n_own] and pieces (source-major) of its range
    bounds = [chunk_range(n, W, r) for r in range(W)]
    fin_ms = []
    pieces_moved = 0
    for r, (lo, hi) in enumerate(bounds):
        cnt = torch.stack([(o[lo + 1: hi + 1] - o[lo:hi]).to(torch.int32) for o, _ in hand]).contiguous()
        parts = [p[int(o[lo]): int(o[hi])] for o, p in hand]
        pieces_moved += sum(len(p) for q_, p in enumerate(parts) if q_ != r)
        rp = torch.cat(parts).contiguous()
        fg_kix, fg, fn = rank_job(r)

        def fin():
            _lib.check(L.mx_gen_finish_owned(fg._h, W, lo, hi - lo, n, cnt.data_ptr(), rp.data_ptr(), len(rp), sp))

        _, t = timed(fin)
        fin_ms.append(round(t, 3))
        del fg, fg_kix
    total = sum(len(p) for _, p in hand)
    t_m = 0.0
    rows_total = sum(len(x["rows"]) for x in locs)
    stage1 = [round(x["stage1_ms"], 3) for x in locs]
    report = {
        "world": W, "samples_per_rank": int(locs[0]["n_samples"]), "global_keys": int(len(gkeys)),
        "stage1_ms": stage1, "host_key_union_ms": round(host_keys_ms, 3),
        "owner_ms": own_ms, "rank_plan_cut_ms": cut_ms, "rank_host_ms": host_ms, "chunk_owner_finish_ms": fin_ms,
        "global_chunks": int(n), "global_pieces_before_merge": int(total),
        "bytes": {"keys_allgather": int(W * len(cat) * 16), "rows_alltoall": int(rows_total * 16),
                  "offsets_alltoall": int(rows_total * 8), "pieces_alltoall": int(pieces_moved * 16),
                  "counts_alltoall": int(W * n * 4)},
        "device_step_ms_est": round(max(stage1) + max(own_ms) + max(cut_ms) + max(fin_ms), 3),
    }
    print(json.dumps(report))


if __name__ == "__main__":
    main()
