"""Benchmark of the Mixtera hot path on B200 (contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], SURVEY.md §8d cfg 2): 100M samples in
10,000 files, 5 int32 property columns (cards 4,5,5,4,5 -> 2,000 component
keys), run layout R=64, static multi-property best-effort mixture, chunk 1024,
job seed 42. Synthetic metadata (seeded run table expanded on the device).
Catalog layout (--layout): "tuples" (default) dictionary-encodes the rows once
at registration into ONE u16 row-tuple code column (200 MB); "columns" keeps
one int32 column per property (2 GB). Both exceed the 126 MB L2, so no L2
flush is needed between steps.

One STEP = the whole job on the device: stage 1 (filter + key pack + runs +
grouping into the ChunkerIndex) + RangeCursor layout + emission of EVERY chunk
of the job (planner + cut + normalise + CSR + seeds). value = samples/s
(N / step time); chunks/s is reported beside it. `e2e` runs the same step
through the public API from PINNED HOST columns (H2D inside the timed region)
and copies the full chunk CSR back (D2H inside). The roofline line is for the
dominant kernel (scan_runs, stage 1's streaming pass), timed with CUDA events
recorded by the library on the launching stream.

--impl reference times the reference's own CPU path -- the unmodified
mixplane package installed under baseline/_ref (filter_intervals ->
build_index -> ChunkGenerator.generate to exhaustion) -- on a bounded slice of
the same workload on the host cores; without baseline/_ref the CPU oracle port
(oracle/oracle.py) stands in and the line says kind "port".

Under torchrun with N > 1 rank r owns its own 100M-sample shard = global files [r*F, (r+1)*F) of ONE N x 100M-sample catalog
(weak scaling, cfg 3 shape; --scaling strong splits a fixed total, default
1B) and the step is the key-partitioned pipeline (run_step): local stage 1,
NCCL all-gather of per-key totals, all-to-all of block rows to the key
owners and of block offsets back, replicated key-level plan, local cut, and
an all-to-all of each chunk range's pieces to its owner rank, which
normalises its chunks; every rank reads its own chunks back (e2e). Step
time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples indexed/sec + chunks/sec (1/2/4/8 B200) vs host-CPU ref; % HBM roofline"
UNIT = "samples/s"
CFG = dict(workload="cfg2: 100M samples, 10k files, 5 props (4,5,5,4,5) -> 2000 keys, R=64, "
                    "static 4-key best-effort mixture, chunk 1024, seed 42",
           n_samples=100_000_000, n_files=10_000, props=5, run_mean=64, chunk_size=1024, job_seed=42,
           l2="inputs (2 GB of columns) exceed the 126 MB L2; no flush needed")
LAYOUT_NOTE = {
    "tuples": "row tuples: one u16 code column (rows dictionary-encoded at registration, 2,000 tuples) + per-query tuple LUT",
    "columns": "one int32 code column per property + per-query per-property LUTs",
}
REF_SAMPLE = 2_000_000  # --impl reference: samples per step (bounded CPU slice, ~5 s through the reference)
CPU_SAMPLE = 10_000_000  # cpu_baseline leg of our arm


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clock + throttle reasons sampled through NVML (the same counters
    nvidia-smi reads) every ~2 ms in a thread while the timed steps run; the
    timed region is only milliseconds long, too short for nvidia-smi -lms."""

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap"}

    def __init__(self, index: int):
        import threading

        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while self._nv is not None and not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                bits = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.reasons.update(n for b, n in self._REASONS.items() if bits & b)
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self) -> dict:
        self._stop.set()
        self._t.join()
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml, 2 ms polling"}


def make_workload(rank: int, scale: float):
    from paper_2502_19790_b200 import synth

    n = int(CFG["n_samples"] * scale)
    f = max(1, int(CFG["n_files"] * scale))
    rt = synth.make_runs(n, f, synth.CFG2_PROPS, CFG["run_mean"], seed=2 + 1000 * rank)
    return rt


def device_columns(rt, device):
    import torch

    lens = torch.from_numpy(rt.run_lengths()).to(device)
    return {p: torch.repeat_interleave(torch.from_numpy(c).to(device), lens) for p, c in rt.run_codes.items()}


def device_catalog(meta, cols, table=None):
    """The catalog over HBM-resident columns (built once per catalog, like the
    reference's registered MetadataCatalog; every job reuses it). With
    `table` (row-tuple layout) `cols` is {"tuples": int32 tuple-code column}."""
    from paper_2502_19790_b200 import DeviceCatalog

    if table is not None:
        return DeviceCatalog(meta, tuples=(cols["tuples"], table), nullable={p: False for p in meta.vocab})
    return DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols})


def layout_columns(rt, cols, layout):
    """(columns dict, tuple table or None) in the requested catalog layout:
    "tuples" dictionary-encodes the rows once at registration (untimed, like
    the reference's value interning) into one int32 row-tuple code column."""
    if layout != "tuples":
        return cols, None
    from paper_2502_19790_b200 import DeviceCatalog

    codes, table = DeviceCatalog.encode_row_tuples_device(cols, [len(rt.vocab[p]) for p in sorted(rt.vocab)])
    return {"tuples": codes}, table


def run_step(dcat, spec, stream=None, shard=None):
    """One job on the device: index + cursor layout + every chunk. Returns
    (index, gen, batch) so callers can read sizes. With `shard` = (file_lo,
    file_ds, file_ids) of the global catalog (N > 1): the key-partitioned
    pipeline (parallel.py) -- local stage 1, all-gather of per-key totals,
    all-to-all of (key, file) block rows to the key owners, which lay out
    their keys' cursor streams and return block offsets (all-to-all), plan
    on the key-level index, local cut of every chunk, all-to-all of each
    chunk range's pieces to its owner, which normalises its chunks
    (parallel.plan_owned). MX_BENCH_MULTI=hybrid selects the file-sharded
    hybrid index + full-piece all-gather of round 1 instead."""
    from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog
    from paper_2502_19790_b200.parallel import build_partitioned_index, build_sharded_index, plan_owned

    if shard is None:
        idx = build_index_from_catalog(dcat, [], stream=stream)
    elif os.environ.get("MX_BENCH_MULTI") == "hybrid":
        idx = build_sharded_index(dcat, [], *shard, stream=stream)
    else:
        idx = build_partitioned_index(dcat, [], *shard, stream=stream)
        gen = ChunkGenerator(idx, CFG["job_seed"], stream=stream)
        return idx, gen, plan_owned(gen, spec, 1 << 40)
    gen = ChunkGenerator(idx, CFG["job_seed"], stream=stream)
    batch = gen.plan_batch(spec, 1 << 40)
    return idx, gen, batch


def cpu_port(n_samples: int, rank: int = 0):
    """Oracle port on a bounded slice of the workload (host cores, 1 thread)."""
    from oracle import oracle as orc
    from paper_2502_19790_b200 import synth

    f = max(1, n_samples // (CFG["n_samples"] // CFG["n_files"]))
    cc = synth.expand_numpy(synth.make_runs(n_samples, f, synth.CFG2_PROPS, CFG["run_mean"], seed=2))
    spec = synth.cfg2_mixture(CFG["chunk_size"])
    w = {orc.as_key(k): v for k, v in spec.weights.items()}
    t0 = time.perf_counter()
    idx = orc.build_index(cc, [])
    gen = orc.OracleGenerator(idx, CFG["job_seed"])
    chunks = 0
    while gen.generate(w, spec.chunk_size, spec.strict) is not None:
        chunks += 1
    dt = time.perf_counter() - t0
    return dt, chunks


def _reference_pkg():
    """The unmodified reference (mixplane) installed under baseline/_ref, or
    None when it is absent (then the oracle port stands in)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mixplane").is_dir():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import mixplane  # noqa: F401
    except Exception:
        return None
    return mixplane


def _reference_catalog(cc):
    """A reference MetadataCatalog holding exactly cc's int32 code columns
    (the columnar _FileStore layout the reference keeps after registration,
    catalog.py:265-275; SURVEY.md §8d "oracle injector")."""
    from mixplane import catalog as rcat

    cat = rcat.MetadataCatalog()
    props = sorted(cc.columns)
    cat._props = {p: rcat.PropertyDef(p, "string", True, False) for p in props}
    cat._vocab = {p: list(cc.vocab[p]) for p in props}
    cat._vocab_idx = {p: {v: i for i, v in enumerate(cc.vocab[p])} for p in props}
    nds = int(cc.file_ds.max()) + 1
    cat._dataset_names = [f"ds{d}" for d in range(nds)]
    cat._dataset_schemas = {d: rcat.PropertySchema([cat._props[p] for p in props]) for d in range(nds)}
    cat._dataset_files = {d: [] for d in range(nds)}
    for i, fid in enumerate(cc.file_ids.tolist()):
        ds = int(cc.file_ds[i])
        a, b = int(cc.file_offsets[i]), int(cc.file_offsets[i + 1])
        store = rcat._FileStore(path=f"/synthetic/{fid}.jsonl", dataset_id=ds, n_samples=b - a, content_hash="0" * 32)
        for p in props:
            store.codes[p] = cc.columns[p][a:b].astype(np.int32).copy()
        cat._files[fid] = store
        cat._dataset_files[ds].append(fid)
    return cat


def reference_prepare(n_samples: int, seed: int = 2):
    """A reference catalog over a bounded slice of the cfg2 layout (registration
    is not timed) and the cfg2 mixture as a reference MixtureSpec."""
    from mixplane.mixtures import MixtureKey as RKey, MixtureSpec as RSpec

    from paper_2502_19790_b200 import synth

    f = max(1, n_samples // (CFG["n_samples"] // CFG["n_files"]))
    cc = synth.expand_numpy(synth.make_runs(n_samples, f, synth.CFG2_PROPS, CFG["run_mean"], seed=seed))
    cat = _reference_catalog(cc)
    spec = synth.cfg2_mixture(CFG["chunk_size"])
    rspec = RSpec({RKey.of({p: list(v) for p, v in k.entries}): w for k, w in spec.weights.items()}, spec.chunk_size)
    return cat, rspec


def reference_job(cat, rspec):
    """The reference's own job: filter_intervals -> build_index ->
    ChunkGenerator.generate until None (server.py:112-163), one thread
    (GIL-bound, build_index workers=1)."""
    from mixplane.chunks import ChunkGenerator as RGen
    from mixplane.index import build_index as rbuild

    t0 = time.perf_counter()
    gen = RGen(rbuild(cat.filter_intervals([])), CFG["job_seed"])
    chunks = 0
    while gen.generate(rspec) is not None:
        chunks += 1
    return time.perf_counter() - t0, chunks


def reference_run(n_samples: int):
    return reference_job(*reference_prepare(n_samples))


def _ref_proc(wid, n_samples, rounds, barrier, q):
    """One host process of the reference arm: its own slice (seed per worker),
    every round started together with the other workers."""
    _reference_pkg()
    cat, rspec = reference_prepare(n_samples, seed=2 + wid)
    for r in range(rounds):
        barrier.wait()
        dt, chunks = reference_job(cat, rspec)
        q.put((wid, r, dt, chunks))


def reference_parallel(n_samples: int, workers: int, warmup: int, steps: int):
    """The reference on `workers` host processes at once (the reference is
    pure Python and GIL-bound, so processes are how it uses the cores): each
    process runs the job on its own n_samples slice; a step's time is the
    slowest worker's. Returns (per-step max times, chunks per worker-job)."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(workers), ctx.Queue()
    procs = [ctx.Process(target=_ref_proc, args=(w, n_samples, warmup + steps, barrier, q), daemon=True)
             for w in range(workers)]
    for pr in procs:
        pr.start()
    res = [q.get() for _ in range(workers * (warmup + steps))]
    for pr in procs:
        pr.join()
    per_round = {}
    for _, r, dt, ch in res:
        per_round.setdefault(r, []).append((dt, ch))
    times = [max(dt for dt, _ in per_round[r]) for r in range(warmup, warmup + steps)]
    chunks = sum(ch for _, ch in per_round[warmup + steps - 1]) / workers
    return times, chunks


def host_workers() -> int:
    """Processes of the reference arm: 1 -- the reference's own path is one
    GIL-bound process (build_index(rows, workers=1), server.py:115).
    MX_REF_WORKERS=k runs k file-slice processes instead (a sharded upper
    bound, labelled as such)."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    cap = int(os.environ.get("MX_REF_WORKERS", "1") or 1)
    return max(1, min(n, cap))


def arm_config(world: int, layout: str) -> dict:
    """The workload description both arms print (identical dicts)."""
    code_bytes, n_cols = (2, 1) if layout == "tuples" else (4, CFG["props"])
    n = CFG["n_samples"] * world
    multi = ("file-sharded hybrid" if os.environ.get("MX_BENCH_MULTI") == "hybrid" else "key-partitioned")
    return dict(CFG, parallelism=f"{multi} x{world}" if world > 1 else "single GPU",
                layout=LAYOUT_NOTE[layout],
                l2=f"inputs ({n * code_bytes * n_cols / 1e9:.1f} GB of code columns) exceed the 126 MB L2; "
                   "no flush needed")


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    real = _reference_pkg() is not None
    workers = host_workers() if real else 1
    if real:
        times, chunks = reference_parallel(REF_SAMPLE, workers, args.warmup, args.steps)
    else:
        for _ in range(args.warmup):
            cpu_port(REF_SAMPLE)
        times, chunks = [], 0
        for _ in range(args.steps):
            dt, chunks = cpu_port(REF_SAMPLE)
            times.append(dt)
    t = sum(times) / len(times)
    v = workers * REF_SAMPLE / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": arm_config(args.gpus, args.layout),
        "chunks_per_s": workers * chunks / t,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "reference" if real else "port",
                         "sample": ((f"the job on the first {REF_SAMPLE:,} samples (200 files) of the cfg2 "
                                     "layout per step, one process (the reference's own path is single-core: "
                                     "GIL-bound, build_index workers=1 at server.py:115), through "
                                     if workers == 1 else
                                     f"SHARDED UPPER BOUND: {workers} host processes at once, each running the job "
                                     f"on its own {REF_SAMPLE:,}-sample slice of the cfg2 layout per step, through ")
                                    if real else f"{REF_SAMPLE:,} samples of the cfg2 layout per step through ")
                                   + ("the unmodified reference (baseline/_ref mixplane: filter_intervals, "
                                      "build_index, ChunkGenerator.generate to exhaustion)"
                                      + ("; step time = the slowest process" if workers > 1 else "")
                                      if real else "oracle/oracle.py (numpy + CPython stdlib), single thread")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def our_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2502_19790_b200 import _lib, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    rank, world, local = env_rank()
    device = torch.device("cuda", local % torch.cuda.device_count() if world > 1 else 0)
    torch.cuda.set_device(device)
    if world > 1:
        # nccl on the real multi-GPU run; MX_BENCH_BACKEND=gloo lets N ranks
        # share one GPU to exercise the same code path
        dist.init_process_group(os.environ.get("MX_BENCH_BACKEND", "nccl"))
    L = _lib.lib()
    strong = args.scaling == "strong"
    # strong scaling: a fixed total (default the cfg3 1B catalog) split over the
    # ranks by file; weak: every rank owns its own 100M-sample shard
    scale = args.total_samples / (world * CFG["n_samples"]) if strong else args.scale
    rt = make_workload(rank, scale)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    if strong and args.layout == "tuples":
        codes, table = run_level_tuples(rt, device)  # no 20 GB int32 expansion at 1B
        cols = {"tuples": codes}
    else:
        cols, table = layout_columns(rt, device_columns(rt, device), args.layout)
    n_cols = len(cols)
    code_bytes = next(iter(cols.values())).element_size()  # 2: u16 row-tuple codes
    spec = synth.cfg2_mixture(CFG["chunk_size"])
    shard = None
    if world > 1:  # rank r owns global files [r*F, (r+1)*F) of one W*F-file catalog
        nf = len(rt.file_sizes)
        shard = (rank * nf, np.zeros(world * nf, np.int32), np.arange(1, world * nf + 1, dtype=np.int64))
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    dcat = device_catalog(meta, cols, table)
    for _ in range(args.warmup):
        idx, gen, batch = run_step(dcat, spec, shard=shard)
        del idx, gen, batch
    barrier()
    # ---------------------------------------------------------------- timed
    L.mx_profile_reset()
    L.mx_profile_enable(2)  # the scan kernel's events only (roofline); phases below
    clocks = Clocks(device.index)
    launches0 = L.mx_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    n_chunks = n_ranges = n_iv = 0
    for _ in range(args.steps):
        idx, gen, batch = run_step(dcat, spec, shard=shard)
        # global chunks (this rank's owned range under the partitioned path)
        n_chunks, n_ranges = getattr(batch, "global_chunks", batch.n_chunks), batch.n_ranges
        part = getattr(idx, "partition", None)
        n_iv = (part.local if part is not None else getattr(idx, "local_index", idx)).n_intervals
        n_keys, n_blocks = idx.n_keys, idx.n_blocks
        del idx, gen, batch
    ev1.record(stream)
    barrier()
    launches = (L.mx_launch_count() - launches0) / args.steps
    clk = clocks.stop()
    L.mx_profile_enable(0)
    ms = ev0.elapsed_time(ev1) / args.steps
    scan_timed = _lib.profile_read("scan_runs")
    # per-phase breakdown: a separate untimed pass with every phase's events
    L.mx_profile_reset()
    L.mx_profile_enable(1)
    for _ in range(min(args.steps, 5)):
        run_step(dcat, spec, shard=shard)
    L.mx_profile_enable(0)
    phases = {p: _lib.profile_read(p) for p in ("scan_runs", "radix_sort", "index_scans", "cursor_layout",
                                                 "cursor_shuffle", "plan", "emit")}
    phases["scan_runs"] = scan_timed
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    n = rt.n_samples
    # ------------------------------------------------------------ two jobs in flight
    # (the reference server runs one thread per job): 2 host threads, 2 streams
    concurrent = None
    if world == 1 and args.concurrent:
        import threading

        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        per = max(1, args.steps // 2)

        def worker(st):
            with torch.cuda.stream(st):
                for _ in range(per):
                    i_, g_, b_ = run_step(dcat, spec, stream=st)
                    del i_, g_, b_

        for _ in range(2):  # warm the second stream / thread-local state
            worker(streams[1])
        barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for st in streams:
            st.wait_stream(stream)
        ths = [threading.Thread(target=worker, args=(st,)) for st in streams]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        for st in streams:
            stream.wait_stream(st)
        c1.record(stream)
        barrier()
        cms = c0.elapsed_time(c1) / (2 * per)
        concurrent = {"jobs_in_flight": 2, "jobs": 2 * per, "ms_per_job": cms, "value": n / (cms * 1e-3),
                      "unit": UNIT, "note": "two host threads, one CUDA stream each, the same job repeated; "
                                            "amortised time per job"}
    # ------------------------------------------------------------ e2e (host buffers)
    pinned = {p: c.cpu().pin_memory() for p, c in cols.items()}
    del cols, dcat
    torch.cuda.empty_cache()
    h2d = sum(x.numel() * x.element_size() for x in pinned.values())

    # the catalog is registered once (its device buffers allocated, codec and
    # LUTs built, like the reference's registered MetadataCatalog); every
    # step re-uploads the code columns from pinned host memory into it
    dbufs = {p: torch.empty_like(x, device=device) for p, x in pinned.items()}
    dcat_e2e = device_catalog(meta, dbufs, table)

    def e2e_step():
        for p, x in pinned.items():
            dbufs[p].copy_(x, non_blocking=True)
        idx, gen, batch = run_step(dcat_e2e, spec, shard=shard)
        if rank != 0 and not hasattr(batch, "chunk_lo"):  # hybrid: the merged global chunks are read on the root
            return 0
        h = batch.to_host()  # partitioned: every rank reads back its own chunk range
        return sum(v.nbytes for k, v in h.items() if k in ("off", "ids", "seeds")) + 16 * batch.n_ranges

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    d2h = 0
    for _ in range(args.steps):
        d2h = e2e_step()
    e1.record(stream)
    barrier()
    ems = e0.elapsed_time(e1) / args.steps
    te = torch.tensor([ems], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ems = float(te.item())
    if rank != 0:
        dist.destroy_process_group()
        return
    # ------------------------------------------------------------ roofline
    peak, peak_kind = peaks()
    scan_ms, scan_n = phases["scan_runs"]
    scan_avg = scan_ms / max(scan_n, 1)
    scan_bytes = n * code_bytes * n_cols + 16 * n_iv
    step_bytes = scan_bytes + 8 * n_blocks + 16 * n_keys + 16 * n_iv + 20 * n_ranges + 8 * n_chunks
    achieved = scan_bytes / (scan_avg * 1e-3) / 1e9
    b_per_sample = code_bytes * n_cols
    traffic, prof = None, {}
    tf = ROOT / "profiles" / "scan_traffic.json"
    if tf.exists():
        prof = json.loads(tf.read_text()).get(args.layout, {})
        traffic = prof.get("bytes_per_launch")
    # the u16 single-column scan is issue / latency bound (ncu issue-active,
    # warps active), not HBM bound: say so next to its HBM fraction
    issue = prof.get("issue_active_pct")
    line = {
        "metric": METRIC, "value": world * n / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "u16" if code_bytes == 2 else "int32", "data": "synthetic",
        "config": (dict(arm_config(world, args.layout), workload=f"cfg3 shape: {int(args.total_samples):,} samples "
                        "in total over all ranks (10k per file), cfg2 properties and mixture, R=64, chunk 1024, "
                        "seed 42", n_samples=int(args.total_samples), n_files=int(args.total_samples) // 10_000)
                   if strong else arm_config(world, args.layout)),
        "chunks_per_s": n_chunks / (ms_max * 1e-3),
        "job": {"samples": n, "intervals": n_iv, "keys": n_keys, "blocks": n_blocks, "chunks": n_chunks,
                "ranges": n_ranges},
        "phases_ms": {p: round(v[0] / max(v[1], 1), 4) for p, v in phases.items()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": ("scan_u16_kernel (the scan_runs phase: change-driven warp segments over the u16 row-tuple column)"
                                if code_bytes == 2 else "scan_fast_kernel (the scan_runs phase: scan_fast + "
                                "deferred-tile scan_list + tail scan_direct)"),
                     "bytes_per_launch": scan_bytes, "peak_kind": peak_kind,
                     "note": "algorithmic bytes = N*b*C code-column reads (C = 1 row-tuple column of b = 2-byte codes, or P per-property int32 columns) + 16 B per interval record"
                             + (f"; at {b_per_sample} B/sample this kernel is bound by instruction issue and "
                                f"latency, not HBM (ncu: {issue:.0f}% issue-active at "
                                f"{prof.get('warps_active_pct', 0):.0f}% warps active, "
                                f"{prof.get('inst_executed', 0) / n:.2f} warp instructions per sample)"
                                if issue and code_bytes * n_cols <= 2 else "")},
        # the whole job against the same peak (B1 + B2 per step)
        "roofline_step": {
            "bytes": step_bytes, "achieved": step_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
            "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
            "note": "B1 = N*b*C + 16*I + 8*B + 16*K, B2 = 16*I (intervals touched) + 20*ranges + 8*chunks; "
                    "the gap to the scan's fraction is the latency-bound cursor / plan / emission work and "
                    "the host synchronisations between them"},
        "e2e": {"value": world * n / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": int(d2h), "ms_per_step": ems},
        "gpu_launches": int(launches * args.steps),
        **({"concurrent_jobs": concurrent} if concurrent else {}),
        "clocks": clk,
    }
    if world == 1 and not args.no_extras:
        line["more"] = extra_measurements(args, rt, meta, spec, device)
    if not args.no_cpu_baseline and world == 1:
        real = _reference_pkg() is not None
        if real:
            # the reference arm itself (one step), in a fresh process (no fork
            # of this CUDA-initialised one)
            out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                                  "--warmup", "0"], capture_output=True, text=True, timeout=600)
            ref = json.loads(out.stdout.strip().splitlines()[-1])
            line["cpu_baseline"] = dict(ref["cpu_baseline"], chunks_per_s=ref["chunks_per_s"])
        else:
            dt, chunks = cpu_port(CPU_SAMPLE)
            line["cpu_baseline"] = {
                "value": CPU_SAMPLE / dt, "unit": UNIT, "cores": 1, "kind": "port", "chunks_per_s": chunks / dt,
                "sample": f"first {CPU_SAMPLE:,} samples ({CPU_SAMPLE // 10_000} files) of the cfg2 layout "
                          "through oracle/oracle.py (numpy + CPython stdlib), 1 thread"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _timed_steps(fn, steps, warmup):
    """Device time per call of fn (CUDA events on the current stream)."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def extra_measurements(args, rt, meta, spec, device) -> dict:
    """Secondary lines of the N=1 run (rank 0): what a drop-in user gets.

    * columns_layout: the same job over one int32 code column per property
      (the layout DeviceCatalog.from_reference builds for a reference catalog);
    * registration: the one-time row-tuple dictionary encoding of those
      columns on the device (encode_row_tuples_device), which the headline
      layout needs before its first job;
    * north_star_1b: the cfg3 catalog (1B samples, 100k files, R=64) indexed
      and chunked on ONE B200, u16 row-tuple layout, every chunk emitted;
    * dropin_serving: the whole cfg2 job through the reference seam the
      server calls per chunk (ChunkGenerator.generate + Chunk.serialize,
      server.py:143-163), host wall clock."""
    import torch

    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, _lib, build_index_from_catalog, synth

    out = {}
    steps = max(3, min(args.steps, 10))
    peak, _ = peaks()
    # ---- per-property int32 columns + registration of the tuple layout
    cols = device_columns(rt, device)
    dcat = device_catalog(meta, cols, None)
    cres = {}

    def cjob():
        i_, g_, b_ = run_step(dcat, spec)
        cres["intervals"] = i_.n_intervals

    cjob()
    _lib.lib().mx_profile_reset()
    _lib.lib().mx_profile_enable(2)
    ms = _timed_steps(cjob, steps, 1)
    scan_ms, scan_n = _lib.profile_read("scan_runs")
    _lib.lib().mx_profile_enable(0)
    n = rt.n_samples
    scan_bytes = n * 4 * len(cols) + 16 * cres["intervals"]
    scan_avg = scan_ms / max(scan_n, 1)
    out["columns_layout"] = {
        "ms_per_step": ms, "value": n / (ms * 1e-3), "unit": UNIT,
        "scan_ms": scan_avg, "scan_roofline_frac": scan_bytes / (scan_avg * 1e-3) / 1e9 / peak,
        "note": "one int32 code column per property (2 GB at cfg2): DeviceCatalog.from_reference(cat, "
                "layout='columns'); drop-in catalogs default to the row-tuple layout"}
    cards = [len(rt.vocab[p]) for p in sorted(rt.vocab)]
    enc_ms = _timed_steps(lambda: DeviceCatalog.encode_row_tuples_device(cols, cards), 3, 1)
    out["registration"] = {
        "tuple_encode_ms": enc_ms,
        "note": "row-tuple dictionary encoding of the int32 columns on the device (mixed-radix tuple value + "
                "unique), once per registered catalog; not part of a job"}
    out["registration"]["jsonl"] = jsonl_registration(device)
    del dcat, cols
    torch.cuda.empty_cache()
    # ---- drop-in serving: per-chunk generate() + serialize() for the whole job
    tcols, table = layout_columns(rt, device_columns(rt, device), "tuples")
    dcat = device_catalog(meta, tcols, table)
    idx = build_index_from_catalog(dcat, [])
    for rep in range(2):  # the first pass warms the pinned pools
        gen = ChunkGenerator(idx, CFG["job_seed"])
        t0 = time.perf_counter()
        n_ch = n_bytes = 0
        while (c := gen.generate(spec)) is not None:
            n_bytes += len(c.serialize())
            n_ch += 1
        dt = time.perf_counter() - t0
    out["dropin_serving"] = {
        "chunks": n_ch, "seconds": dt, "chunks_per_s": n_ch / dt, "bytes_per_s": n_bytes / dt,
        "note": "ChunkGenerator.generate(spec) + Chunk.serialize() once per chunk until None, as the reference "
                "server calls them (server.py:143-163); the generator plans ahead on the device (look-ahead "
                "doubling) and chunks carry device-built canonical bytes with a lazy data dict; index built "
                "once, host wall clock"}
    del gen, idx, dcat, tcols
    torch.cuda.empty_cache()
    # ---- north star: 1B samples on one GPU
    big = synth.config("cfg3", scale=args.scale)
    bmeta = synth.ColumnarCatalog.meta_only(big.vocab, big.file_sizes)
    codes, btable = run_level_tuples(big, device)
    bcat = device_catalog(bmeta, {"tuples": codes}, btable)
    res = {}

    def job():
        i_, g_, b_ = run_step(bcat, spec)
        res.update(chunks=b_.n_chunks, ranges=b_.n_ranges, intervals=i_.n_intervals, blocks=i_.n_blocks)

    bms = _timed_steps(job, 3, 1)
    bn = big.n_samples
    b_bytes = bn * 2 + 16 * res["intervals"] + 8 * res["blocks"] + 16 * 2000 + 16 * res["intervals"] + \
        20 * res["ranges"] + 8 * res["chunks"]
    out["north_star_1b"] = {
        "samples": bn, "files": len(big.file_sizes), "ms_per_job": bms, "value": bn / (bms * 1e-3), "unit": UNIT,
        "chunks": res["chunks"], "chunks_per_s": res["chunks"] / (bms * 1e-3), "intervals": res["intervals"],
        "roofline_step": {"bytes": b_bytes, "achieved": b_bytes / (bms * 1e-3) / 1e9, "peak": peak,
                          "frac": b_bytes / (bms * 1e-3) / 1e9 / peak},
        "note": "cfg3 catalog (seed 3) on ONE device, u16 row-tuple column (2 GB), cfg2 mixture, every chunk; "
                "bit-exact vs the oracle in tests/test_gpu_parity_scale.py::test_cfg3_one_billion_samples_one_gpu"}
    del bcat, codes
    torch.cuda.empty_cache()
    return out


REG_SAMPLES, REG_FILES, REF_REG_FILES = 2_000_000, 200, 10


def jsonl_registration(device) -> dict:
    """cfg2-shaped metadata (2M records in 200 JSON-lines
    files, 5 properties + id + text) registered by DeviceMetadataCatalog
    (records, JSON validation and normalised values on the device, interning
    into HBM code columns) vs the reference's MetadataCatalog.register_dataset
    on a 10-file slice of the same files, host wall clock."""
    import tempfile

    import torch

    from paper_2502_19790_b200 import synth
    from paper_2502_19790_b200.register import DeviceMetadataCatalog

    mp = _reference_pkg()
    props = sorted(synth.CFG2_PROPS)
    if mp is not None:
        parser = mp.JsonFieldParser.for_properties(props)
        schema = mp.PropertySchema([mp.PropertyDef(p) for p in props])
    else:
        from types import SimpleNamespace

        parser = SimpleNamespace(fields=tuple((p, p) for p in props))
        schema = SimpleNamespace(properties=tuple(SimpleNamespace(name=p, kind="string", nullable=True, multiple=False,
                                                                  categories=None) for p in props),
                                 names=lambda: list(props))
    rt = synth.make_runs(REG_SAMPLES, REG_FILES, synth.CFG2_PROPS, CFG["run_mean"], seed=2)
    with tempfile.TemporaryDirectory() as td:
        paths = synth.write_jsonl_corpus(rt, td)
        nbytes = sum(p.stat().st_size for p in paths)
        DeviceMetadataCatalog(device).register_dataset("warm", paths, parser, schema)  # pinned staging, kernels
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = DeviceMetadataCatalog(device)
        dev.register_dataset("cfg2", paths, parser, schema)
        torch.cuda.synchronize()
        gpu_s = time.perf_counter() - t0
        out = {"records": rt.n_samples, "files": len(paths), "bytes": nbytes, "seconds": gpu_s,
               "records_per_s": rt.n_samples / gpu_s, "bytes_per_s": nbytes / gpu_s,
               "breakdown_s": dict(dev.timings)}
        if mp is not None:
            sl = paths[:REF_REG_FILES]
            n_ref = int(sum(rt.file_sizes[:REF_REG_FILES]))
            t0 = time.perf_counter()
            mp.MetadataCatalog().register_dataset("cfg2", sl, parser, schema)
            ref_s = time.perf_counter() - t0
            out["reference"] = {"records": n_ref, "seconds": ref_s, "records_per_s": n_ref / ref_s, "cores": 1,
                                "sample": f"first {REF_REG_FILES} files of the same corpus, workers=1"}
    out["note"] = ("device registration of JSON-lines metadata (csrc/register.cu + register.py), host wall clock "
                   "incl. reading the files from the page cache, BLAKE2b content hashes, H2D, JSON validation, "
                   "value extraction, interning and the HBM code columns")
    return out


def run_level_tuples(rt, device):
    """u16 row-tuple column of a run table, encoded at RUN level (every sample
    of a run holds its run's tuple), identical to encode_row_tuples_device on
    the expanded columns without materialising 20 GB of int32 columns."""
    import torch

    from paper_2502_19790_b200.catalog import narrow_codes, row_tuple_table, _tuple_radix

    props = sorted(rt.run_codes)
    cards = [len(rt.vocab[p]) for p in props]
    mult = _tuple_radix(cards)
    r = np.zeros(len(rt.run_starts), dtype=np.int64)
    for p, m in zip(props, mult):
        r += (rt.run_codes[p].astype(np.int64) + 1) * m
    u, inv = np.unique(r, return_inverse=True)
    table = row_tuple_table(u, cards)
    run_codes = torch.from_numpy(narrow_codes(inv.astype(np.int32), len(u))).to(device)
    lens = torch.from_numpy(rt.run_lengths()).to(device)
    return torch.repeat_interleave(run_codes, lens), table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layout", default="tuples", choices=["tuples", "columns"],
                    help="catalog layout in HBM: one row-tuple code column, or one code column per property")
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the cfg2 size (debug only)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): N x 100M samples; strong: --total-samples split over the N ranks")
    ap.add_argument("--total-samples", type=float, default=1e9, help="strong scaling: samples over all ranks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary lines (columns layout, registration, 1B job, drop-in serving)")
    ap.add_argument("--concurrent", action="store_true",
                    help="also time two jobs in flight (two host threads, two streams); diagnostic")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()
