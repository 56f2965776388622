"""Measurements of the BASELINE.json configs other than the headline one
(bench.py measures cfg2): device time per job next to the CPU oracle on the
same synthetic inputs (one host thread, like the GIL-bound reference).

  cfg1  1M samples, 2 properties (20 keys), R=1 (iid) and R=64; static 50/50
        mixture, chunk 1024 -- index + cursor layout + every chunk
  cfg4  ADO over 22 domains: per step, 8 ranks x 131,072 tokens reduced by
        domain (per_domain_loss), observe_feedback (refits at 1000, 2000, ...),
        current_spec + generate() of one chunk
  cfg5  100M samples, 3 properties (~10k realized keys, Zipf joint key, R=16),
        best-effort mixture over all keys with shuffled Zipf(0.8) weights

    python tools/bench_configs.py [--only cfg1,cfg4,cfg5] [--ado-steps 2000]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _events():
    import torch

    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _gpu_job(dcat, spec, seed=42):
    from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog

    idx = build_index_from_catalog(dcat, [])
    gen = ChunkGenerator(idx, seed)
    batch = gen.plan_batch(spec, 1 << 40)
    return idx, batch


def _time_gpu(dcat, spec, reps=5):
    import torch

    for _ in range(2):
        _gpu_job(dcat, spec)
    torch.cuda.synchronize()
    a, b = _events()
    a.record()
    for _ in range(reps):
        idx, batch = _gpu_job(dcat, spec)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, idx, batch


def _oracle_job(cc, spec, limit=None):
    from oracle import oracle as orc

    w = {orc.as_key(k): v for k, v in spec.weights.items()}
    t0 = time.perf_counter()
    idx = orc.build_index(cc, [])
    gen = orc.OracleGenerator(idx, 42)
    n = 0
    while (limit is None or n < limit) and gen.generate(w, spec.chunk_size, spec.strict) is not None:
        n += 1
    return time.perf_counter() - t0, n


def cfg1(out):
    from paper_2502_19790_b200 import DeviceCatalog, synth

    spec = synth.cfg1_mixtures()["disjoint"]
    for r in (1, 64):
        cc = synth.expand_numpy(synth.config("cfg1", layout_r=r))
        ms, idx, batch = _time_gpu(DeviceCatalog(cc), spec)
        dt, n = _oracle_job(cc, spec)
        assert n == batch.n_chunks, (n, batch.n_chunks)
        out[f"cfg1_R{r}"] = {
            "samples": cc.n_samples, "intervals": idx.n_intervals, "chunks": batch.n_chunks,
            "gpu_ms_per_job": round(ms, 3), "gpu_samples_per_s": cc.n_samples / ms * 1e3,
            "gpu_chunks_per_s": batch.n_chunks / ms * 1e3,
            "cpu_oracle_s_per_job": round(dt, 3), "cpu_samples_per_s": cc.n_samples / dt,
            "cpu_chunks_per_s": n / dt, "speedup": dt * 1e3 / ms, "cpu_cores": 1,
        }


def cfg5(out):
    import torch

    from paper_2502_19790_b200 import DeviceCatalog, MixtureSpec, build_index_from_catalog, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    import bench

    rt = synth.config("cfg5")
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    dev = torch.device("cuda", 0)
    cols = bench.device_columns(rt, dev)
    dcat = DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols})
    keys = build_index_from_catalog(dcat, []).component_keys()
    rng = np.random.Generator(np.random.PCG64(5))
    w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
    w = w[rng.permutation(len(keys))]
    w = w / w.sum()
    spec = MixtureSpec({k: float(x) for k, x in zip(keys, w)}, 1024)
    # bounded: index + cursor layout + the first N_CHUNKS chunks (the full job
    # has ~97k chunks and thousands of depletion / redistribution events)
    from paper_2502_19790_b200 import ChunkGenerator

    n_chunks = 2000

    def job():
        idx = build_index_from_catalog(dcat, [])
        gen = ChunkGenerator(idx, 42)
        t = _events()
        t[0].record()
        batch = gen.plan_batch(spec, n_chunks)
        t[1].record()
        return idx, batch, t

    job()
    torch.cuda.synchronize()
    a, b = _events()
    a.record()
    idx, batch, t = job()
    b.record()
    torch.cuda.synchronize()
    ms, plan_ms = a.elapsed_time(b), t[0].elapsed_time(t[1])
    # CPU oracle: 1M samples of the same generator, index + first 5 chunks
    small = synth.make_runs(1_000_000, 100, synth.CFG5_PROPS, 16, seed=5, zipf=1.1)
    cc = synth.expand_numpy(small)
    dt, n = _oracle_job(cc, spec, limit=5)
    out["cfg5"] = {
        "samples": rt.n_samples, "keys": idx.n_keys, "intervals": idx.n_intervals,
        "chunks_timed": batch.n_chunks, "gpu_ms_index_plus_chunks": round(ms, 3),
        "gpu_ms_plan_emit": round(plan_ms, 3), "gpu_chunks_per_s": batch.n_chunks / plan_ms * 1e3,
        "gpu_index_samples_per_s": rt.n_samples / max(ms - plan_ms, 1e-6) * 1e3,
        "cpu_oracle_sample": "1M samples (100 files, same generator), index + first 5 chunks",
        "cpu_oracle_s": round(dt, 3), "cpu_chunks_per_s": n / dt, "cpu_cores": 1,
    }


def cfg4(out, steps):
    import torch

    from paper_2502_19790_b200 import (AdoConfig, AdoSource, AdoState, ChunkGenerator, DeviceCatalog, MixtureKey,
                                       build_index_from_catalog, synth)
    from paper_2502_19790_b200.ado import domain_loss_device
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    D, ranks, tok = 22, 8, 131_072
    dom = [f"x{i:02d}" for i in range(D)]
    rt = synth.make_runs(10_000_000, 1000, {"domain": dom}, 64, seed=4)
    cc = synth.expand_numpy(rt)
    idx = build_index_from_catalog(DeviceCatalog(cc), [])
    keys = [MixtureKey.of({"domain": d}) for d in dom]
    prior = np.random.Generator(np.random.PCG64(4)).dirichlet(np.ones(D))
    src = AdoSource(AdoState(AdoConfig(), dict(zip(keys, prior))), 1024)
    gen = ChunkGenerator(idx, 42)
    g = torch.Generator(device="cuda").manual_seed(4)
    dev = torch.device("cuda", 0)
    losses = [torch.rand(tok, device=dev, generator=g) + 1.5 for _ in range(ranks)]
    # single-domain sequences of 2,048 tokens: 64 per rank per step
    tags = [torch.randint(0, D, (tok // 2048,), device=dev, generator=g, dtype=torch.int32).repeat_interleave(2048)
            for _ in range(ranks)]
    torch.cuda.synchronize()
    t_step, t_reduce = [], []
    for step in range(1, steps + 1):
        t0 = time.perf_counter()
        spec = src.current_spec()
        chunk = gen.generate(spec)
        assert chunk is not None
        t1 = time.perf_counter()
        sums = torch.zeros(D, dtype=torch.float64, device=dev)
        counts = torch.zeros(D, dtype=torch.int64, device=dev)
        for r in range(ranks):  # the 8 DP ranks' reductions (all-reduce = sum)
            s_, c_ = domain_loss_device(losses[r], tags[r], D)
            sums += s_
            counts += c_
        hs, hc = sums.cpu().numpy(), counts.cpu().numpy()
        t2 = time.perf_counter()
        src.observe_feedback(step, {keys[i]: (float(hs[i]), int(hc[i])) for i in range(D)})
        t3 = time.perf_counter()
        t_step.append(t3 - t0)
        t_reduce.append(t2 - t1)
    fit_steps = list(src.state.fit_steps)
    st = np.array(t_step) * 1e6
    # one rank's reduction (131,072 tokens, the per-step DP shard), and the
    # streaming rate on 64M tokens (B3 = T x (4 + 4) bytes)
    lat = []
    for _ in range(200):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        domain_loss_device(losses[0], tags[0], D)
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - t0)
    big_l = torch.rand(64 << 20, device=dev, generator=g) + 1.5
    big_t = torch.randint(0, D, ((64 << 20) // 2048,), device=dev, generator=g, dtype=torch.int32)
    big_t = big_t.repeat_interleave(2048)
    rnd_t = torch.randint(0, D, (64 << 20,), device=dev, generator=g, dtype=torch.int32)

    def rate(tg):
        domain_loss_device(big_l, tg, D)
        a, b = _events()
        a.record()
        for _ in range(5):
            domain_loss_device(big_l, tg, D)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 5

    big_ms, rnd_ms = rate(big_t), rate(rnd_t)
    # CPU oracle for the same per-step work (numpy per_domain_loss on 8 x 131k
    # tokens + oracle ADO + oracle chunk generation), a bounded sample of steps
    from oracle import oracle as orc

    oidx = orc.build_index(cc, [])
    ogen = orc.OracleGenerator(oidx, 42)
    ado = orc.OracleAdo(list(prior))
    hl = [x.cpu().numpy() for x in losses]
    ht = [x.cpu().numpy() for x in tags]
    osteps = min(steps, 200)
    t0 = time.perf_counter()
    for step in range(1, osteps + 1):
        pi = ado.compute_pi()
        ogen.generate({orc.as_key(k): float(p) for k, p in zip(keys, pi)}, 1024, False)
        s = np.zeros(D)
        c = np.zeros(D, np.int64)
        for r in range(ranks):
            s_, c_ = orc.per_domain_loss_np(hl[r], ht[r], D)
            s += s_
            c += c_
        ado.observe(step, s, c)
    cpu_us = (time.perf_counter() - t0) / osteps * 1e6
    out["cfg4"] = {
        "domains": D, "tokens_per_step": ranks * tok, "steps": steps, "fit_steps": fit_steps,
        "gpu_us_per_step_median": float(np.median(st)), "gpu_us_per_step_mean": float(st.mean()),
        "gpu_us_per_refit_step_max": float(st.max()),
        "gpu_8rank_reduce_us_median": float(np.median(np.array(t_reduce) * 1e6)),
        "gpu_one_rank_reduce_us_median": float(np.median(lat) * 1e6),
        "gpu_64M_tokens_ms": big_ms, "gpu_64M_tokens_per_s": (64 << 20) / big_ms * 1e3,
        "gpu_64M_gbs": (64 << 20) * 8 / big_ms / 1e6, "gpu_64M_random_tags_ms": rnd_ms,
        "tags": "single-domain sequences of 2,048 tokens (random per-token tags: gpu_64M_random_tags_ms)",
        "cpu_oracle_us_per_step": cpu_us, "cpu_oracle_steps": osteps, "cpu_cores": 1,
        "note": "host wall clock per step incl. the device syncs of the API (one chunk per step is latency-bound)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg4,cfg5")
    ap.add_argument("--ado-steps", type=int, default=2000)
    args = ap.parse_args()
    todo = args.only.split(",")
    for name in todo:  # one JSON line per config, flushed as it completes
        out = {}
        t0 = time.perf_counter()
        {"cfg1": lambda: cfg1(out), "cfg4": lambda: cfg4(out, args.ado_steps), "cfg5": lambda: cfg5(out)}[name]()
        for k, v in out.items():
            v["wall_s"] = round(time.perf_counter() - t0, 1)
            print(json.dumps({k: v}), flush=True)


if __name__ == "__main__":
    main()
