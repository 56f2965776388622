"""Probe BASELINE configs 4 (ADO latency) and 5 (VLM, ~10k keys) on the GPU.

    python tools/cfg_probe.py cfg5 [--scale 1.0] [--chunks 2000]
    python tools/cfg_probe.py cfg4 [--steps 300]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def cfg5(scale: float, chunks: int):
    import torch

    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, MixtureSpec, build_index_from_catalog, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    rt = synth.config("cfg5", scale)
    lens = torch.from_numpy(rt.run_lengths()).cuda()
    cols = {p: torch.repeat_interleave(torch.from_numpy(c).cuda(), lens) for p, c in rt.run_codes.items()}
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        idx = build_index_from_catalog(DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols}), [])
        torch.cuda.synchronize()
        t_idx = time.perf_counter() - t
    keys = idx.component_keys()
    rng = np.random.Generator(np.random.PCG64(55))
    w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
    w = w[rng.permutation(len(keys))]
    w = w / w.sum()
    spec = MixtureSpec({k: float(x) for k, x in zip(keys, w)}, 1024)
    t = time.perf_counter()
    gen = ChunkGenerator(idx, 42)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t
    t = time.perf_counter()
    batch = gen.plan_batch(spec, chunks)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t
    print(f"cfg5 scale={scale}: N={rt.n_samples} keys={len(keys)} intervals={idx.n_intervals} "
          f"index {t_idx * 1e3:.2f} ms, generator {t_gen * 1e3:.2f} ms, {batch.n_chunks} chunks in "
          f"{t_plan * 1e3:.1f} ms ({t_plan / max(batch.n_chunks, 1) * 1e6:.1f} us/chunk)")


def cfg4(steps: int):
    import torch

    from paper_2502_19790_b200 import (AdoConfig, AdoSource, AdoState, ChunkGenerator, DeviceCatalog, MixtureKey,
                                       build_index_from_catalog, synth)
    from paper_2502_19790_b200.ado import domain_loss_device

    D = 22
    props = {"domain": [f"d{i:02d}" for i in range(D)]}
    rt = synth.make_runs(20_000_000, 2000, props, 64, seed=4)
    cc = synth.expand_numpy(rt)
    idx = build_index_from_catalog(DeviceCatalog(cc), [])
    dom = [MixtureKey.of({"domain": f"d{i:02d}"}) for i in range(D)]
    rng = np.random.default_rng(4)
    prior = rng.dirichlet(np.ones(D))
    cfg = AdoConfig(fit_start_step=100, refit_every=100, discard_first=10, subsample_every=2)
    src = AdoSource(AdoState(cfg, {k: float(p) for k, p in zip(dom, prior / prior.sum())}), 1024)
    gen = ChunkGenerator(idx, 42)
    T = 131072
    tags = torch.randint(0, D, (T,), dtype=torch.int32, device="cuda")
    t_chunk, t_fb = [], []
    for step in range(1, steps + 1):
        t = time.perf_counter()
        spec = src.current_spec()
        chunk = gen.generate(spec)
        t_chunk.append(time.perf_counter() - t)
        losses = (torch.rand(T, device="cuda") + 2.0 + 5.0 / (step ** 0.3)).float()
        t = time.perf_counter()
        sums, counts = domain_loss_device(losses, tags, D)
        s, c = sums.cpu().numpy(), counts.cpu().numpy()
        src.observe_feedback(step, {dom[i]: (float(s[i]), int(c[i])) for i in range(D)})
        t_fb.append(time.perf_counter() - t)
        assert chunk is not None
    print(f"cfg4: {steps} steps, generate {np.median(t_chunk) * 1e6:.0f} us/chunk (median), "
          f"feedback {np.median(t_fb) * 1e6:.0f} us/step, refits at {src.state.fit_steps[:3]}..., "
          f"max feedback {max(t_fb) * 1e3:.1f} ms")
    # breakdown of one step
    import ctypes as C

    from paper_2502_19790_b200 import MixtureSpec, _lib

    parts = {k: [] for k in ("compute_pi", "spec", "plan", "to_host", "chunk", "feedback")}
    for step in range(steps + 1, steps + 101):
        t = time.perf_counter()
        pi = src.state.compute_pi()
        parts["compute_pi"].append(time.perf_counter() - t)
        t = time.perf_counter()
        spec = MixtureSpec(pi, 1024)
        parts["spec"].append(time.perf_counter() - t)
        t = time.perf_counter()
        n, _, (mkeys, _) = gen._plan(spec, 1)
        parts["plan"].append(time.perf_counter() - t)
        t = time.perf_counter()
        b = gen._result(spec, mkeys, None)
        b.to_host()
        parts["to_host"].append(time.perf_counter() - t)
        t = time.perf_counter()
        b.chunk(0)
        parts["chunk"].append(time.perf_counter() - t)
        gen._next_id += n
        t = time.perf_counter()
        sums, counts = domain_loss_device(losses, tags, D)
        s, c = sums.cpu().numpy(), counts.cpu().numpy()
        src.observe_feedback(step, {dom[i]: (float(s[i]), int(c[i])) for i in range(D)})
        parts["feedback"].append(time.perf_counter() - t)
    print("cfg4 breakdown (median us):", {k: round(np.median(v) * 1e6) for k, v in parts.items()})


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("which")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--chunks", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=300)
    a = ap.parse_args()
    cfg5(a.scale, a.chunks) if a.which == "cfg5" else cfg4(a.steps)
