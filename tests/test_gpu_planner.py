"""GPU: the cooperative many-key planner (plan_big_kernel, > 256 mixture keys)
against the serial single-thread planner (MX_PLAN_SERIAL=1), which the golden
cases pin to the reference. cfg5_wide (tests/golden) pins the cooperative
planner to the reference directly; this covers more keys, ties and strict."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wide_index():
    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog, synth

    rt = synth.make_runs(1_500_000, 48, synth.numbered_props((10, 12, 16), ["caption_len", "dataset", "resolution"]),
                         16, seed=9, zipf=1.05)
    idx = build_index_from_catalog(DeviceCatalog(synth.expand_numpy(rt)), [])
    assert len(idx.component_keys()) > 1000
    return idx


def _chunks(idx, spec, n, serial):
    from paper_2502_19790_b200 import ChunkGenerator

    old = os.environ.pop("MX_PLAN_SERIAL", None)
    if serial:
        os.environ["MX_PLAN_SERIAL"] = "1"
    try:
        gen = ChunkGenerator(idx, 42)
        out = []
        while len(out) < n:
            c = gen.generate(spec)
            if c is None:
                break
            out.append(c.serialize())
        return out, gen.state_dict(), gen.last_report
    finally:
        os.environ.pop("MX_PLAN_SERIAL", None)
        if old is not None:
            os.environ["MX_PLAN_SERIAL"] = old


def _zipf(keys, seed, s=0.8):
    rng = np.random.Generator(np.random.PCG64(seed))
    w = 1.0 / np.arange(1, len(keys) + 1) ** s
    w = w[rng.permutation(len(keys))]
    w = w / w.sum()
    return {k: float(x) for k, x in zip(keys, w)}


@pytest.mark.parametrize("kind", ["zipf", "uniform", "subset", "strict", "two_level"])
def test_cooperative_planner_equals_serial(wide_index, kind):
    from paper_2502_19790_b200 import MixtureSpec

    keys = wide_index.component_keys()
    if kind == "zipf":
        spec = MixtureSpec(_zipf(keys, 1), 1024)
    elif kind == "uniform":  # every share ties: leftovers by key order
        spec = MixtureSpec({k: 1.0 / len(keys) for k in keys}, 3000)
    elif kind == "subset":
        sub = keys[::3]
        spec = MixtureSpec({k: 1.0 / len(sub) for k in sub}, 777)
    elif kind == "strict":
        spec = MixtureSpec({k: 1.0 / len(keys) for k in keys}, 4096, True)
    else:  # two weight levels: big shortfalls hit the exact cooperative apportion
        w = {k: (500.0 if i % 97 == 0 else 1.0) for i, k in enumerate(keys)}
        tot = sum(w.values())
        spec = MixtureSpec({k: v / tot for k, v in w.items()}, 2048)
    a, st_a, rep_a = _chunks(wide_index, spec, 25, serial=False)
    b, st_b, rep_b = _chunks(wide_index, spec, 25, serial=True)
    assert len(a) == len(b)
    for i, (x, y) in enumerate(zip(a, b)):
        assert x == y, f"{kind} chunk {i}"
    assert st_a == st_b
    assert rep_a == rep_b


def test_cooperative_bulk_plan_to_exhaustion(wide_index):
    """plan_batch over the whole stream equals chunk-by-chunk generate()."""
    from paper_2502_19790_b200 import ChunkGenerator, MixtureSpec

    keys = wide_index.component_keys()
    spec = MixtureSpec(_zipf(keys, 2), 4096)
    gen = ChunkGenerator(wide_index, 7)
    batch = gen.plan_batch(spec, 100_000)
    assert batch.n_chunks > 100
    seq, _, _ = _chunks_seeded(wide_index, spec, 7, limit=batch.n_chunks + 1)
    assert len(seq) == batch.n_chunks
    for i in (0, 1, batch.n_chunks // 2, batch.n_chunks - 1):
        c = batch.chunk(i)
        c.mixture = spec
        assert c.serialize() == seq[i], i


def _chunks_seeded(idx, spec, seed, limit):
    from paper_2502_19790_b200 import ChunkGenerator

    gen = ChunkGenerator(idx, seed)
    out = []
    while len(out) < limit:
        c = gen.generate(spec)
        if c is None:
            break
        out.append(c.serialize())
    return out, gen.state_dict(), gen.last_report
