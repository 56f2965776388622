"""GPU parity at the BASELINE sizes, bit-exact against the pinned oracle.

* cfg 2 (the bench workload: 100M samples, 10k files, 5 props, R=64), built
  exactly as ``bench.py`` builds it -- u16 row-tuple layout -- and again in the
  per-property int32 columns layout: the full interval table and EVERY chunk
  of the job (83,006) against the oracle's digests (``tests/golden/
  digests.json``, made by ``make_digests.py`` from ``oracle/oracle.py``),
  compared as per-1024-chunk blake2b digests of the canonical chunk bytes,
  plus the shortfall report and the final cursor state;
* the iid (R=1) cfg 2 variant on a 10M-sample slice, every chunk;
* cfg 5 (10k Zipf keys, R=16, best-effort over all keys): the index and the
  first 2,000 chunks;
* cfg 3's 1B-sample catalog on ONE device (the north-star job), when its
  digest exists;
* cfg 4 (ADO, 22 domains, 8 DP ranks x 131,072 tokens per step, 2,100 steps):
  pi within 1e-5 relative of the oracle at every step;
* the device ``apportion`` (plan_kernel / plan_big_kernel): 10,000 random
  (weights, total) through single-chunk strict plans vs the reference's
  ``apportion`` (``mixtures.py:158-184``) and the oracle's.
"""

from __future__ import annotations

import hashlib
import json
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

sys.path.insert(0, str(GOLDEN))
from digests import blob_digest, index_digest  # noqa: E402

DIGESTS = json.loads((GOLDEN / "digests.json").read_text()) if (GOLDEN / "digests.json").exists() else {}


def _need(case):
    if case not in DIGESTS:
        pytest.skip(f"no digest for {case} (tests/golden/make_digests.py {case})")
    return DIGESTS[case]


def _catalog(rt, layout):
    """The bench's own construction (bench.py: device_columns ->
    layout_columns -> device_catalog)."""
    import torch

    import bench
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    dev = torch.device("cuda", 0)
    cols = bench.device_columns(rt, dev)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    lcols, table = bench.layout_columns(rt, cols, layout)
    del cols
    return bench.device_catalog(meta, lcols, table)


def _check_index(idx, want):
    t = idx.interval_table()
    ks = [k.canonical_string() for k in idx.component_keys()]
    assert idx.n_intervals == want["intervals"]
    assert len(ks) == want["keys"]
    assert idx.n_samples == want["samples"]
    assert index_digest(ks, t["key"], t["ds"], t["fid"], t["start"], t["end"]) == want["index_sha256"]


def _check_chunks(gen, batch, want):
    assert batch.n_chunks == want["chunks"]
    assert batch.n_ranges == want["ranges"]
    blob, off = batch.serialize_all()
    got = blob_digest(blob, off)
    bad = [i for i, (a, b) in enumerate(zip(got, want["chunk_blocks"])) if a != b]
    assert not bad, f"chunk blocks differ: first at chunks [{bad[0] * 1024}, {bad[0] * 1024 + 1024})"
    assert len(got) == len(want["chunk_blocks"])
    if want["exhausted"]:
        assert batch.exhausted
        assert {k.canonical_string(): v for k, v in (batch.report or {}).items()} == want["report"]
    st = gen.state_dict()
    assert hashlib.sha256(json.dumps(st, sort_keys=True).encode()).hexdigest() == want["final_state_sha256"]


def _job(dcat, spec, limit=None):
    from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog

    idx = build_index_from_catalog(dcat, [])
    gen = ChunkGenerator(idx, 42)
    batch = gen.plan_batch(spec, limit or (1 << 40))
    return idx, gen, batch


@pytest.mark.parametrize("layout", ["tuples", "columns"])
def test_cfg2_full_job_bit_exact(layout):
    import torch

    import bench
    from paper_2502_19790_b200 import synth

    want = _need("cfg2")
    rt = bench.make_workload(0, 1.0)  # == synth.config("cfg2")
    dcat = _catalog(rt, layout)
    idx, gen, batch = _job(dcat, synth.cfg2_mixture())
    _check_index(idx, want)
    _check_chunks(gen, batch, want)
    # a second job on the same resident catalog (the bench's timed step) is identical
    idx2, gen2, batch2 = _job(dcat, synth.cfg2_mixture())
    blob, off = batch2.serialize_all()
    assert blob_digest(blob, off) == want["chunk_blocks"]
    del dcat
    torch.cuda.empty_cache()


def test_cfg2_iid_tenth_bit_exact():
    from paper_2502_19790_b200 import DeviceCatalog, synth

    want = _need("cfg2_iid")
    rt = synth.make_runs(10_000_000, 1000, synth.CFG2_PROPS, 1, seed=2)
    idx, gen, batch = _job(DeviceCatalog(synth.expand_numpy(rt)), synth.cfg2_mixture())
    _check_index(idx, want)
    _check_chunks(gen, batch, want)


def test_cfg5_index_and_first_2000_chunks():
    from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog, synth

    want = _need("cfg5")
    dcat = _catalog(synth.config("cfg5"), "columns")
    idx = build_index_from_catalog(dcat, [])
    _check_index(idx, want)
    spec = synth.cfg5_mixture(idx.component_keys())
    gen = ChunkGenerator(idx, 42)
    batch = gen.plan_batch(spec, want["chunks"])
    _check_chunks(gen, batch, want)


def test_cfg3_one_billion_samples_one_gpu():
    """The north-star job: 1B samples (100k files) indexed and chunked on one
    B200 in the u16 row-tuple layout, every chunk against the oracle."""
    import torch

    from paper_2502_19790_b200 import synth

    import bench
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    want = _need("cfg3")
    rt = synth.config("cfg3")
    codes, table = bench.run_level_tuples(rt, torch.device("cuda", 0))  # the bench's 1B construction
    dcat = bench.device_catalog(ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes), {"tuples": codes}, table)
    idx, gen, batch = _job(dcat, synth.cfg2_mixture())
    _check_index(idx, want)
    _check_chunks(gen, batch, want)
    del dcat, idx, gen, batch
    torch.cuda.empty_cache()


# ----------------------------------------------------------------- cfg 4 (ADO)


def test_cfg4_ado_pi_trajectory_22_domains_8_ranks():
    """SURVEY.md §8d cfg 4: 22 Pile-style domains, Dirichlet(1) prior, 8 DP
    ranks x 64 single-domain sequences x 2,048 tokens per step, per-token loss
    = hidden law eps + beta n^-alpha times noise; each rank reduces on the
    device (per_domain_loss), the 8 results are summed (the all-reduce) and
    fed to the device AdoSource. The oracle (OracleAdo) gets the same sums
    from its own host reduction. Every step's pi within 1e-5 relative; refits
    at exactly 1000 and 2000."""
    import torch

    from oracle import oracle as orc
    from paper_2502_19790_b200 import AdoConfig, AdoSource, AdoState, MixtureKey
    from paper_2502_19790_b200.ado import domain_loss_device

    D, ranks, seqs, seq_len, steps = 22, 8, 64, 2048, 2100
    rng = np.random.Generator(np.random.PCG64(4))
    prior = rng.dirichlet(np.ones(D))
    eps, beta, alpha = rng.uniform(1.5, 2.5, D), rng.uniform(2, 10, D), rng.uniform(0.2, 0.5, D)
    keys = [MixtureKey.of({"domain": f"d{i:02d}"}) for i in range(D)]
    src = AdoSource(AdoState(AdoConfig(), dict(zip(keys, prior))), 1024)
    ado = orc.OracleAdo(list(prior))
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(4)
    n_tok = np.zeros(D)
    worst = 0.0
    for step in range(1, steps + 1):
        spec = src.current_spec()
        pi_ref = np.array(ado.compute_pi())
        pi = np.array([spec.weights.get(k, 0.0) for k in keys])
        worst = max(worst, float(np.max(np.abs(pi - pi_ref) / pi_ref)))
        # sequences drawn from the oracle's pi (identical inputs on both sides)
        dom = torch.from_numpy(rng.choice(D, size=ranks * seqs, p=pi_ref / pi_ref.sum())).to(dev)
        n_tok += np.bincount(dom.cpu().numpy(), minlength=D) * seq_len
        law = torch.from_numpy(eps + beta * np.maximum(n_tok, 1.0) ** -alpha).to(dev)
        tags = dom.to(torch.int32).repeat_interleave(seq_len).view(ranks, -1)
        noise = 1.0 + 0.1 * (torch.rand(ranks * seqs * seq_len, device=dev, generator=g) - 0.5)
        losses = (law[tags.view(-1).long()] * noise).float().view(ranks, -1)
        sums = torch.zeros(D, dtype=torch.float64, device=dev)
        counts = torch.zeros(D, dtype=torch.int64, device=dev)
        for r in range(ranks):
            s_, c_ = domain_loss_device(losses[r], tags[r], D)
            sums += s_
            counts += c_
        hs, hc = sums.cpu().numpy(), counts.cpu().numpy()
        hl, ht = losses.cpu().numpy(), tags.cpu().numpy()
        os_, oc = np.zeros(D), np.zeros(D, np.int64)
        for r in range(ranks):
            a, b = orc.per_domain_loss_np(hl[r], ht[r], D)
            os_ += a
            oc += b
        assert np.array_equal(hc, oc)
        np.testing.assert_allclose(hs, os_, rtol=1e-12)
        src.observe_feedback(step, {keys[i]: (float(hs[i]), int(hc[i])) for i in range(D) if hc[i] > 0})
        ado.observe(step, os_, oc)
    assert src.state.fit_steps == ado.fit_steps == [1000, 2000]
    assert worst < 1e-5, worst


# ----------------------------------------------------------------- apportion


def _ref_apportion():
    ref = ROOT / "baseline" / "_ref"
    if (ref / "mixplane").exists():
        sys.path.insert(0, str(ref))
        from mixplane.mixtures import MixtureKey as RK, apportion

        return RK, apportion
    return None, None


def test_device_apportion_10k_random_strict_chunks(oracle):
    """10,000 random (weights, total) pairs, each planned as ONE strict chunk
    on the device from the same cursor state: the chunk's per-key sample
    counts are exactly apportion(weights, total) (Appendix B: Neumaier wsum,
    w / wsum * total, int(share + 1e-9), (-frac, key order) leftovers)."""
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, MixtureSpec, build_index_from_catalog, synth

    rt = synth.make_runs(40_000_000, 2000, synth.CFG2_PROPS, 64, seed=12)
    idx = build_index_from_catalog(DeviceCatalog(synth.expand_numpy(rt)), [])
    keys = idx.component_keys()
    assert len(keys) == 2000
    gen = ChunkGenerator(idx, 3)
    s0 = gen.state_dict()
    RK, ref_apportion = _ref_apportion()
    rng = np.random.Generator(np.random.PCG64(2502))
    checked = big = 0
    for trial in range(10_000):
        km = int(rng.integers(300, 1200)) if trial % 50 == 0 else int(rng.integers(1, 40))
        sel = np.sort(rng.choice(len(keys), size=km, replace=False))
        kind = trial % 5
        if kind == 0:
            w = rng.random(km)
        elif kind == 1:
            w = rng.dirichlet(np.full(km, 0.05)) + 1e-300
        elif kind == 2:
            w = np.ones(km)  # exact ties: leftovers by key order
        elif kind == 3:
            w = np.round(rng.random(km), 1) + 0.1  # decimal weights, many equal shares
        else:
            w = rng.pareto(1.2, km) + 1e-9
        w = w / w.sum()
        spec_w = {keys[i]: float(x) for i, x in zip(sel.tolist(), w)}
        try:
            total = int(rng.integers(km, max(km + 1, 5000)))
            spec = MixtureSpec(spec_w, total, strict=True)
        except Exception:
            continue  # MixtureSpec rejects sums off 1 by > 1e-9 (the reference does too)
        gen.load_state(s0)
        c = gen.generate(spec)
        assert c is not None, trial
        got = {k.canonical_string(): v for k, v in c.samples_per_key().items()}
        ow = {oracle.as_key(k): v for k, v in spec.weights.items()}
        want = {oracle.key_string(k): v for k, v in oracle.apportion(ow, total).items() if v > 0}
        assert got == want, trial
        if ref_apportion is not None:
            rw = {RK.parse(k.canonical_string()): v for k, v in spec.weights.items()}
            r = {k.canonical_string(): v for k, v in ref_apportion(rw, total).items() if v > 0}
            assert got == r, trial
        checked += 1
        big += km > 256
    assert checked > 9000 and big > 100
