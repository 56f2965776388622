"""GPU parity at full BASELINE sizes.

* cfg 1 (1M samples, 1,000 files; iid R=1 and clustered R=64): the complete
  interval table, every cursor's range order, and every chunk of a job under
  the disjoint and the overlapping mixture are compared with the CPU oracle.
* cfg 2 at 10% (10M samples): complete index + every chunk vs the oracle.
* cfg 2 at full size (100M samples): size-independent invariants -- each
  sample indexed exactly once, every chunk has exactly chunk_size samples,
  no sample is handed out twice, per-key counts of on-mixture chunks equal
  ``apportion`` -- plus bulk == sequential emission on a prefix.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpu_index(cc, preds=()):
    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog

    return build_index_from_catalog(DeviceCatalog(cc), list(preds))


def _assert_same_index(gidx, oidx, orc):
    t = gidx.interval_table()
    assert [k.canonical_string() for k in gidx.component_keys()] == [orc.key_string(k) for k in oidx.keys]
    np.testing.assert_array_equal(t["key"].astype(np.int64), oidx.rank)
    np.testing.assert_array_equal(t["ds"].astype(np.int64), oidx.ds)
    np.testing.assert_array_equal(t["fid"], oidx.fid)
    np.testing.assert_array_equal(t["start"].astype(np.int64), oidx.start)
    np.testing.assert_array_equal(t["end"].astype(np.int64), oidx.end)


def _chunks_equal(gidx, oidx, orc, spec, limit=None, bulk=False):
    from paper_2502_19790_b200 import ChunkGenerator

    gen = ChunkGenerator(gidx, 42)
    ogen = orc.OracleGenerator(oidx, 42)
    w = {orc.as_key(k): v for k, v in spec.weights.items()}
    n = 0
    if bulk:
        batch = gen.plan_batch(spec, limit or (1 << 40))
        for i in range(batch.n_chunks):
            c = batch.chunk(i)
            c.mixture = spec
            assert c.serialize() == ogen.generate(w, spec.chunk_size, spec.strict).serialize(), i
        return batch.n_chunks
    while limit is None or n < limit:
        a, b = gen.generate(spec), ogen.generate(w, spec.chunk_size, spec.strict)
        assert (a is None) == (b is None), n
        if a is None:
            break
        assert a.serialize() == b.serialize(), n
        n += 1
    return n


@pytest.mark.parametrize("layout_r", [1, 64])
def test_cfg1_full_index_cursors_and_chunks(oracle, layout_r):
    from paper_2502_19790_b200 import ChunkGenerator, synth

    cc = synth.expand_numpy(synth.make_runs(1_000_000, 1000, synth.CFG1_PROPS, layout_r, seed=1))
    gidx = _gpu_index(cc)
    oidx = oracle.build_index(cc, [])
    _assert_same_index(gidx, oidx, oracle)
    gen = ChunkGenerator(gidx, 42)
    ogen = oracle.OracleGenerator(oidx, 42)
    keys = gidx.component_keys()
    assert [k.canonical_string() for k in gen._component_order] == [
        oracle.key_string(oidx.keys[r]) for r in ogen.order]
    for r in (0, len(keys) // 2, len(keys) - 1):
        assert gen.cursor_ranges(keys[r]) == ogen.ranges[r]
    mixes = synth.cfg1_mixtures()
    n = _chunks_equal(gidx, oidx, oracle, mixes["disjoint"])
    assert n > 900
    assert _chunks_equal(gidx, oidx, oracle, mixes["overlap"], limit=300) == 300
    assert _chunks_equal(gidx, oidx, oracle, mixes["disjoint_strict"], bulk=True) > 400


def test_cfg2_tenth_scale_every_chunk(oracle):
    from paper_2502_19790_b200 import synth

    cc = synth.expand_numpy(synth.make_runs(10_000_000, 1000, synth.CFG2_PROPS, 64, seed=2))
    gidx = _gpu_index(cc)
    oidx = oracle.build_index(cc, [])
    _assert_same_index(gidx, oidx, oracle)
    n = _chunks_equal(gidx, oidx, oracle, synth.cfg2_mixture(), bulk=True)
    assert n > 8000


def test_cfg2_full_size_invariants():
    import torch

    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, apportion, build_index_from_catalog, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    rt = synth.config("cfg2")
    lens = torch.from_numpy(rt.run_lengths()).cuda()
    cols = {p: torch.repeat_interleave(torch.from_numpy(c).cuda(), lens) for p, c in rt.run_codes.items()}
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    idx = build_index_from_catalog(DeviceCatalog(meta, columns=cols), [])
    assert idx.n_samples == rt.n_samples  # every sample indexed exactly once
    assert idx.n_keys == 2000
    spec = synth.cfg2_mixture()
    gen = ChunkGenerator(idx, 42)
    batch = gen.plan_batch(spec, 1 << 40)
    h = batch.to_host()
    sizes = np.add.reduceat(h["end"].astype(np.int64) - h["start"], h["off"][:-1])
    assert (sizes == spec.chunk_size).all()
    # no sample twice: ranges sorted by (file, start) never overlap
    order = np.lexsort((h["start"], h["fid"]))
    f, s, e = h["fid"][order], h["start"][order].astype(np.int64), h["end"][order].astype(np.int64)
    same = f[1:] == f[:-1]
    assert not np.any(same & (s[1:] < e[:-1]))
    assert np.all(e > s)
    # on-mixture chunks carry exactly apportion(spec) per mixture key
    want = apportion(spec.weights, spec.chunk_size)
    c0 = batch.chunk(0).samples_per_key()
    assert {k.canonical_string(): v for k, v in c0.items()} == {k.canonical_string(): v for k, v in want.items()}
    # bulk == sequential on a prefix (look-ahead, then rewind on checkpoint)
    gen2 = ChunkGenerator(idx, 42)
    for i in range(20):
        c = gen2.generate(spec)
        ref = batch.chunk(i)
        ref.mixture = spec
        assert c.serialize() == ref.serialize()
    assert gen2.state_dict()["next_chunk_id"] == 20


def test_empty_result_and_error_contract():
    from paper_2502_19790_b200 import (
        ChunkGenerator,
        MixtureError,
        MixtureKey,
        MixtureSpec,
        QueryError,
        synth,
    )
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    cc = synth.expand_numpy(synth.make_runs(5_000, 4, synth.CFG1_PROPS, 8, seed=4))
    idx = _gpu_index(cc, [("language", "==", "nope")])
    assert idx.n_intervals == 0 and not idx and idx.component_keys() == []
    assert ChunkGenerator(idx, 1).generate(synth.cfg1_mixtures()["disjoint"]) is None
    with pytest.raises(QueryError):
        _gpu_index(cc, [("colour", "==", "red")])
    nulls = ColumnarCatalog.from_arrays({"a": np.array([0, -1, 0], np.int32)}, {"a": ["x"]}, [3])
    with pytest.raises(QueryError, match="no non-null properties"):
        _gpu_index(nulls)
    full = _gpu_index(cc)
    spec = MixtureSpec({MixtureKey.of({"language": "en"}): 0.5, MixtureKey.of({"language": "de"}): 0.5}, 1, strict=True)
    with pytest.raises(MixtureError):
        ChunkGenerator(full, 1).generate(spec)
    with pytest.raises(MixtureError):
        ChunkGenerator(full, 1).generate_arbitrary(0)


@pytest.mark.parametrize("chunk_size", [4096, 8192])
def test_cfg1_iid_chunks_beyond_shared_memory_sort(oracle, chunk_size):
    """iid cfg 1 with chunk_size >> 2,048: chunks of thousands of pieces
    before merging take the in-place global-memory sort (normalize_kernel,
    sort_merge_global); every chunk of the job equals the oracle's, in bulk
    and through generate()."""
    from paper_2502_19790_b200 import MixtureKey, MixtureSpec, synth

    cc = synth.expand_numpy(synth.make_runs(1_000_000, 1000, synth.CFG1_PROPS, 1, seed=1))
    gidx = _gpu_index(cc)
    oidx = oracle.build_index(cc, [])
    spec = MixtureSpec({MixtureKey.of({"language": "en"}): 0.5,
                        MixtureKey.of({"language": ["de", "es", "fr"]}): 0.5}, chunk_size)
    assert _chunks_equal(gidx, oidx, oracle, spec, bulk=True) > 1_000_000 // chunk_size // 2
    assert _chunks_equal(gidx, oidx, oracle, spec, limit=20) == 20
