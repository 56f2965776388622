"""GPU parity: stage 1 (index), cursor layout, component order and stage 2
(chunk sequences) through the C-ABI vs the reference's golden vectors."""

from __future__ import annotations

import pytest

from conftest import STAGE12_CASES, golden_predicates, load_golden, spec_from_json

pytestmark = pytest.mark.gpu


def tuple_catalog(cc, narrow=False):
    """The same catalog in the row-tuple layout (one tuple-code column: int32,
    or u16 with `narrow`)."""
    import numpy as np
    import torch

    from paper_2502_19790_b200 import DeviceCatalog
    from paper_2502_19790_b200.catalog import encode_row_tuples, narrow_codes

    props = sorted(cc.vocab)
    codes, table = encode_row_tuples([cc.columns[p] for p in props], [len(cc.vocab[p]) for p in props])
    assert np.array_equal(table[codes].T, np.stack([cc.columns[p] for p in props]))
    if narrow:
        codes = narrow_codes(codes, len(table))
        assert codes.dtype == np.int16
    return DeviceCatalog(cc, tuples=(torch.from_numpy(codes).cuda(), table))


def _index(case, layout="columns"):
    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog

    cc, g = load_golden(case)
    dcat = DeviceCatalog(cc) if layout == "columns" else tuple_catalog(cc, narrow=layout == "tuples16")
    idx = build_index_from_catalog(dcat, golden_predicates(g))
    return idx, g


LAYOUTS = ["columns", "tuples", "tuples16"]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("case", STAGE12_CASES)
def test_index_matches_reference(case, layout):
    idx, g = _index(case, layout)
    assert [list(r) for r in idx.table()] == g["index"]
    assert idx.n_intervals == len(g["index"])


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("case", STAGE12_CASES)
def test_cursors_and_component_order_match_reference(case, layout):
    from paper_2502_19790_b200 import ChunkGenerator

    idx, g = _index(case, layout)
    gen = ChunkGenerator(idx, g["job_seed"])
    assert [k.canonical_string() for k in gen._component_order] == g["component_order"]
    for k in idx.component_keys():
        assert [list(r) for r in gen.cursor_ranges(k)] == g["cursors"][k.canonical_string()]


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("case", STAGE12_CASES)
def test_chunk_sequences_match_reference(case, layout):
    from paper_2502_19790_b200 import ChunkGenerator

    idx, g = _index(case, layout)
    for name, run in g["runs"].items():
        gen = ChunkGenerator(idx, g["job_seed"])
        got, states = [], {}
        for i in range(len(run["chunks"]) + int(run.get("exhausted", True))):
            if i in (1, 3):
                states[str(i)] = gen.state_dict()
            if name.startswith("arbitrary"):
                c = gen.generate_arbitrary(int(name[len("arbitrary"):]))
            else:
                c = gen.generate(spec_from_json(g["mixtures"][name]))
            if c is None:
                break
            got.append(c.serialize().decode("ascii"))
        assert len(got) == len(run["chunks"]), name
        for i, (a, b) in enumerate(zip(got, run["chunks"])):
            assert a == b, f"{case}/{name} chunk {i}"
        if run["report"] is not None:
            assert {k.canonical_string(): v for k, v in gen.last_report.items()} == run["report"]
        for i, st in run["states"].items():
            assert states[i] == st, f"{case}/{name} state@{i}"
        assert gen.state_dict() == run["final_state"], f"{case}/{name} final state"


@pytest.mark.parametrize("case", ["cfg1_r64", "cfg2_small", "filters_nulls"])
def test_bulk_plan_equals_sequential(case):
    """plan_batch(spec, n) emits exactly the chunks of n generate() calls."""
    from paper_2502_19790_b200 import ChunkGenerator

    idx, g = _index(case)
    name = next(n for n in g["runs"] if not n.startswith("arbitrary"))
    spec = spec_from_json(g["mixtures"][name])
    gen = ChunkGenerator(idx, g["job_seed"])
    batch = gen.plan_batch(spec, 10_000)
    got = []
    for i in range(batch.n_chunks):
        c = batch.chunk(i)
        c.mixture = spec
        got.append(c.serialize().decode("ascii"))
    assert got == g["runs"][name]["chunks"]


def test_restore_mid_stream_resumes_identically():
    from paper_2502_19790_b200 import ChunkGenerator

    idx, g = _index("cfg1_r64")
    run = g["runs"]["disjoint"]
    spec = spec_from_json(g["mixtures"]["disjoint"])
    gen = ChunkGenerator(idx, g["job_seed"])
    gen.load_state(run["states"]["3"])
    assert gen.generate(spec).serialize().decode() == run["chunks"][3]
    # switching spec mid look-ahead rewinds to the handed-out chunk
    gen2 = ChunkGenerator(idx, g["job_seed"])
    for i in range(5):
        gen2.generate(spec)
    st = gen2.state_dict()
    gen3 = ChunkGenerator(idx, g["job_seed"])
    for i in range(5):
        gen3.generate(spec)
    assert gen3.state_dict() == st


@pytest.mark.parametrize("case", ["cfg1_r64", "filters_nulls"])
def test_index_cursor_take_and_state(case):
    """ChunkerIndex.cursor(key, seed) (index.py:78-79, RangeCursor :118-189):
    the seeded layout is the golden one and take / depletion / state follow
    the reference semantics (replayed here on the golden range list)."""
    idx, g = _index(case)
    for k in idx.component_keys()[:6]:
        cur = idx.cursor(k, g["job_seed"])
        ranges = [tuple(r) for r in g["cursors"][k.canonical_string()]]
        assert cur._ranges == ranges
        total = sum(e - s for _, _, s, e in ranges)
        with pytest.raises(ValueError):
            cur.take(0)
        # reference take() replayed on the golden list
        pos, off, served = 0, 0, 0
        for n in (1, 7, 100, 3, 10_000, 10_000_000):
            got = cur.take(n)
            want, need = [], n
            while need > 0 and pos < len(ranges):
                ds, fid, s, e = ranges[pos]
                c = s + off
                if e - c <= need:
                    want.append((ds, fid, c, e))
                    need -= e - c
                    pos, off = pos + 1, 0
                else:
                    want.append((ds, fid, c, c + need))
                    off += need
                    need = 0
            served += n - need
            assert got == want
            assert cur.remaining_total == total - served
            if n == 100:
                st = cur.state_dict()
                assert st == {"pos": pos, "offset": off}
                other = idx.cursor(k, g["job_seed"])
                other.load_state(st)
                assert other.remaining_total == cur.remaining_total
        assert cur.depleted and cur.take(5) == []


def test_concurrent_jobs_on_two_streams():
    """Distinct jobs on distinct streams from two host threads (the reference
    server runs one thread per connection) give the sequential results."""
    import threading

    import torch

    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog

    cc, g = load_golden("cfg2_small")
    dcat = DeviceCatalog(cc)
    spec = spec_from_json(g["mixtures"]["cfg2"])

    def job(stream, seed, out, key):
        with torch.cuda.stream(stream):
            for _ in range(3):
                idx = build_index_from_catalog(dcat, golden_predicates(g), stream=stream)
                gen = ChunkGenerator(idx, seed, stream=stream)
                batch = gen.plan_batch(spec, 10_000)
                h = batch.to_host()
                out[key] = {k: v.copy() for k, v in h.items()}

    want = {}
    job(torch.cuda.current_stream(), g["job_seed"], want, "a")
    job(torch.cuda.current_stream(), 7, want, "b")
    got = {}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t1 = threading.Thread(target=job, args=(s1, g["job_seed"], got, "a"))
    t2 = threading.Thread(target=job, args=(s2, 7, got, "b"))
    t1.start(); t2.start(); t1.join(); t2.join()
    for key in ("a", "b"):
        for f in want[key]:
            assert (got[key][f] == want[key][f]).all(), (key, f)


def test_device_tuple_encoding_matches_host():
    """encode_row_tuples_device == encode_row_tuples (codes and table)."""
    import numpy as np
    import torch

    from paper_2502_19790_b200 import DeviceCatalog
    from paper_2502_19790_b200.catalog import encode_row_tuples

    cc, _ = load_golden("filters_nulls")
    props = sorted(cc.vocab)
    cards = [len(cc.vocab[p]) for p in props]
    hc, ht = encode_row_tuples([cc.columns[p] for p in props], cards)
    dc, dt = DeviceCatalog.encode_row_tuples_device(
        {p: torch.from_numpy(cc.columns[p]).cuda() for p in props}, cards)
    assert np.array_equal(dc.cpu().numpy(), hc) and np.array_equal(dt, ht)


@pytest.mark.parametrize("n_files", [1, 37])
def test_u16_tuple_codes_above_32767_match_columns(n_files):
    """> 32,768 distinct row tuples (u16 codes with the top bit set) index
    exactly like the per-property layout, across file boundaries."""
    import numpy as np
    import torch

    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    rng = np.random.default_rng(7)
    n = 300_001
    vocab = {"a": [f"a{i}" for i in range(50)], "b": [f"b{i}" for i in range(50)], "c": [f"c{i}" for i in range(30)]}
    # runs of random length so intervals are not all length 1
    lens = rng.integers(1, 8, size=n)
    cols = {p: np.repeat(rng.integers(0, len(v), size=n), lens)[:n].astype(np.int32) for p, v in vocab.items()}
    cuts = np.sort(rng.choice(np.arange(1, n), size=n_files - 1, replace=False)) if n_files > 1 else np.array([], int)
    offs = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    cc = ColumnarCatalog.from_arrays(cols, vocab, np.diff(offs))
    want = build_index_from_catalog(DeviceCatalog(cc), [])
    dcat16 = tuple_catalog(cc, narrow=True)
    assert len(dcat16.tuple_table) > 1 << 15
    got = build_index_from_catalog(dcat16, [])
    for k in ("key", "ds", "fid", "start", "end"):
        assert np.array_equal(got.interval_table()[k], want.interval_table()[k]), k
    assert np.array_equal(got.packed_keys()[0], want.packed_keys()[0])
    # device encoder narrows the same way
    dc, dt = DeviceCatalog.encode_row_tuples_device({p: torch.from_numpy(c).cuda() for p, c in cols.items()},
                                                    [len(vocab[p]) for p in sorted(vocab)])
    assert dc.dtype == torch.int16 and np.array_equal(dt, dcat16.tuple_table)
    assert np.array_equal(dc.cpu().numpy(), dcat16.tuple_codes.cpu().numpy())


@pytest.mark.parametrize("n_samples,n_files,cards", [(80_000, 40_000, (2,)), (60_000, 4_000, (30, 30, 20))])
def test_shuffles_beyond_shared_memory(n_samples, n_files, cards):
    """The draw-then-apply Fisher-Yates (csrc/mt19937.cuh WarpMT::draws +
    fy_apply) in its global-scratch form: keys with more blocks than the kernel's
    shared-memory capacity (16,000) and a component order of more ranks than
    component_order_kernel keeps in shared memory (16,384), vs the oracle's
    random.shuffle (index.py:134-144, chunks.py:139-141)."""
    import random

    from oracle import oracle as orc
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog, synth

    props = synth.numbered_props(cards)
    rt = synth.make_runs(n_samples, n_files, props, 1 if len(cards) > 1 else 2, seed=7)
    cc = synth.expand_numpy(rt)
    idx = build_index_from_catalog(DeviceCatalog(cc), [])
    ref = orc.build_index(cc, [])
    assert idx.table() == ref.table()
    gen = ChunkGenerator(idx, 99)
    n = len(ref.keys)
    order = list(range(n))
    random.Random(orc.seed_of(99, "component-order")).shuffle(order)
    assert [k.canonical_string() for k in gen._component_order] == [orc.key_string(ref.keys[r]) for r in order]
    if len(cards) == 1:
        assert max(ref.key_bounds[1:] - ref.key_bounds[:-1]) > 16_000
        for r in range(n):
            got = [tuple(x) for x in gen.cursor_ranges(idx.component_keys()[r])]
            assert got == ref.cursor_ranges(r, 99)
    else:
        assert n > 16_384
        for r in range(0, n, 997):
            got = [tuple(x) for x in gen.cursor_ranges(idx.component_keys()[r])]
            assert got == ref.cursor_ranges(r, 99)
