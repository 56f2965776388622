"""GPU: ``build_index(rows)`` (``index.py:88-115``) -- the device build from
explicit interval rows (sort by (key, file, start), empty / overlap checks,
adjacent merge on the GPU). The rows of every golden catalog (cut into
adjacent pieces and shuffled) must give the golden index, cursors and chunk
bytes; bad rows raise ``IndexBuildError`` like the reference."""

from __future__ import annotations

from collections import namedtuple

import numpy as np
import pytest

from conftest import STAGE12_CASES, golden_predicates, load_golden, spec_from_json

pytestmark = pytest.mark.gpu

Row = namedtuple("Row", "dataset_id file_id key start end")


def _rows(case, split_seed=None):
    from oracle import oracle as orc
    from paper_2502_19790_b200 import MixtureKey

    cc, g = load_golden(case)
    iv = orc.filter_intervals(cc, golden_predicates(g))
    keys = [MixtureKey.parse(orc.key_string(k)) for k in iv["keys"]]
    rows = [Row(int(d), int(f), keys[int(k)], int(s), int(e))
            for d, f, k, s, e in zip(iv["ds"], iv["fid"], iv["key"], iv["start"], iv["end"])]
    if split_seed is not None:  # cut rows into adjacent pieces (build_index merges them back) and shuffle
        rng = np.random.default_rng(split_seed)
        out = []
        for r in rows:
            cuts = sorted({int(x) for x in rng.integers(r.start + 1, r.end, size=2)} if r.end - r.start > 2 else set())
            b = [r.start, *cuts, r.end]
            out += [Row(r.dataset_id, r.file_id, r.key, x, y) for x, y in zip(b[:-1], b[1:])]
        rng.shuffle(out)
        rows = out
    return rows, g


@pytest.mark.parametrize("case", STAGE12_CASES)
def test_rows_index_equals_golden_index_and_chunks(case):
    from paper_2502_19790_b200 import ChunkGenerator, build_index

    rows, g = _rows(case, split_seed=1)
    idx = build_index(rows, workers=4)
    assert [list(r) for r in idx.table()] == g["index"]
    gen = ChunkGenerator(idx, g["job_seed"])
    assert [k.canonical_string() for k in gen._component_order] == g["component_order"]
    for k in idx.component_keys():
        assert [list(r) for r in gen.cursor_ranges(k)] == g["cursors"][k.canonical_string()]
    name = next(n for n in g["runs"] if not n.startswith("arbitrary"))
    run = g["runs"][name]
    spec = spec_from_json(g["mixtures"][name])
    got = []
    for _ in range(len(run["chunks"]) + int(run.get("exhausted", True))):
        c = gen.generate(spec)
        if c is None:
            break
        got.append(c.serialize().decode("ascii"))
    assert got == run["chunks"]
    assert gen.state_dict() == run["final_state"]


def test_rows_index_is_order_and_worker_independent():
    from paper_2502_19790_b200 import build_index

    rows, _ = _rows("cfg1_r64")
    a = build_index(rows)
    b = build_index(list(reversed(rows)), workers=8)
    assert a == b and a.table() == b.table()
    assert a.key_sample_counts() == b.key_sample_counts()
    assert a.total_samples() == sum(r.end - r.start for r in rows)


def test_rows_index_errors_and_reference_examples():
    from paper_2502_19790_b200 import IndexBuildError, MixtureKey, build_index

    PY, JS = MixtureKey.of({"language": "python"}), MixtureKey.of({"language": "javascript"})
    rows = [Row(1, 1, PY, 0, 10), Row(1, 1, PY, 10, 15), Row(1, 2, PY, 3, 8), Row(1, 1, JS, 20, 30),
            Row(2, 5, JS, 0, 4)]
    idx = build_index(rows)
    assert idx.entries(PY)[1][1] == [(0, 15)]
    assert idx.key_sample_counts() == {PY: 20, JS: 14}
    assert idx.component_keys() == [JS, PY]
    assert idx.matching_keys(MixtureKey.of({"license": "mit"})) == [JS, PY]
    with pytest.raises(IndexBuildError, match="overlapping"):
        build_index([Row(1, 1, PY, 0, 10), Row(1, 1, PY, 5, 12)])
    with pytest.raises(IndexBuildError, match="empty interval"):
        build_index([Row(1, 1, PY, 4, 4)])
    # the same ranges under different keys may share a file (the reference
    # checks overlaps per key -> dataset -> file)
    assert build_index([Row(1, 1, PY, 0, 10), Row(1, 1, JS, 5, 12)]).n_intervals == 2
    empty = build_index([])
    assert empty.n_intervals == 0 and empty.component_keys() == []


def test_rows_index_large_random_vs_reference_build_index():
    """200k random rows (many keys, datasets, adjacent pieces) vs the
    reference's own build_index when it is installed (baseline/_ref)."""
    import sys

    from conftest import ROOT
    from paper_2502_19790_b200 import MixtureKey, build_index

    rng = np.random.default_rng(7)
    keys = [MixtureKey.of({"a": f"v{i % 37}", "b": f"w{i // 37}"}) for i in range(500)]
    rows = []
    for f in range(2000):
        ds, pos = f % 3, 0
        while pos < 1000:
            n = int(rng.integers(1, 40))
            rows.append(Row(ds, 10 * f + ds, keys[int(rng.integers(0, len(keys)))], pos, pos + n))
            pos += n + int(rng.integers(0, 2))
    rng.shuffle(rows)
    idx = build_index(rows)
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mixplane").exists():
        pytest.skip("reference not installed")
    sys.path.insert(0, str(ref))
    from mixplane.catalog import IntervalRow
    from mixplane.index import build_index as ref_build
    from mixplane.mixtures import MixtureKey as RK

    rk = {k: RK.parse(k.canonical_string()) for k in keys}
    want = ref_build([IntervalRow(r.dataset_id, r.file_id, rk[r.key], r.start, r.end) for r in rows])
    assert idx == want
    assert idx.key_sample_counts() == want.key_sample_counts()
