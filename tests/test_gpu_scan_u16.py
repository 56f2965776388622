"""GPU: the change-driven u16 row-tuple scan (csrc/scan_u16.cuh) against the
pinned oracle on catalogs built to hit its edge cases -- empty files, files
of 1..3 samples, files that start exactly on and next to the 1024-sample
warp-segment boundaries, runs crossing many segments, a partial last
segment, filters that fail whole runs, nulls, and iid codes (a change at
every sample). Each case is compared as the full interval table, in the
u16 tuple layout and, as a cross-check, in the int32 per-property layout."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _catalog(seed, n_files, sizes, mean_run, null_frac=0.0):
    from paper_2502_19790_b200 import synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    rng = np.random.default_rng(seed)
    props = synth.numbered_props((3, 4, 5))
    n = int(np.sum(sizes))
    rt = synth.make_runs(max(n, 1), 1, props, mean_run, seed=seed, null_frac=null_frac)
    lens = rt.run_lengths()
    cols = {p: np.repeat(c, lens)[:n].astype(np.int32) for p, c in rt.run_codes.items()}
    del rng, n_files
    return ColumnarCatalog.from_arrays(cols, rt.vocab, sizes)


def _sizes(kind, rng):
    if kind == "segment_edges":
        return [1023, 1, 1024, 1025, 0, 0, 2047, 1, 1, 1, 3072, 5, 1024, 999]
    if kind == "tiny_and_empty":
        return rng.choice([0, 0, 1, 2, 3, 7, 31, 33, 1000, 4000], size=400).tolist()
    if kind == "one_big_file":
        return [250_001]
    return rng.integers(1, 20_000, size=60).tolist()


CASES = [
    ("segment_edges", 8, 0.0, []),
    ("segment_edges", 1, 0.0, [("p0", "!=", "v00001")]),
    ("tiny_and_empty", 4, 0.0, []),
    ("tiny_and_empty", 2, 0.2, [("p1", "in", ("v00000", "v00002"))]),
    ("one_big_file", 64, 0.0, [("p2", "==", "v00003")]),
    ("one_big_file", 300, 0.0, []),
    ("random", 1, 0.0, []),
    ("random", 16, 0.1, [("p0", "not-in", ("v00002",))]),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_u16_scan_matches_oracle(case, oracle):
    import torch

    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog
    from paper_2502_19790_b200.catalog import encode_row_tuples, narrow_codes

    kind, mean_run, null_frac, preds = CASES[case]
    rng = np.random.default_rng(100 + case)
    sizes = _sizes(kind, rng)
    cc = _catalog(7 + case, len(sizes), sizes, mean_run, null_frac)
    try:
        want = oracle.build_index(cc, preds)
    except oracle.OracleError:
        pytest.skip("un-keyable sample in this draw")
    props = sorted(cc.vocab)
    codes, table = encode_row_tuples([cc.columns[p] for p in props], [len(cc.vocab[p]) for p in props])
    u16 = narrow_codes(codes, len(table))
    assert u16.dtype == np.int16
    for dcat in (DeviceCatalog(cc, tuples=(torch.from_numpy(u16).cuda(), table)), DeviceCatalog(cc)):
        idx = build_index_from_catalog(dcat, preds)
        t = idx.interval_table()
        assert idx.n_intervals == len(want.start)
        np.testing.assert_array_equal(t["key"].astype(np.int64), want.rank)
        np.testing.assert_array_equal(t["fid"], want.fid)
        np.testing.assert_array_equal(t["start"].astype(np.int64), want.start)
        np.testing.assert_array_equal(t["end"].astype(np.int64), want.end)


def test_u16_scan_unaligned_column_falls_back(oracle):
    """A u16 column that is not 16-byte aligned takes the generic path and
    gives the same index."""
    import torch

    from paper_2502_19790_b200 import DeviceCatalog, build_index_from_catalog
    from paper_2502_19790_b200.catalog import encode_row_tuples, narrow_codes

    sizes = [5000, 3000, 1]
    cc = _catalog(3, 3, sizes, 16)
    props = sorted(cc.vocab)
    codes, table = encode_row_tuples([cc.columns[p] for p in props], [len(cc.vocab[p]) for p in props])
    u16 = torch.from_numpy(narrow_codes(codes, len(table))).cuda()
    buf = torch.empty(len(u16) + 4, dtype=torch.int16, device="cuda")
    buf[1:1 + len(u16)] = u16
    idx = build_index_from_catalog(DeviceCatalog(cc, tuples=(buf[1:1 + len(u16)], table)), [])
    want = oracle.build_index(cc, [])
    assert [list(r) for r in idx.table()] == [list(r) for r in want.table()]
