"""CPU tests of the host-side logic: key codec (order-preserving packing,
decode, matching tables), mixture algebra vs the reference / oracle, synth
determinism, error types. No GPU needed."""

from __future__ import annotations

import random
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from paper_2502_19790_b200 import MixtureKey, MixtureSpec, apportion, synth
from paper_2502_19790_b200.catalog import ColumnarCatalog, FilterPredicate
from paper_2502_19790_b200.codec import KeyCodec
from paper_2502_19790_b200.errors import MixtureError, QueryError

REF_SRC = Path("/root/reference/pkg/src")


def _random_vocab(rng, n_props=4, multi=False):
    vocab = {}
    for j in range(n_props):
        card = rng.randint(1, 9)
        vals = [f"{rng.choice('abcxyz')}{rng.randint(0, 99)}" for _ in range(card)]
        vals = list(dict.fromkeys(vals))
        if multi and j == 0:
            tuples = {tuple(sorted(set(rng.sample(vals, rng.randint(1, len(vals)))))) for _ in range(6)}
            vocab[f"p{j}"] = sorted(tuples)
        else:
            vocab[f"p{j}"] = vals
    return vocab


@pytest.mark.parametrize("seed", range(12))
def test_packed_key_order_equals_sort_key(seed):
    rng = random.Random(seed)
    vocab = _random_vocab(rng, n_props=rng.randint(1, 5), multi=seed % 2 == 1)
    nullable = {p: rng.random() < 0.5 for p in vocab}
    codec = KeyCodec.build(vocab, nullable)
    props = codec.props
    keys = {}
    for _ in range(300):
        packed = 0
        pairs = {}
        for j, p in enumerate(props):
            if nullable[p] and rng.random() < 0.3:
                code = -1
            else:
                code = rng.randrange(len(vocab[p]))
            lut, off = codec.luts(ColumnarCatalog.meta_only(vocab, [1]), [])
            packed += int(lut[off[j] + code + 1])
            if code >= 0:
                v = vocab[p][code]
                pairs[p] = list(v) if isinstance(v, tuple) else v
        if not pairs:
            continue
        key = MixtureKey.of(pairs)
        keys[packed] = key
        assert codec.decode(packed) == key
    ordered = [keys[k] for k in sorted(keys)]
    assert ordered == sorted(keys.values(), key=MixtureKey.sort_key)


@pytest.mark.parametrize("seed", range(6))
def test_allow_table_equals_key_matching(seed):
    rng = random.Random(100 + seed)
    vocab = _random_vocab(rng, n_props=3, multi=seed % 2 == 0)
    codec = KeyCodec.build(vocab, {p: True for p in vocab})
    comps = []
    for _ in range(60):
        pairs = {}
        for p in codec.props:
            if rng.random() < 0.8:
                v = rng.choice(vocab[p])
                pairs[p] = list(v) if isinstance(v, tuple) else v
        if pairs:
            comps.append(MixtureKey.of(pairs))
    flat = {p: sorted({x for v in vocab[p] for x in ((v,) if isinstance(v, str) else v)}) for p in vocab}
    mkeys = []
    for _ in range(20):
        pairs = {}
        for p in list(codec.props) + ["absent_prop"]:
            if rng.random() < 0.5:
                pool = flat.get(p, ["q1", "q2"]) + ["unknown"]
                pairs[p] = rng.sample(pool, rng.randint(1, min(3, len(pool))))
        mkeys.append(MixtureKey.of(pairs or {"p0": "unknown"}))
    table, base, words = codec.allow_table(mkeys)
    for c in comps:
        ranks = []
        for j, p in enumerate(codec.props):
            held = c.values_for(p)
            ranks.append(0 if held is None else codec.sorted_values[j].index(held) + 1)
        for m, mk in enumerate(mkeys):
            ok = all((table[m][(base[j] + r) >> 5] >> ((base[j] + r) & 31)) & 1 for j, r in enumerate(ranks))
            assert ok == mk.matches(c), (mk, c)


def test_apportion_known_answers_and_exact_rational_agreement():
    K = MixtureKey.of
    a, b, c = K({"d": "a"}), K({"d": "b"}), K({"d": "c"})
    assert apportion({a: 0.7, b: 0.3}, 1024) == {a: 717, b: 307}
    assert apportion({a: 1 / 3, b: 1 / 3, c: 1 / 3}, 10) == {a: 4, b: 3, c: 3}
    rng = np.random.default_rng(7)
    keys = [K({"d": str(i)}) for i in range(8)]
    for _ in range(2000):
        dims = int(rng.integers(2, 9))
        w = {k: float(x) for k, x in zip(keys[:dims], rng.uniform(0.01, 10.0, dims))}
        total = int(rng.integers(1, 4097))
        got = apportion(w, total)
        assert sum(got.values()) == total and all(v >= 0 for v in got.values())
        ws = sum(Fraction(x) for x in w.values())
        for k, v in got.items():  # within one unit of the exact share
            assert abs(Fraction(w[k]) / ws * total - v) < 1


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not mounted")
def test_apportion_matches_reference_bit_for_bit():
    sys.path.insert(0, str(REF_SRC))
    from mixplane.mixtures import MixtureKey as RK, apportion as ref_apportion

    rng = np.random.default_rng(11)
    for _ in range(3000):
        dims = int(rng.integers(1, 12))
        raw = rng.dirichlet(np.ones(dims)) if rng.random() < 0.5 else rng.uniform(0.001, 5, dims)
        total = int(rng.integers(0, 5000))
        mine = apportion({MixtureKey.of({"k": f"v{i}"}): float(x) for i, x in enumerate(raw)}, total)
        ref = ref_apportion({RK.of({"k": f"v{i}"}): float(x) for i, x in enumerate(raw)}, total)
        assert {k.canonical_string(): v for k, v in mine.items()} == {
            k.canonical_string(): v for k, v in ref.items()}


def test_oracle_apportion_equals_host_apportion(oracle):
    rng = np.random.default_rng(3)
    for _ in range(1000):
        dims = int(rng.integers(1, 10))
        w = {MixtureKey.of({"k": f"v{i}"}): float(x) for i, x in enumerate(rng.uniform(0.01, 3, dims))}
        total = int(rng.integers(0, 3000))
        host = apportion(w, total)
        orc = oracle.apportion({oracle.as_key(k): v for k, v in w.items()}, total)
        assert {k.entries: v for k, v in host.items()} == orc


def test_mixture_key_canonical_round_trip_with_escapes():
    k = MixtureKey.of({"a;b": ["x,y", "z:w", "back\\slash"], "c": "d"})
    assert MixtureKey.parse(k.canonical_string()) == k
    with pytest.raises(MixtureError):
        MixtureKey.of({})
    with pytest.raises(MixtureError):
        MixtureKey.parse("a:b\\")


def test_spec_validation_matches_reference_rules():
    K = MixtureKey.of
    with pytest.raises(MixtureError):
        MixtureSpec({K({"a": "x"}): 0.5}, 10)
    with pytest.raises(MixtureError):
        MixtureSpec({K({"a": "x"}): 1.0}, 0)
    spec = MixtureSpec({K({"a": "x"}): 1.0, K({"a": "y"}): 0.0}, 10)
    assert list(spec.weights) == [K({"a": "x"})]
    with pytest.raises(MixtureError):
        MixtureSpec({K({"a": "x"}): 0.5, K({"a": "y"}): 0.5}, 1, strict=True).counts()
    assert MixtureSpec.from_json(spec.to_json()) == spec


def test_filter_pass_tables_and_validation():
    cc = ColumnarCatalog.from_arrays({"lang": np.array([0, 1, -1, 2], np.int32)}, {"lang": ["py", "go", "c"]}, [4])
    preds = cc.validated([("lang", "in", ["py", "nope"])])
    assert cc.pass_table("lang", preds).tolist() == [False, True, False, False]
    neg = cc.validated([("lang", "!=", "go")])
    assert cc.pass_table("lang", neg).tolist() == [True, True, False, True]
    with pytest.raises(QueryError):
        cc.validated([("missing", "==", "x")])
    with pytest.raises(QueryError):
        FilterPredicate("lang", "~=", "x")


def test_synth_is_deterministic_and_covers_every_sample():
    a = synth.make_runs(50_000, 7, synth.CFG2_PROPS, 16, seed=9)
    b = synth.make_runs(50_000, 7, synth.CFG2_PROPS, 16, seed=9)
    assert np.array_equal(a.run_starts, b.run_starts)
    assert a.run_lengths().sum() == 50_000 and a.file_sizes.sum() == 50_000
    fs = np.concatenate(([0], np.cumsum(a.file_sizes)[:-1]))
    assert np.isin(fs, a.run_starts).all()  # runs are cut at every file start


@pytest.mark.parametrize("case", ["filters_nulls", "multi_tags", "cfg5_small"])
def test_row_tuple_lut_equals_per_property_status(case):
    """Row-tuple layout: the folded LUT gives every row the status (packed key,
    fail bit) the per-property scan computes from its codes."""
    from conftest import golden_predicates, load_golden
    from paper_2502_19790_b200.catalog import encode_row_tuples
    from paper_2502_19790_b200.codec import FAIL

    cc, g = load_golden(case)
    props = sorted(cc.vocab)
    nullable = {p: bool((cc.columns[p] < 0).any()) for p in props}
    codec = KeyCodec.build(cc.vocab, nullable)
    preds = cc.validated(golden_predicates(g))
    lut, off = codec.luts(cc, preds)
    key = np.zeros(cc.n_samples, np.uint64)
    fail = np.zeros(cc.n_samples, bool)
    for j, p in enumerate(props):
        e = lut[off[j] + cc.columns[p] + 1]
        key += (e & ~FAIL).astype(np.uint64)
        fail |= (e & FAIL) != 0
    want = key.astype(np.uint32) | np.where(fail, FAIL, np.uint32(0)).astype(np.uint32)
    codes, table = encode_row_tuples([cc.columns[p] for p in props], [len(cc.vocab[p]) for p in props])
    assert np.array_equal(table[codes].T, np.stack([cc.columns[p] for p in props]))
    tl, toff = codec.tuple_luts(cc, preds, table)
    assert list(toff) == [0, len(table) + 1]
    assert np.array_equal(tl[codes + 1], want)
