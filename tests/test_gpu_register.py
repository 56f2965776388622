"""§8f-3: metadata registration on the device vs the reference's
``MetadataCatalog.register_dataset`` on the same JSON-lines files.

The same files are registered by the unmodified reference (baseline/_ref)
and by ``DeviceMetadataCatalog``; the resulting catalogs must give the same
index (``filter_intervals`` + ``build_index`` vs the device index, also under
filters) and the same chunk bytes, and every registration error must be the
reference's exception with the reference's message (first failing record in
file order)."""

from __future__ import annotations

import json
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def mp():
    if not (REF / "mixplane").exists():
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, str(REF))
    import mixplane

    return mixplane


def _write(path, lines, final_newline=True):
    data = "\n".join(lines) + ("\n" if final_newline else "")
    path.write_bytes(data.encode("utf-8"))
    return path


def _records(rng, n, f):
    langs = ["python", "go", "rust", "c", "日本語", "naïve"]
    lic = ["mit", "apache", "gpl"]
    tags = ["a", "b", "c", "d"]
    out, cur = [], None
    for i in range(n):
        if cur is None or rng.random() < 0.1:
            cur = {"language": str(rng.choice(langs)), "license": str(rng.choice(lic))}
            r = rng.random()
            if r < 0.1:
                cur["license"] = None           # null
            elif r < 0.2:
                del cur["license"]              # missing
            k = int(rng.integers(0, 4))
            cur["tags"] = sorted(set(rng.choice(tags, size=k).tolist())) if k else []
            if rng.random() < 0.1:
                cur["tags"] = list(reversed(cur["tags"])) + cur["tags"][:1]  # unsorted + duplicate
        rec = {"id": f * 100000 + i, "text": f"f{f} s{i} \"quoted\" \\ tail", "meta": {"x": [1, 2.5, None, True]},
               **cur}
        out.append(json.dumps(rec, ensure_ascii=bool(rng.random() < 0.5)))
        if rng.random() < 0.02:
            out.append("")                          # empty line: not a record
    return out


def _specials():
    # records the device hands to the host: escapes in a value, a number,
    # a boolean, duplicate keys, whitespace, a single-element list for a
    # single-valued property
    return [
        '{"language": "py\\u0074hon", "license": "mit", "tags": ["a"]}',
        '{"language": 7, "license": "gpl", "tags": []}',
        '{"language": true, "license": "gpl"}',
        '{"language": "go", "license": "mit", "language": "rust", "tags": ["b", "a"]}',
        '  {"language" : "c" , "license":null ,"tags":[ "d" ,"d"]}  \r',
        '{"language": ["go"], "license": ["apache"], "tags": "a"}',
    ]


def _corpus(tmp_path, seed=5, files=4):
    rng = np.random.default_rng(seed)
    paths = []
    for f in range(files):
        lines = _records(rng, int(rng.integers(400, 900)), f)
        if f == 1:
            lines[5:5] = _specials()
        paths.append(_write(tmp_path / f"part{f}.jsonl", lines, final_newline=f != 2))
    return paths


def _schema(mp, nullable_license=True):
    return mp.PropertySchema([
        mp.PropertyDef("language"),
        mp.PropertyDef("license", kind="categorical", categories=("apache", "gpl", "mit"), nullable=nullable_license),
        mp.PropertyDef("tags", multiple=True),
    ])


def _both(mp, paths, schema=None, parser=None, name="code"):
    from paper_2502_19790_b200.register import DeviceMetadataCatalog

    schema = schema or _schema(mp)
    parser = parser or mp.JsonFieldParser.for_properties(["language", "license", "tags"])
    ref = mp.MetadataCatalog()
    ref.register_dataset(name, paths, parser, schema)
    dev = DeviceMetadataCatalog()
    dev.register_dataset(name, paths, parser, schema)
    return ref, dev


def _ref_table(mp, ref, preds):
    idx = mp.build_index(ref.filter_intervals(preds))
    rows = []
    for key, dss in sorted(idx._index.items(), key=lambda kv: kv[0].sort_key()):
        for ds in sorted(dss):
            for fid in sorted(dss[ds]):
                for s, e in dss[ds][fid]:
                    rows.append((key.canonical_string(), ds, fid, s, e))
    return rows


@pytest.mark.parametrize("preds", [[], [("license", "==", "mit")], [("tags", "in", ("a", "c"))],
                                   [("language", "!=", "go"), ("license", "not-in", ("gpl",))]])
def test_device_registration_gives_the_reference_index(mp, tmp_path, preds):
    from paper_2502_19790_b200 import build_index_from_catalog

    paths = _corpus(tmp_path)
    ref, dev = _both(mp, paths)
    got = build_index_from_catalog(dev.device_catalog(), preds).table()
    assert got == _ref_table(mp, ref, preds)
    assert sorted(dev._files) == sorted(ref._files)
    assert [dev._files[f]["n_samples"] for f in sorted(dev._files)] == [ref._files[f].n_samples for f in sorted(ref._files)]


def test_device_registration_chunks_and_second_dataset(mp, tmp_path):
    """Two datasets (the second with another schema): chunk bytes through the
    device generator equal the reference generator's."""
    from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog
    from paper_2502_19790_b200.mixtures import MixtureKey, MixtureSpec

    paths = _corpus(tmp_path)
    ref, dev = _both(mp, paths)
    (tmp_path / "b").mkdir()
    rng = np.random.default_rng(9)
    more = [_write(tmp_path / "b" / f"x{i}.jsonl",
                   [json.dumps({"language": str(rng.choice(["go", "zig"])), "source": str(rng.choice(["s1", "s2"]))})
                    for _ in range(300)]) for i in range(2)]
    schema2 = mp.PropertySchema([mp.PropertyDef("language"), mp.PropertyDef("source")])
    p2 = mp.JsonFieldParser.for_properties(["language", "source"])
    assert ref.register_dataset("more", more, p2, schema2) == dev.register_dataset("more", more, p2, schema2) == 1
    spec = MixtureSpec({MixtureKey.of({"language": "go"}): 0.5, MixtureKey.of({"language": ["python", "rust"]}): 0.3,
                        MixtureKey.of({"source": "s2"}): 0.2}, 64)
    rgen = mp.ChunkGenerator(mp.build_index(ref.filter_intervals([])), 42)
    dgen = ChunkGenerator(build_index_from_catalog(dev.device_catalog(), []), 42)
    rspec = mp.MixtureSpec({mp.MixtureKey.parse(k.canonical_string()): w for k, w in spec.weights.items()}, 64)
    n = 0
    while True:
        a, b = rgen.generate(rspec), dgen.generate(spec)
        assert (a is None) == (b is None)
        if a is None:
            break
        assert a.serialize() == b.serialize(), n
        n += 1
    assert n > 10


def _errors_equal(mp, fn_ref, fn_dev):
    with pytest.raises(Exception) as er:
        fn_ref()
    with pytest.raises(Exception) as ed:
        fn_dev()
    assert type(ed.value).__name__ == type(er.value).__name__
    assert str(ed.value) == str(er.value)


@pytest.mark.parametrize("case", ["malformed", "categorical", "nonnull", "multi_single", "unknown_prop", "dict_value",
                                  "nan"])
def test_registration_errors_match_the_reference(mp, tmp_path, case):
    from paper_2502_19790_b200.register import DeviceMetadataCatalog

    rng = np.random.default_rng(1)
    good = _records(rng, 200, 0)
    bad = {
        "malformed": '{"language": "go", "license": "mit"',
        "categorical": '{"language": "go", "license": "bsd"}',
        "nonnull": '{"language": "go"}',
        "multi_single": '{"language": ["go", "c"], "license": "mit"}',
        "unknown_prop": '{"language": "go", "license": "mit", "extra": 1}',
        "dict_value": '{"language": {"a": 1}, "license": "mit"}',
        "nan": '{"language": "go", "license": "mit", "x": NaN}',
    }[case]
    lines = good[:50] + ["", bad] + good[50:] + [bad]
    p0 = _write(tmp_path / "ok.jsonl", good[:30])
    p1 = _write(tmp_path / "bad.jsonl", lines)
    schema = _schema(mp, nullable_license=case != "nonnull")
    fields = ["language", "license", "tags"] + (["extra"] if case == "unknown_prop" else [])
    parser = mp.JsonFieldParser.for_properties(fields)
    if case == "nan":  # NaN is valid for json.loads: both must register it
        ref, dev = _both(mp, [p0, p1], schema, parser)
        assert sorted(dev._files) == sorted(ref._files)
        return
    _errors_equal(mp, lambda: mp.MetadataCatalog().register_dataset("d", [p0, p1], parser, schema),
                  lambda: DeviceMetadataCatalog().register_dataset("d", [p0, p1], parser, schema))


def test_registration_file_checks_and_reregistration(mp, tmp_path):
    from paper_2502_19790_b200.register import DeviceMetadataCatalog

    paths = _corpus(tmp_path, files=2)
    schema = _schema(mp)
    parser = mp.JsonFieldParser.for_properties(["language", "license", "tags"])
    for files in ([], [tmp_path / "missing.jsonl"], [tmp_path / "part0.jsonl", tmp_path / "x.csv"]):
        if files and str(files[-1]).endswith(".csv"):
            files[-1].write_text("a,b\n")
        _errors_equal(mp, lambda: mp.MetadataCatalog().register_dataset("d", files, parser, schema),
                      lambda: DeviceMetadataCatalog().register_dataset("d", files, parser, schema))
    ref, dev = _both(mp, paths, schema, parser)
    assert dev.register_dataset("code", paths, parser, schema) == ref.register_dataset("code", paths, parser, schema)
    other = _write(tmp_path / "other.jsonl", ['{"language": "go", "license": "mit"}'])
    _errors_equal(mp, lambda: ref.register_dataset("code", [other], parser, schema),
                  lambda: dev.register_dataset("code", [other], parser, schema))
    s2 = mp.PropertySchema([mp.PropertyDef("language")])
    _errors_equal(mp, lambda: ref.register_dataset("code", paths, parser, s2),
                  lambda: dev.register_dataset("code", paths, parser, s2))
