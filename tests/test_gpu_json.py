"""Canonical chunk bytes built on the device (csrc/serialize.cu, SURVEY.md
§8(f)-1) vs the reference's serialized chunks (golden vectors) and vs the host
serializer on catalogs whose dataset / file ids need string ordering."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, golden_predicates, spec_from_json

pytestmark = pytest.mark.gpu


def _split(blob: bytes, off) -> list[str]:
    return [blob[off[i]:off[i + 1]].decode("ascii") for i in range(len(off) - 1)]


@pytest.mark.parametrize("case", ["cfg1_r1", "cfg1_r64", "cfg2_small", "filters_nulls", "multi_tags", "depletion",
                                  "cfg5_small"])
def test_device_json_matches_reference_chunks(case):
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog

    cc, g = load_golden(case)
    idx = build_index_from_catalog(DeviceCatalog(cc), golden_predicates(g))
    for name, run in g["runs"].items():
        gen = ChunkGenerator(idx, g["job_seed"])
        if name.startswith("arbitrary"):
            batch = gen.plan_batch(None, 10_000, arbitrary_size=int(name[len("arbitrary"):]))
        else:
            batch = gen.plan_batch(spec_from_json(g["mixtures"][name]), 10_000)
        if batch.n_chunks == 0:
            continue
        blob, off = batch.serialize_all()
        got = _split(blob, off)
        n = len(run["chunks"])
        assert got[:n] == run["chunks"][:n], f"{case}/{name}"


def test_device_json_string_order_of_ids():
    """12 datasets and 120 files: str(ds) / str(fid) order differs from the
    numeric order ("10" < "2"); device bytes == host serializer bytes."""
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    cc = synth.expand_numpy(synth.make_runs(60_000, 120, synth.CFG1_PROPS, 8, seed=5))
    ds = np.repeat(np.arange(12, dtype=np.int32), 10)
    cat = ColumnarCatalog(columns=cc.columns, vocab=cc.vocab, multiple=cc.multiple,
                          file_ids=np.arange(1, 121, dtype=np.int64) * 7, file_ds=ds,
                          file_offsets=cc.file_offsets, dataset_names=[f"d{i}" for i in range(12)])
    idx = build_index_from_catalog(DeviceCatalog(cat), [])
    for spec in synth.cfg1_mixtures().values():
        gen = ChunkGenerator(idx, 42)
        batch = gen.plan_batch(spec, 10_000)
        blob, off = batch.serialize_all()
        got = _split(blob, off)
        want = []
        for i in range(batch.n_chunks):
            c = batch.chunk(i)
            c.mixture = spec
            want.append(c.serialize().decode("ascii"))
        assert got == want


def test_served_chunks_carry_device_bytes():
    """Chunks handed out from a large look-ahead batch serialise to the
    device-built bytes, identical to the host canonical JSON."""
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog
    from paper_2502_19790_b200.seeding import canonical_json_bytes

    cc, g = load_golden("cfg2_small")
    idx = build_index_from_catalog(DeviceCatalog(cc), golden_predicates(g))
    spec = spec_from_json(g["mixtures"]["cfg2"])
    gen = ChunkGenerator(idx, g["job_seed"])
    batch = gen.plan_batch(spec, 10_000)
    assert batch.n_chunks >= batch.DEVICE_JSON_MIN
    for i in range(batch.n_chunks):
        c = batch.chunk(i)
        assert getattr(c, "_device_bytes", None) is not None
        assert c.serialize() == canonical_json_bytes(c.to_json())
    # the sequential API: look-ahead batches double (1, 2, ..., 64, 128)
    gen2 = ChunkGenerator(idx, g["job_seed"])
    got = []
    while True:
        c = gen2.generate(spec)
        if c is None:
            break
        got.append(c.serialize().decode("ascii"))
    assert got == g["runs"]["cfg2"]["chunks"]
