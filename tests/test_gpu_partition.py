"""GPU parity of the key-partitioned path (SURVEY.md §8(e), strong scaling:
parallel.build_partitioned_index, csrc/stage2.cu emit_local).

world_size 2 and 3 processes share cuda:0 over gloo. Each rank indexes only
its file shard; the key owners lay out their keys' cursor streams and return
block offsets; every rank plans on the key-level index and cuts only its own
intervals; the merged chunks must be the REFERENCE's chunk bytes and
shortfall reports (tests/golden, produced by the reference itself).
Every plan mode is covered: disjoint mixtures (fused and general planner),
keys sharing components, arbitrary chunks. The chunk-owner output
(parallel.plan_owned: pieces all-to-all'd to the owner of each contiguous
chunk range, normalised there) must tile the same plan. Cursor checkpoints (reference
format) are refused with NotImplementedError."""

from __future__ import annotations

import sys

import pytest

from test_gpu_shard import ROOT, _free_port

import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, case, out):
    import os

    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = _run_case(rank, world, case)
    finally:
        dist.destroy_process_group()


def _run_case(rank, world, case):
    from conftest import golden_predicates, load_golden, spec_from_json

    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog
    from paper_2502_19790_b200.parallel import (build_partitioned_index, file_shard, global_nullable, plan_owned,
                                                shard)

    cc, g = load_golden(case)
    f0, _ = file_shard(cc.n_files, world, rank)
    part = shard(cc, world, rank)
    dcat = DeviceCatalog(part, nullable=global_nullable(part))
    idx = build_partitioned_index(dcat, golden_predicates(g), f0, cc.file_ds, cc.file_ids)
    res = {"keys": [k.canonical_string() for k in idx.component_keys()],
           "counts": {k.canonical_string(): v for k, v in idx.key_sample_counts().items()}, "runs": {}}
    for name, run in g["runs"].items():
        arb = int(name[len("arbitrary"):]) if name.startswith("arbitrary") else None
        spec = None if arb else spec_from_json(g["mixtures"][name])
        gen = ChunkGenerator(idx, g["job_seed"])
        got = []
        for i in range(len(run["chunks"]) + int(run.get("exhausted", True))):
            c = gen.generate_arbitrary(arb) if arb else gen.generate(spec)
            if c is None:
                break
            got.append(c.serialize().decode("ascii"))
        report = None if gen.last_report is None else {k.canonical_string(): v for k, v in gen.last_report.items()}
        gen = ChunkGenerator(idx, g["job_seed"])
        batch = gen.plan_batch(spec, 10_000, arbitrary_size=arb)
        bulk = []
        for i in range(batch.n_chunks):
            c = batch.chunk(i)
            if spec is not None:
                c.mixture = spec
            bulk.append(c.serialize().decode("ascii"))
        # chunk-owner output: this rank's contiguous range of the same plan
        gen = ChunkGenerator(idx, g["job_seed"])
        ob = plan_owned(gen, spec, 10_000, arbitrary_size=arb)
        owned = []
        for i in range(ob.n_chunks):
            c = ob.chunk(i)
            if spec is not None:
                c.mixture = spec
            owned.append(c.serialize().decode("ascii"))
        blob, offs = ob.serialize_all() if ob.n_chunks else (b"", [0])
        dev_json = [blob[offs[i]:offs[i + 1]].decode("ascii") for i in range(ob.n_chunks)]
        after = gen.generate_arbitrary(arb) if arb else gen.generate(spec)  # state moved past every chunk
        res["runs"][name] = {"chunks": got, "report": report, "bulk": bulk, "owned": owned, "owned_json": dev_json,
                             "owned_lo": ob.chunk_lo, "owned_of": ob.global_chunks,
                             "after": None if after is None else after.serialize().decode("ascii")}
    try:
        ChunkGenerator(idx, g["job_seed"]).state_dict()
    except NotImplementedError:
        res["state_dict"] = "refused"

    return res


def _check(case, world):
    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import load_golden

    _, g = load_golden(case)
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    res = dict(out)
    assert sorted(res) == list(range(world))
    n_ok = 0
    for rank, r in res.items():
        assert r.get("state_dict") == "refused"
        for name, run in g["runs"].items():
            mine = r["runs"][name]
            n_ok += 1
            assert len(mine["chunks"]) == len(run["chunks"]), f"{case}/{name} rank {rank}"
            for i, (a, b) in enumerate(zip(mine["chunks"], run["chunks"])):
                assert a == b, f"{case}/{name} chunk {i} rank {rank}"
            if run["report"] is not None:
                assert mine["report"] == run["report"], f"{case}/{name} report rank {rank}"
            n = len(run["chunks"])
            assert mine["bulk"][:n] == run["chunks"], f"{case}/{name} bulk rank {rank}"
            if run.get("exhausted", True):
                assert len(mine["bulk"]) == n
    assert n_ok > 0
    for name, run in g["runs"].items():  # chunk-owner output: the ranks' ranges tile the bulk plan
        parts = sorted((r["runs"][name]["owned_lo"], r["runs"][name]["owned"]) for r in res.values())
        joined = [c for _, cs in parts for c in cs]
        bulk = res[0]["runs"][name]["bulk"]
        assert joined == bulk, f"{case}/{name} owned chunks"
        for rank, r in res.items():
            mine = r["runs"][name]
            assert mine["owned_json"] == mine["owned"], f"{case}/{name} owned device JSON rank {rank}"
            assert mine["owned_of"] == len(bulk)
            assert mine["after"] is None  # plan_owned consumed the whole plan (bulk = to exhaustion here)
    return res


@pytest.mark.parametrize("case", ["cfg1_r64", "cfg1_r1", "cfg2_small", "filters_nulls", "depletion", "cfg5_small"])
def test_partitioned_two_ranks_match_reference(case):
    _check(case, 2)


@pytest.mark.parametrize("case", ["cfg1_r64", "filters_nulls", "multi_tags", "cfg2_small", "cfg5_wide"])
def test_partitioned_three_ranks_match_reference(case):
    _check(case, 3)
