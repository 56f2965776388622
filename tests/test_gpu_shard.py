"""GPU parity of the file-sharded path (csrc/shard.cu).

world_size 2 and 3 processes share cuda:0 (the GPU box has one GPU) and
exchange over gloo; each indexes only its contiguous file shard of a golden
catalog, builds the hybrid index from the all-gathered block tables, and
generates the golden runs. Every rank must return the REFERENCE's chunk bytes,
checkpoint states and shortfall reports -- the same vectors the single-GPU
path is pinned to (tests/golden, produced by the reference itself)."""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
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
    from paper_2502_19790_b200.parallel import build_sharded_index, file_shard, global_nullable, shard

    cc, g = load_golden(case)
    f0, _ = file_shard(cc.n_files, world, rank)
    part = shard(cc, world, rank)
    dcat = DeviceCatalog(part, nullable=global_nullable(part))
    idx = build_sharded_index(dcat, golden_predicates(g), f0, cc.file_ds, cc.file_ids)
    res = {"keys": [k.canonical_string() for k in idx.component_keys()],
           "counts": {k.canonical_string(): v for k, v in idx.key_sample_counts().items()},
           "local_table": [list(r) for r in idx.local_index.table()],
           "runs": {}}
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
        report = None if gen.last_report is None else {k.canonical_string(): v for k, v in gen.last_report.items()}
        res["runs"][name] = {"chunks": got, "states": states, "final_state": gen.state_dict(), "report": report}
    # bulk path + restore from a reference checkpoint
    name = next(n for n in g["runs"] if not n.startswith("arbitrary"))
    spec = spec_from_json(g["mixtures"][name])
    gen = ChunkGenerator(idx, g["job_seed"])
    batch = gen.plan_batch(spec, 10_000)
    bulk = []
    for i in range(batch.n_chunks):
        c = batch.chunk(i)
        c.mixture = spec
        bulk.append(c.serialize().decode("ascii"))
    res["bulk"] = bulk
    run = g["runs"][name]
    if "3" in run["states"] and len(run["chunks"]) > 3:
        gen = ChunkGenerator(idx, g["job_seed"])
        gen.load_state(run["states"]["3"])
        res["resumed"] = gen.generate(spec).serialize().decode("ascii")
    return res


def _spawn(case, world):
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    return dict(out)


def _check(case, world):
    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import load_golden

    _, g = load_golden(case)
    res = _spawn(case, world)
    assert sorted(res) == list(range(world))
    # stage 1 on the shards: the union of the ranks' local tables is the
    # reference's index (key order, then dataset, file id, start)
    order = {k: i for i, k in enumerate(res[0]["keys"])}
    rows = sorted((r for x in res.values() for r in x["local_table"]), key=lambda r: (order[r[0]], r[1], r[2], r[3]))
    assert rows == g["index"], f"{case} sharded stage 1"
    for rank, r in res.items():
        assert r["keys"] == sorted(r["counts"], key=r["keys"].index)
        for name, run in g["runs"].items():
            mine = r["runs"][name]
            assert len(mine["chunks"]) == len(run["chunks"]), f"{case}/{name} rank {rank}"
            for i, (a, b) in enumerate(zip(mine["chunks"], run["chunks"])):
                assert a == b, f"{case}/{name} chunk {i} rank {rank}"
            if run["report"] is not None:
                assert mine["report"] == run["report"], f"{case}/{name} report rank {rank}"
            for i, st in run["states"].items():
                assert mine["states"][i] == st, f"{case}/{name} state@{i} rank {rank}"
            assert mine["final_state"] == run["final_state"], f"{case}/{name} final state rank {rank}"
        name = next(n for n in g["runs"] if not n.startswith("arbitrary"))
        ref = g["runs"][name]
        n = len(ref["chunks"]) if ref.get("exhausted", True) else min(len(ref["chunks"]), len(r["bulk"]))
        assert len(r["bulk"]) >= len(ref["chunks"]) and r["bulk"][:n] == ref["chunks"][:n], f"{case} bulk rank {rank}"
        if ref.get("exhausted", True):
            assert len(r["bulk"]) == len(ref["chunks"])
        if "resumed" in r:
            assert r["resumed"] == g["runs"][name]["chunks"][3]


@pytest.mark.parametrize("case", ["cfg1_r64", "cfg1_r1", "cfg2_small", "filters_nulls", "depletion", "cfg5_small"])
def test_sharded_two_ranks_match_reference(case):
    _check(case, 2)


@pytest.mark.parametrize("case", ["cfg1_r64", "filters_nulls", "multi_tags", "cfg5_wide"])
def test_sharded_three_ranks_match_reference(case):
    _check(case, 3)
