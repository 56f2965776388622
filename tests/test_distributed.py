"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 host paths:
file sharding, the block-table all-gather for the global cursor merge, the
key-partitioned exchanges (block rows to the key owners and their replies
back, chunk ranges to their owners), and the data-parallel per-domain loss
all-reduce (stage 3)."""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn_name, out):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = globals()[fn_name](rank, world)
    finally:
        dist.destroy_process_group()


def _run(fn_name, world=2):
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, fn_name, out), nprocs=world, join=True)
    return dict(out)


def _catalog():
    from paper_2502_19790_b200 import synth

    return synth.expand_numpy(synth.make_runs(40_000, 13, synth.CFG2_PROPS, 16, seed=21))


def _oracle_blocks(cc):
    from oracle import oracle as orc
    from paper_2502_19790_b200.codec import KeyCodec
    from paper_2502_19790_b200.mixtures import MixtureKey
    from paper_2502_19790_b200.parallel import block_table

    idx = orc.build_index(cc, [])
    codec = KeyCodec.build(cc.vocab, {p: False for p in cc.vocab})
    lut, off = codec.luts(cc, [])
    packed_of = {}
    for key in idx.keys:
        mk = MixtureKey(key)
        code = 0
        for j, p in enumerate(codec.props):
            v = mk.values_for(p)
            c = cc.vocab[p].index(v[0])
            code += int(lut[off[j] + c + 1])
        packed_of[key] = code
    packed = np.array([packed_of[idx.keys[r]] for r in idx.rank], dtype=np.int64)
    return block_table(packed, idx.fid, idx.end - idx.start)


def blocks_job(rank, world):
    from paper_2502_19790_b200.parallel import gather_blocks, shard

    cc = _catalog()
    local = _oracle_blocks(shard(cc, world, rank))
    return gather_blocks(local).tolist()


def loss_job(rank, world):
    import torch

    from paper_2502_19790_b200.ado import allreduce_domain_loss

    rng = np.random.default_rng(rank)
    sums = torch.tensor(rng.uniform(0, 10, 5), dtype=torch.float64)
    counts = torch.tensor(rng.integers(0, 100, 5), dtype=torch.int64)
    s, c = allreduce_domain_loss(sums, counts)
    return s.tolist(), c.tolist()


def test_file_shards_partition_files():
    from paper_2502_19790_b200.parallel import file_shard

    for n in (1, 7, 100, 10_000):
        for world in (1, 2, 3, 8):
            spans = [file_shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_sharded_blocks_gather_to_global_index():
    got = _run("blocks_job")
    full = _oracle_blocks(_catalog()).tolist()
    assert got[0] == full and got[1] == full


def test_domain_loss_allreduce_sums_ranks():
    got = _run("loss_job")
    exp_s, exp_c = 0.0, 0
    for r in range(2):
        rng = np.random.default_rng(r)
        exp_s = exp_s + rng.uniform(0, 10, 5)
        exp_c = exp_c + rng.integers(0, 100, 5)
    for r in range(2):
        np.testing.assert_allclose(got[r][0], exp_s, rtol=1e-12)
        assert got[r][1] == exp_c.tolist()


def owners_job(rank, world):
    """Every rank routes its (key rank, payload) rows to the key owners; each
    owner answers f(row) and the replies come back in the sender's row order."""
    import torch

    from paper_2502_19790_b200.parallel import _all_to_all_rows, route_to_owners

    rng = np.random.default_rng(100 + rank)
    n = int(rng.integers(0, 50))
    key_rank = torch.from_numpy(rng.integers(0, 7, n).astype(np.int64))
    rows = torch.stack([key_rank.to(torch.int32), torch.from_numpy(rng.integers(0, 1000, n).astype(np.int32)),
                        torch.full((n,), rank, dtype=torch.int32)], 1) if n else torch.zeros((0, 3), dtype=torch.int32)
    perm, splits = route_to_owners(key_rank, world)
    recv, in_splits = _all_to_all_rows(rows[perm].contiguous(), splits, None)
    assert bool((recv[:, 0].to(torch.int64) % world == rank).all())  # only this owner's keys arrive
    reply = (recv[:, 0].to(torch.int64) * 100000 + recv[:, 1].to(torch.int64) * 10 + recv[:, 2].to(torch.int64))
    back, _ = _all_to_all_rows(reply.contiguous(), in_splits, None)
    out = torch.empty_like(back)
    out[perm] = back
    want = rows[:, 0].to(torch.int64) * 100000 + rows[:, 1].to(torch.int64) * 10 + rank
    return bool(torch.equal(out, want)), n, sum(in_splits)


def test_key_owner_routing_round_trip():
    got = _run("owners_job")
    assert all(ok for ok, _, _ in got.values())
    assert sum(n for _, n, _ in got.values()) == sum(m for _, _, m in got.values())


def test_key_level_rows_split_large_totals():
    from paper_2502_19790_b200.parallel import U32_SPLIT, key_level_rows

    gkeys = np.array([3, 9, 40], dtype=np.uint32)
    totals = np.array([5, 2 * U32_SPLIT + 7, U32_SPLIT], dtype=np.int64)
    rows = key_level_rows(gkeys, totals, n_files=4)
    assert rows[:, 0].tolist() == [3, 9, 9, 9, 40]
    assert rows[:, 1].tolist() == [0, 0, 1, 2, 0]
    assert rows[:, 3].tolist() == [0, 1, 1, 1, 2]
    for k, t in zip(gkeys, totals):
        assert int(rows[rows[:, 0] == k, 2].astype(np.int64).sum()) == int(t)
    with pytest.raises(ValueError):
        key_level_rows(gkeys, totals, n_files=2)


def test_chunk_ranges_tile_the_plan():
    from paper_2502_19790_b200.parallel import chunk_range

    for n in (0, 1, 5, 83_006):
        for world in (1, 2, 3, 8):
            spans = [chunk_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
