"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 host paths:
file sharding, the block-table all-gather for the global cursor merge, and
the data-parallel per-domain loss all-reduce (stage 3)."""

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
