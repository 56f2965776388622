"""Multi-GPU plumbing (one process per GPU, torch.distributed).

SURVEY.md §8(e): stage 1 shards by file -- intervals never cross files
(``catalog.py:559-604``) -- so rank r indexes the contiguous file range
``file_shard(F, world, r)`` with no data-path collective (weak scaling).
The real exchange steps are:

* stage 3: the per-domain (loss sum, token count) vectors of the
  data-parallel ranks are summed (``ado.allreduce_domain_loss``);
* global cursor layout: every rank needs every key's full (dataset, file)
  list to reproduce the reference's per-key shuffle (``index.py:134-144``).
  ``gather_blocks`` all-gathers the compact per-(key, file) block tables
  (packed key, file id, samples) and merges them into the global order
  (packed key, file id); packed keys are globally consistent because the
  vocabulary (and hence the codec) is shared by all ranks.
"""

from __future__ import annotations

import numpy as np

from .catalog import ColumnarCatalog


def file_shard(n_files: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced file-index range [f0, f1) of ``rank``."""
    base, extra = divmod(n_files, world)
    f0 = rank * base + min(rank, extra)
    return f0, f0 + base + (1 if rank < extra else 0)


def shard(cc: ColumnarCatalog, world: int, rank: int) -> ColumnarCatalog:
    """The files of ``rank`` as a catalog (file ids and vocabularies kept)."""
    f0, f1 = file_shard(cc.n_files, world, rank)
    a, b = int(cc.file_offsets[f0]), int(cc.file_offsets[f1])
    return ColumnarCatalog(
        columns={p: c[a:b] for p, c in cc.columns.items()},
        vocab=cc.vocab,
        multiple=cc.multiple,
        file_ids=cc.file_ids[f0:f1],
        file_ds=cc.file_ds[f0:f1],
        file_offsets=cc.file_offsets[f0 : f1 + 1] - a,
        dataset_names=cc.dataset_names,
    )


def block_table(packed_key: np.ndarray, file_id: np.ndarray, length: np.ndarray) -> np.ndarray:
    """Per-(key, file) samples from an interval table, as int64 [B, 3] rows
    (packed key, file id, samples) sorted by (packed key, file id)."""
    if len(packed_key) == 0:
        return np.zeros((0, 3), dtype=np.int64)
    k = np.asarray(packed_key, dtype=np.int64)
    f = np.asarray(file_id, dtype=np.int64)
    order = np.lexsort((f, k))
    k, f, n = k[order], f[order], np.asarray(length, dtype=np.int64)[order]
    head = np.ones(len(k), dtype=bool)
    head[1:] = (k[1:] != k[:-1]) | (f[1:] != f[:-1])
    idx = np.flatnonzero(head)
    return np.stack([k[idx], f[idx], np.add.reduceat(n, idx)], axis=1)


def index_block_table(index) -> np.ndarray:
    """Block table of a device ``ChunkerIndex`` (host copy)."""
    packed, _ = index.packed_keys()
    t = index.interval_table()
    return block_table(packed[t["key"]], t["fid"], t["end"].astype(np.int64) - t["start"])


def merge_blocks(tables: list[np.ndarray]) -> np.ndarray:
    """Global (packed key, file id) order of per-rank tables (disjoint files)."""
    cat = np.concatenate([t for t in tables if len(t)] or [np.zeros((0, 3), np.int64)])
    if len(cat) == 0:
        return cat
    return cat[np.lexsort((cat[:, 1], cat[:, 0]))]


def gather_blocks(table: np.ndarray, group=None, device=None) -> np.ndarray:
    """All-gather every rank's block table (variable length) and merge."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return merge_blocks([table])
    dev = torch.device(device) if device is not None else torch.device("cpu")
    world = dist.get_world_size(group)
    n = torch.tensor([len(table)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    cap = int(max(s.item() for s in sizes))
    buf = torch.zeros((cap, 3), dtype=torch.int64, device=dev)
    if len(table):
        buf[: len(table)] = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return merge_blocks([o[: int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)])
