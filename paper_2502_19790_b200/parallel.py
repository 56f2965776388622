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


# ---------------------------------------------------------------------------
# File-sharded device index + chunk emission (csrc/shard.cu)
# ---------------------------------------------------------------------------
def _coll_device(group, device):
    """Where collective tensors live: the GPU for NCCL, host memory otherwise
    (gloo; used by the multi-process tests on one GPU)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_rows(t, group=None):
    """All-gather a [n, ...] tensor whose n differs per rank. Returns the
    stacked, zero-padded [world, cap, ...] tensor (on t's device) and the
    per-rank row counts (host list)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cdev = _coll_device(group, t.device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=cdev)
    sizes = torch.zeros(world, dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(sizes, n, group=group)
    counts = [int(x) for x in sizes.tolist()]
    cap = max(max(counts), 1)
    buf = torch.zeros((cap, *t.shape[1:]), dtype=t.dtype, device=cdev)
    if t.shape[0]:
        buf[: t.shape[0]] = t.to(cdev)
    out = torch.empty((world * cap, *t.shape[1:]), dtype=t.dtype, device=cdev)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out.view(world, cap, *t.shape[1:]).to(t.device), counts


def global_nullable(part: ColumnarCatalog, group=None) -> dict:
    """Collective: per-property "holds a null anywhere in the catalog" flags
    (MAX over ranks). The packed-key layout depends on them (codec.py), so
    every shard's DeviceCatalog must be built with the GLOBAL flags."""
    import torch
    import torch.distributed as dist

    props = sorted(part.vocab)
    flags = np.array([bool((np.asarray(part.columns[p]) < 0).any()) for p in props], dtype=np.int64)
    if dist.is_available() and dist.is_initialized():
        flags = _max_allreduce(flags, group, None)
    return {p: bool(f) for p, f in zip(props, flags.tolist())}


class ShardInfo:
    def __init__(self, world, rank, group, file_lo, file_hi, file_ds, file_ids):
        self.world, self.rank, self.group = world, rank, group
        self.file_lo, self.file_hi = file_lo, file_hi
        self.file_ds, self.file_ids = file_ds, file_ids


def build_sharded_index(local_catalog, predicates=(), file_lo: int = 0, file_ds=None, file_ids=None,
                        group=None, stream=None):
    """Collective: every rank passes its contiguous file shard (a
    ``DeviceCatalog`` whose files are the global files
    ``[file_lo, file_lo + n_local)``) and the GLOBAL file table
    (``file_ds``, ``file_ids``). Returns the hybrid ``ChunkerIndex``: global
    keys, blocks and per-key totals, this rank's intervals (csrc/shard.cu).
    Exchange: one all-gather of key lists (tiny) and one of block tables."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _lib
    from .index import ChunkerIndex, build_index_from_catalog

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    codec = local_catalog.codec
    layout = np.array([codec.key_bits, *codec.shift, *codec.width], dtype=np.int64)
    lay, _ = all_gather_rows(torch.from_numpy(layout).view(1, -1), group)
    if not bool((lay == lay[0]).all()):
        raise ValueError("ranks disagree on the packed-key layout: build every shard's DeviceCatalog with the "
                         "same vocabulary and parallel.global_nullable() flags")
    local = build_index_from_catalog(local_catalog, predicates, stream=stream)
    L = _lib.lib()
    dev = local_catalog.device
    packed = np.zeros(local.n_keys, np.uint32)
    _lib.check(L.mx_index_packed_keys(local.handle, _lib.ptr(packed)))
    keys, kcounts = all_gather_rows(torch.from_numpy(packed.astype(np.int64)), group)
    gkeys = np.unique(np.concatenate([keys[q, : kcounts[q]].numpy() for q in range(world)])).astype(np.uint32)
    rows = torch.empty((max(local.n_blocks, 1), 4), dtype=torch.int32, device=dev)
    if local.n_blocks:
        _lib.check(L.mx_index_block_table(local.handle, int(file_lo), rows.data_ptr(),
                                          C.c_void_p(_lib.stream_ptr(stream))))
    tables, counts = all_gather_rows(rows[: local.n_blocks], group)
    return hybrid_index(local, local_catalog, tables.contiguous(), counts, gkeys, file_lo, file_ds, file_ids,
                        world, rank, group, stream)


def hybrid_index(local, local_catalog, tables, counts, gkeys, file_lo, file_ds, file_ids, world, rank,
                 group=None, stream=None):
    """The hybrid ChunkerIndex from already-exchanged block tables
    (device int32 [world, cap, 4]), per-rank row counts and the sorted global
    key union (mx_index_build_sharded)."""
    import ctypes as C

    from . import _lib
    from .index import ChunkerIndex

    L = _lib.lib()
    file_ds = np.ascontiguousarray(file_ds, dtype=np.int32)
    file_ids = np.ascontiguousarray(file_ids, dtype=np.int64)
    counts_np = np.asarray(counts, dtype=np.int64)
    d = _lib.ShardDesc()
    P = C.POINTER
    d.world, d.rank = world, rank
    d.file_lo, d.file_hi = int(file_lo), int(file_lo) + local_catalog.host.n_files
    d.n_files = len(file_ids)
    d.file_ds = file_ds.ctypes.data_as(P(C.c_int32))
    d.file_ids = file_ids.ctypes.data_as(P(C.c_int64))
    d.tables = tables.data_ptr()
    d.counts = counts_np.ctypes.data_as(P(C.c_int64))
    d.cap = tables.shape[1]
    d.global_keys = gkeys.ctypes.data_as(P(C.c_uint32))
    d.n_global_keys = len(gkeys)
    out = C.c_void_p()
    _lib.check(L.mx_index_build_sharded(local.handle, C.byref(d), C.c_void_p(_lib.stream_ptr(stream)),
                                        C.byref(out)))
    idx = ChunkerIndex(out.value, local_catalog, stream)
    idx.shard = ShardInfo(world, rank, group, d.file_lo, d.file_hi, file_ds, file_ids)
    idx.local_index = local
    return idx


def _max_allreduce(arr: np.ndarray, group, device) -> np.ndarray:
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(_coll_device(group, device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().numpy()


class MergedChunkBatch:
    """Global chunk CSR (every rank's pieces interleaved into the reference's
    (mixture key, file, start) order); identical on every rank."""

    def __init__(self, local_batch, off, pieces, file_ds, file_ids):
        self.__dict__.update({k: v for k, v in local_batch.__dict__.items() if not k.startswith("_")})
        self._gen = local_batch._gen
        self._off, self._pieces = off, pieces
        self._file_ds, self._file_ids = file_ds, file_ids
        self.n_ranges = int(pieces.shape[1])
        self._host = None

    def to_host(self) -> dict:
        from . import _lib

        if self._host is None:
            n = self.n_chunks
            ids, seeds = np.zeros(n, np.int64), np.zeros(n, np.uint64)
            loc_off = np.zeros(n + 1, np.int64)
            _lib.check(_lib.lib().mx_gen_result_copy(self._gen._h, _lib.ptr(loc_off), _lib.ptr(ids),
                                                     _lib.ptr(seeds), 0, 0, 0, 0, 0))
            p = self._pieces.cpu().numpy().view(np.uint32)
            fidx = p[1].astype(np.int64)
            self._host = dict(off=self._off.cpu().numpy(), ids=ids, seeds=seeds, mkey=p[0].copy(),
                              ds=self._file_ds[fidx], fid=self._file_ids[fidx], start=p[2].copy(), end=p[3].copy())
        return self._host

    def chunk(self, i: int, mixture=None):
        """Lazy chunk i (host canonical bytes: the device JSON of the local
        result does not describe the merged chunks)."""
        from .chunks import Chunk

        h = self.to_host()
        c = Chunk(int(h["ids"][i]), None, int(h["seeds"][i]), None if self.arbitrary else self.spec)
        c._src = (self, i)
        if mixture is not None:
            c.mixture = mixture
        return c

    def _chunk_data(self, i: int):
        from .chunks import ChunkBatch

        return ChunkBatch._chunk_data(self, i)


def merge_batch(gen, batch, stream=None):
    """Collective: all-gather every rank's local chunk CSR of the same chunks
    and interleave them on the device (mx_chunks_merge)."""
    import ctypes as C

    import torch

    from . import _lib

    sh = getattr(gen.index, "shard", None) or gen.index.partition
    dev = gen.index.catalog.device
    L = _lib.lib()
    n, r = batch.n_chunks, batch.n_ranges
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    pieces = torch.empty((max(r, 1), 4), dtype=torch.int32, device=dev)
    cols = pieces.t().contiguous() if r else torch.empty((4, 1), dtype=torch.int32, device=dev)
    sp = C.c_void_p(_lib.stream_ptr(stream))
    _lib.check(L.mx_gen_result_export(gen._h, off.data_ptr(), *(cols[f].data_ptr() for f in range(4)), sp))
    offs, _ = all_gather_rows(off.view(1, -1), sh.group)  # [W, 1, n+1]
    offs = offs.view(sh.world, n + 1).contiguous()
    g, counts = all_gather_rows(cols.t()[:r].contiguous(), sh.group)  # [W, cap, 4]
    cap = g.shape[1]
    g4 = g.permute(2, 0, 1).contiguous()  # [4, W, cap]
    total = int(sum(counts))
    out_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    out = torch.empty((4, max(total, 1)), dtype=torch.int32, device=dev)
    _lib.check(L.mx_chunks_merge(sh.world, n, cap, offs.data_ptr(), *(g4[f].data_ptr() for f in range(4)),
                                 out_off.data_ptr(), *(out[f].data_ptr() for f in range(4)), sp))
    return MergedChunkBatch(batch, out_off, out[:, :total], sh.file_ds, sh.file_ids)


# ---------------------------------------------------------------------------
# Key-partitioned path (SURVEY.md §8(e), strong scaling): no rank holds the
# global block table. Every global key is OWNED by one rank (its rank in the
# sorted key union, round robin); the owner alone lays out that key's cursor
# stream over the key's files of the whole catalog and hands every file owner
# the offsets of its (key, file) blocks. Every rank plans on the key-level
# index (global per-key totals: all the planner reads, chunks.py:188-259) and
# cuts only its own intervals (csrc/stage2.cu emit_local); the per-rank chunk
# CSRs are interleaved as in the file-sharded path (mx_chunks_merge).
# ---------------------------------------------------------------------------
U32_SPLIT = 1 << 31  # pseudo-interval length cap of the key-level index (u32 interval ends)


class PartitionInfo(ShardInfo):
    def __init__(self, world, rank, group, file_lo, file_hi, file_ds, file_ids, local, rows, key_g, key_g_rows):
        super().__init__(world, rank, group, file_lo, file_hi, file_ds, file_ids)
        self.local = local            # this rank's ChunkerIndex (local file indices)
        self.rows = rows              # device int32 [B, 4] local block rows (global file indices)
        self.key_g = key_g            # device int32 [n_local_keys]: global key rank
        self.key_g_rows = key_g_rows  # device int64 [B]: global key rank of every block row


def _all_to_all_rows(send, splits, group):
    """Variable all-to-all of the rows of ``send`` (rows grouped by
    destination, ``splits`` host list). Returns (received rows on send's
    device, per-source counts)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cdev = _coll_device(group, send.device)
    n_out = torch.tensor(splits, dtype=torch.int64, device=cdev)
    n_in = torch.empty(world, dtype=torch.int64, device=cdev)
    dist.all_to_all_single(n_in, n_out, group=group)
    in_splits = [int(x) for x in n_in.tolist()]
    recv = torch.empty((sum(in_splits), *send.shape[1:]), dtype=send.dtype, device=cdev)
    dist.all_to_all_single(recv, send.to(cdev), in_splits, list(splits), group=group)
    return recv.to(send.device), in_splits


def key_level_rows(gkeys: np.ndarray, totals: np.ndarray, n_files: int) -> np.ndarray:
    """Rows (packed key, pseudo file, samples, dense key rank) uint32[R, 4] of
    the key-level index: one pseudo-interval per key, totals above 2^31 split
    over consecutive pseudo files (u32 interval ends); already in (key, file)
    order."""
    gkeys = np.asarray(gkeys)
    totals = np.asarray(totals, dtype=np.int64)
    pieces = np.maximum(1, -(-totals // U32_SPLIT))
    if int(pieces.max(initial=1)) > n_files:
        raise ValueError("a key holds more than n_files * 2^31 samples")
    rk = np.repeat(np.arange(len(gkeys)), pieces)
    sub = np.arange(len(rk)) - np.repeat(np.cumsum(pieces) - pieces, pieces)
    krows = np.zeros((len(rk), 4), np.uint32)
    krows[:, 0] = gkeys[rk].astype(np.uint32)
    krows[:, 1] = sub
    krows[:, 2] = np.minimum(totals[rk] - sub * U32_SPLIT, U32_SPLIT)
    krows[:, 3] = rk
    return krows


def route_to_owners(key_rank, world: int):
    """Rows grouped by owner rank (key rank mod world), stable: (permutation
    of the rows, rows per owner). The owner's reply comes back in the same
    grouped order: ``reply_in_row_order[perm] = reply``."""
    import torch

    owner = key_rank % world
    perm = torch.argsort(owner, stable=True)
    splits = torch.bincount(owner, minlength=world).tolist() if len(owner) else [0] * world
    return perm, splits


def build_partitioned_index(local_catalog, predicates=(), file_lo: int = 0, file_ds=None, file_ids=None,
                            group=None, stream=None):
    """Collective: the key-level ChunkerIndex every rank plans on (global
    keys and per-key totals, the global file table), with ``.partition``
    describing this rank's files. Exchange: one all-gather of (packed key,
    samples) per key. The block offsets are exchanged per generator seed
    (``attach_partition``, called by ChunkGenerator)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _lib
    from .index import ChunkerIndex, build_index_from_catalog

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    codec = local_catalog.codec
    layout = np.array([codec.key_bits, *codec.shift, *codec.width], dtype=np.int64)
    lay, _ = all_gather_rows(torch.from_numpy(layout).view(1, -1), group)
    if not bool((lay == lay[0]).all()):
        raise ValueError("ranks disagree on the packed-key layout: build every shard's DeviceCatalog with the "
                         "same vocabulary and parallel.global_nullable() flags")
    local = build_index_from_catalog(local_catalog, predicates, stream=stream)
    L = _lib.lib()
    dev = local_catalog.device
    packed, samples = local.packed_keys()
    kt = torch.from_numpy(np.stack([packed.astype(np.int64), samples], axis=1))
    allk, counts = all_gather_rows(kt, group)
    cat = np.concatenate([allk[q, : counts[q]].numpy() for q in range(world)]) if sum(counts) else \
        np.zeros((0, 2), np.int64)
    gkeys, inv = np.unique(cat[:, 0], return_inverse=True)
    totals = np.zeros(len(gkeys), np.int64)
    np.add.at(totals, inv, cat[:, 1])
    file_ds = np.ascontiguousarray(file_ds, dtype=np.int32)
    file_ids = np.ascontiguousarray(file_ids, dtype=np.int64)
    n_files = len(file_ids)
    krows = key_level_rows(gkeys, totals, n_files)
    d_krows = torch.from_numpy(krows.view(np.int32)).to(dev)
    sp = C.c_void_p(_lib.stream_ptr(stream))
    out = C.c_void_p()
    _lib.check(L.mx_index_build_owner(local.handle, d_krows.data_ptr(), len(krows), n_files, _lib.ptr(file_ds),
                                      _lib.ptr(file_ids), _bits(len(gkeys) - 1), sp, C.byref(out)))
    idx = ChunkerIndex(out.value, local_catalog, stream)
    d_gkeys = torch.from_numpy(gkeys).to(dev)
    key_g = torch.searchsorted(d_gkeys, torch.from_numpy(packed.astype(np.int64)).to(dev)).to(torch.int32)
    rows = torch.empty((max(local.n_blocks, 1), 4), dtype=torch.int32, device=dev)
    if local.n_blocks:
        _lib.check(L.mx_index_block_table(local.handle, int(file_lo), rows.data_ptr(), sp))
    rows = rows[: local.n_blocks]
    key_g_rows = torch.searchsorted(d_gkeys, rows[:, 0].to(torch.int64) & 0xFFFFFFFF)
    file_hi = int(file_lo) + local_catalog.host.n_files
    ranges, _ = all_gather_rows(torch.tensor([[int(file_lo), file_hi]], dtype=torch.int64), group)
    ranges = ranges[:, 0].numpy()
    idx.partition = PartitionInfo(world, rank, group, int(file_lo), file_hi, file_ds, file_ids, local, rows, key_g,
                                  key_g_rows)
    # owners can skip the (file, key) sort when rank order is file order
    idx.partition.rank_file_ordered = bool((ranges[1:, 0] >= ranges[:-1, 1]).all())
    idx.partition.n_global_keys = len(gkeys)
    return idx


def _bits(v: int) -> int:
    return max(1, int(v).bit_length())


def attach_partition(gen):
    """Collective (ChunkGenerator on a partitioned index): send every block
    row to its key's owner, let the owners lay out their keys' cursor streams
    (generator seed = gen.seed) and return the block offsets, then point the
    generator's emission at this rank's intervals."""
    import ctypes as C

    import torch

    from . import _lib
    from .seeding import derive_seed, hash_message

    pi = gen.index.partition
    L = _lib.lib()
    dev = gen.index.catalog.device
    sp = C.c_void_p(_lib.stream_ptr(gen.stream))
    perm, splits = route_to_owners(pi.key_g_rows, pi.world)
    send = pi.rows[perm].contiguous()
    dense = 0
    if pi.rank_file_ordered:  # row[3] := the key's rank among the owner's keys
        send[:, 3] = (pi.key_g_rows[perm] // pi.world).to(torch.int32)
        dense = _bits((pi.n_global_keys - 1) // pi.world)
    recv, in_splits = _all_to_all_rows(send, splits, pi.group)
    n = int(recv.shape[0])
    oix = C.c_void_p()
    _lib.check(L.mx_index_build_owner(pi.local.handle, recv.data_ptr() if n else None, n, len(pi.file_ids),
                                      _lib.ptr(pi.file_ds), _lib.ptr(pi.file_ids), dense, sp, C.byref(oix)))
    off = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
    og = C.c_void_p()
    try:
        cur = hash_message(gen.seed, "cursor")
        chk = hash_message(gen.seed, "chunk")
        _lib.check(L.mx_gen_create(oix, cur, len(cur), chk, len(chk), derive_seed(gen.seed, "component-order"), sp,
                                   C.byref(og)))
        try:
            if n:
                _lib.check(L.mx_gen_block_offsets(og, off.data_ptr(), sp))
        finally:
            L.mx_gen_free(og)
    finally:
        L.mx_index_free(oix)
    back, _ = _all_to_all_rows(off[:n], in_splits, pi.group)
    blk_off = torch.empty_like(back)
    blk_off[perm] = back
    gen._partition_bufs = (blk_off, pi.key_g)
    _lib.check(L.mx_gen_set_local(gen._h, pi.local.handle, blk_off.data_ptr() if len(blk_off) else None,
                                  pi.key_g.data_ptr() if len(pi.key_g) else None, pi.file_lo))


def chunk_range(n_chunks: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced range [c0, c1) of the plan's chunks owned by ``rank``."""
    return file_shard(n_chunks, world, rank)


class _DevPtr:
    """Zero-copy view of library-owned device memory (valid until the next plan)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3}


def plan_owned(gen, spec, max_chunks: int, arbitrary_size: int | None = None):
    """Collective bulk plan of a partitioned generator, chunk-owner output
    (SURVEY.md §8(e)): every rank cuts its pieces of every planned chunk; one
    all-to-all sends each contiguous chunk range's pieces (and per-chunk
    counts) to its owner, which normalises only its chunks. Returns this
    rank's ``ChunkBatch`` (global chunks ``batch.chunk_lo`` ..
    ``batch.chunk_lo + batch.n_chunks`` of ``batch.global_chunks``); the
    generator state advances past all of them on every rank. Equivalent to
    ``plan_batch`` whose result is split by chunk over the ranks."""
    import ctypes as C

    import torch

    from . import _lib
    from .chunks import ChunkBatch

    pi = gen.index.partition
    L = _lib.lib()
    sp = C.c_void_p(_lib.stream_ptr(gen.stream))
    dev = gen.index.catalog.device
    gen._rewind()
    _lib.check(L.mx_gen_set_handoff(gen._h, 1))
    try:
        n, exhausted, (mkeys, report) = gen._plan(spec, max_chunks, arbitrary_size)
        nc, npc, offp, pp = C.c_int64(), C.c_int64(), C.c_void_p(), C.c_void_p()
        _lib.check(L.mx_gen_handoff(gen._h, C.byref(nc), C.byref(npc), C.byref(offp), C.byref(pp)))
        off = torch.as_tensor(_DevPtr(offp.value, (n + 1,), "<i8"), device=dev)
        pieces = torch.as_tensor(_DevPtr(pp.value, (npc.value, 4), "<i4"), device=dev) if npc.value else \
            torch.zeros((0, 4), dtype=torch.int32, device=dev)
        bounds = [chunk_range(n, pi.world, r) for r in range(pi.world)]
        cut = off[torch.tensor([b[0] for b in bounds] + [n], device=dev)].cpu().tolist()
        splits = [cut[r + 1] - cut[r] for r in range(pi.world)]
        recv, _ = _all_to_all_rows(pieces, splits, pi.group)
        counts = (off[1:] - off[:-1]).to(torch.int32)
        rcounts, _ = _all_to_all_rows(counts, [b - a for a, b in bounds], pi.group)
        lo, hi = bounds[pi.rank]
        _lib.check(L.mx_gen_finish_owned(gen._h, pi.world, lo, hi - lo, n, rcounts.data_ptr() if len(rcounts) else None,
                                         recv.data_ptr() if len(recv) else None, len(recv), sp))
    finally:
        L.mx_gen_set_handoff(gen._h, 0)
    gen._next_id += n
    cn, cr = C.c_int64(), C.c_int64()
    _lib.check(L.mx_gen_result_sizes(gen._h, C.byref(cn), C.byref(cr)))
    batch = ChunkBatch(gen, cn.value, cr.value, mkeys, spec, arbitrary_size)
    batch.exhausted, batch.report = exhausted, report
    batch.chunk_lo, batch.global_chunks = lo, n
    if exhausted:
        gen.last_report = report
    return batch
