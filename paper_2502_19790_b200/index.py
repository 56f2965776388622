"""Device-resident catalog and ChunkerIndex (stage 1 behind the reference API).

``build_index_from_catalog(catalog, predicates)`` is the drop-in for the
reference's ``build_index(catalog.filter_intervals(predicates))``
(``server.py:112-115``): one CUDA pipeline (``csrc/stage1.cu``) from the int32
code columns in HBM to the key-major interval table, never materialising
Python ``IntervalRow`` objects. ``ChunkerIndex`` exposes the reference's
duck type (``index.py:50-85``) by decoding device tables lazily.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from .catalog import ColumnarCatalog, FilterPredicate
from .codec import KeyCodec
from .errors import QueryError
from .mixtures import MixtureKey, sorted_keys


class DeviceCatalog:
    """A ``ColumnarCatalog`` uploaded to HBM (columns in property-name order)."""

    def __init__(self, host: ColumnarCatalog, columns=None, nullable=None, device=None, tuples=None):
        """``tuples`` = (int32 row-tuple code column in HBM, int32[T, P] tuple
        table in property-name order) selects the row-tuple layout
        (``encode_row_tuples`` / ``encode_row_tuples_device``): stage 1 then
        scans one 4-byte column instead of one per property."""
        import torch

        self.host = host
        self.device = torch.device(device or "cuda")
        props = sorted(host.vocab)
        self.tuple_codes = self.tuple_table = None
        if tuples is not None:
            codes, table = tuples
            if codes.dtype not in (torch.int32, torch.int16):
                raise ValueError("tuple codes must be int32, or int16 holding u16 codes")
            self.tuple_codes = codes.contiguous()
            self.tuple_table = np.ascontiguousarray(table, dtype=np.int32)
            if self.tuple_table.ndim != 2 or self.tuple_table.shape[1] != len(props):
                raise ValueError("tuple table must be [T, n_props]")
            self.columns = None
            if nullable is None:
                nullable = {p: bool((self.tuple_table[:, j] < 0).any()) for j, p in enumerate(props)}
        else:
            if columns is None:
                columns = {p: torch.from_numpy(host.columns[p]).to(self.device) for p in props}
            self.columns = {p: columns[p].contiguous() for p in props}
        if nullable is None:
            nullable = {p: bool((self.columns[p] < 0).any().item()) for p in props}
        self.nullable = nullable
        self.codec = KeyCodec.build(host.vocab, nullable)
        self.file_offsets = torch.from_numpy(np.asarray(host.file_offsets, dtype=np.int64)).to(self.device)
        ds = np.asarray(host.file_ds)
        if len(ds) > 1 and np.any(np.diff(ds) < 0):
            raise ValueError("dataset ids must be nondecreasing in file-id order (registration order)")
        self.file_ds = np.ascontiguousarray(ds, dtype=np.int32)
        self.file_ids = np.ascontiguousarray(host.file_ids, dtype=np.int64)
        self._strings = self.codec.key_strings()

    @staticmethod
    def encode_row_tuples_device(columns: dict, cards, narrow: bool = True) -> tuple:
        """Device twin of ``catalog.encode_row_tuples`` for HBM-resident
        columns ({prop: int32 tensor}, property-name order): (codes in HBM,
        int32[T, P] host tuple table). With ``narrow`` and <= 65,536 tuples
        the codes are u16 (stored as int16: half the bytes to scan / upload)."""
        import torch

        from .catalog import _tuple_radix, row_tuple_table

        props = sorted(columns)
        mult = _tuple_radix(cards)
        r = None
        for p, m in zip(props, mult):
            t = (columns[p].to(torch.int64) + 1) * m
            r = t if r is None else r.add_(t)
        u, inv = torch.unique(r, sorted=True, return_inverse=True)
        del r
        if u.numel() >= 1 << 31:
            raise ValueError("more than 2^31 distinct row tuples")
        table = row_tuple_table(u.cpu().numpy(), cards)
        if narrow and u.numel() <= 1 << 16:
            return torch.where(inv >= 1 << 15, inv - (1 << 16), inv).to(torch.int16), table
        return inv.to(torch.int32), table

    @staticmethod
    def from_reference(cat, device=None, layout: str = "tuples") -> "DeviceCatalog":
        """A reference ``MetadataCatalog`` in HBM. ``layout="tuples"`` (the
        drop-in's default) dictionary-encodes the rows once into one u16 (or
        int32) row-tuple column, the layout stage 1 scans fastest;
        ``"columns"`` keeps one int32 column per property."""
        host = ColumnarCatalog.from_reference(cat)
        if layout == "tuples":
            return DeviceCatalog.with_row_tuples(host, device)
        return DeviceCatalog(host, device=device)

    @staticmethod
    def with_row_tuples(host: ColumnarCatalog, device=None) -> "DeviceCatalog":
        """Upload ``host`` and encode its rows into one row-tuple column on
        the device (``encode_row_tuples_device``); the per-property columns
        are dropped after the encoding."""
        import torch

        dev = torch.device(device or "cuda")
        props = sorted(host.vocab)
        if host.n_samples == 0 or not props:
            return DeviceCatalog(host, device=dev)
        cols = {p: torch.from_numpy(np.ascontiguousarray(host.columns[p], dtype=np.int32)).to(dev) for p in props}
        nullable = {p: bool((cols[p] < 0).any().item()) for p in props}
        codes, table = DeviceCatalog.encode_row_tuples_device(cols, [len(host.vocab[p]) for p in props])
        del cols
        return DeviceCatalog(host, nullable=nullable, device=dev, tuples=(codes, table))

    @property
    def n_samples(self) -> int:
        return self.host.n_samples

    def descriptor(self, preds: list[FilterPredicate]):
        """C struct for mx_index_build; returns (desc, keepalive). Cached per
        predicate list: a catalog serves many jobs with the same filters."""
        key = tuple(preds)
        cache = self.__dict__.setdefault("_desc_cache", {})
        hit = cache.get(key)
        if hit is None:
            if len(cache) > 64:
                cache.clear()
            hit = cache[key] = self._descriptor(preds)
        return hit

    def _descriptor(self, preds: list[FilterPredicate]):
        codec = self.codec
        if self.tuple_codes is not None:
            lut, lut_off = codec.tuple_luts(self.host, preds, self.tuple_table)
            cols = (C.c_void_p * 1)(self.tuple_codes.data_ptr())
        else:
            lut, lut_off = codec.luts(self.host, preds)
            cols = (C.c_void_p * len(codec.props))(*[self.columns[p].data_ptr() for p in codec.props])
        blob, soff, sbase = self._strings
        keep = dict(
            lut=np.ascontiguousarray(lut), lut_off=np.ascontiguousarray(lut_off), cols=cols,
            shift=np.array(codec.shift, dtype=np.uint32), width=np.array(codec.width, dtype=np.uint32),
            blob=np.frombuffer(blob, dtype=np.uint8).copy() if blob else np.zeros(1, np.uint8),
            soff=soff, sbase=sbase,
        )
        P = C.POINTER
        d = _lib.CatalogDesc()
        d.n_props = len(codec.props)
        d.columns = C.cast(cols, P(C.c_void_p))
        d.lut = keep["lut"].ctypes.data_as(P(C.c_uint32))
        d.lut_offsets = keep["lut_off"].ctypes.data_as(P(C.c_int32))
        d.n_samples = self.host.n_samples
        d.n_files = self.host.n_files
        d.file_offsets = self.file_offsets.data_ptr()
        d.file_ds = self.file_ds.ctypes.data_as(P(C.c_int32))
        d.file_ids = self.file_ids.ctypes.data_as(P(C.c_int64))
        d.key_bits = codec.key_bits
        d.rank_mask = codec.rank_mask
        d.field_shift = keep["shift"].ctypes.data_as(P(C.c_uint32))
        d.field_width = keep["width"].ctypes.data_as(P(C.c_uint32))
        d.key_strings = keep["blob"].ctypes.data_as(P(C.c_uint8))
        d.key_string_offsets = keep["soff"].ctypes.data_as(P(C.c_int64))
        d.key_string_base = keep["sbase"].ctypes.data_as(P(C.c_int32))
        if self.tuple_codes is not None:
            d.n_columns = 1
            d.n_key_pieces = len(soff) - 1
            d.column_bytes = self.tuple_codes.element_size()
        return d, keep


class ChunkerIndex:
    """Immutable device index; same duck type as the reference ``ChunkerIndex``."""

    def __init__(self, handle: int, catalog: DeviceCatalog, stream=None):
        self._h = C.c_void_p(handle)
        self.catalog = catalog
        self.codec = catalog.codec
        self.stream = stream
        self._sizes = None  # read on first use: the build returns before its sizes reach the host
        self._keys = None
        self._nested = None
        self._counts = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._handle is not None:
            _lib._handle.mx_index_free(h)
            self._h = None

    def _size(self, i: int) -> int:
        if self._sizes is None:
            k, b, n_iv, n = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64())
            _lib.check(_lib.lib().mx_index_sizes(self._h, C.byref(k), C.byref(b), C.byref(n_iv), C.byref(n)))
            self._sizes = (k.value, b.value, n_iv.value, n.value)
        return self._sizes[i]

    n_keys = property(lambda self: self._size(0))
    n_blocks = property(lambda self: self._size(1))
    n_intervals = property(lambda self: self._size(2))
    n_samples = property(lambda self: self._size(3))

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # ---------------------------------------------------------- exports
    def packed_keys(self) -> tuple[np.ndarray, np.ndarray]:
        packed = np.zeros(self.n_keys, dtype=np.uint32)
        samples = np.zeros(self.n_keys, dtype=np.int64)
        if self.n_keys:
            _lib.check(_lib.lib().mx_index_export_keys(self._h, _lib.ptr(packed), _lib.ptr(samples)))
        return packed, samples

    def interval_table(self) -> dict[str, np.ndarray]:
        """Flat (key rank, ds, file id, start, end) in index order."""
        n = self.n_intervals
        out = dict(key=np.zeros(n, np.uint32), ds=np.zeros(n, np.int32), fid=np.zeros(n, np.int64),
                   start=np.zeros(n, np.uint32), end=np.zeros(n, np.uint32))
        if n:
            _lib.check(_lib.lib().mx_index_export_intervals(
                self._h, *(_lib.ptr(out[x]) for x in ("key", "ds", "fid", "start", "end"))))
        return out

    def table(self) -> list[tuple]:
        """[(key canonical string, ds, fid, start, end)] -- the parity form."""
        keys = self.component_keys()
        ks = [k.canonical_string() for k in keys]
        t = self.interval_table()
        return [(ks[r], int(d), int(f), int(a), int(b))
                for r, d, f, a, b in zip(t["key"], t["ds"], t["fid"], t["start"], t["end"])]

    def file_table(self) -> tuple[np.ndarray, np.ndarray]:
        """(dataset ids, file ids) of the index's file table (the global table
        for a file-sharded index)."""
        sh = getattr(self, "shard", None) or getattr(self, "partition", None)
        if sh is not None:
            return sh.file_ds, sh.file_ids
        return self.catalog.file_ds, self.catalog.file_ids

    def file_string_ranks(self) -> np.ndarray:
        """u32 rank of every file in (str(ds), str(fid)) order: the order in
        which canonical chunk JSON (sort_keys) lists datasets and files."""
        if getattr(self, "_frank", None) is None:
            ds, fid = self.file_table()
            order = np.lexsort((np.asarray(fid).astype(str), np.asarray(ds).astype(str)))
            rank = np.empty(len(order), np.uint32)
            rank[order] = np.arange(len(order), dtype=np.uint32)
            self._frank = rank
        return self._frank

    # ---------------------------------------------------------- reference duck type
    def component_keys(self) -> list[MixtureKey]:
        if self._keys is None:
            packed, samples = self.packed_keys()
            self._keys = [self.codec.decode(int(p)) for p in packed]
            self._counts = samples
        return list(self._keys)

    def _nested_index(self):
        if self._nested is None:
            keys = self.component_keys()
            t = self.interval_table()
            nested: dict = {}
            for r, d, f, a, b in zip(t["key"].tolist(), t["ds"].tolist(), t["fid"].tolist(),
                                     t["start"].tolist(), t["end"].tolist()):
                nested.setdefault(keys[r], {}).setdefault(d, {}).setdefault(f, []).append((a, b))
            self._nested = nested
        return self._nested

    @property
    def _index(self):
        return self._nested_index()

    def entries(self, key: MixtureKey):
        return self._nested_index().get(key, {})

    def matching_keys(self, mixture_key: MixtureKey) -> list[MixtureKey]:
        return [k for k in self.component_keys() if mixture_key.matches(k)]

    def cursor(self, key: MixtureKey, seed: int) -> "RangeCursor":
        """``ChunkerIndex.cursor`` (``index.py:78-79``): the key's RangeCursor for
        a job seed. The seeded layout is the one the device generator builds
        (``csrc/cursor.cu``); take / state are the reference's bookkeeping."""
        from .chunks import ChunkGenerator

        gens = self.__dict__.setdefault("_cursor_gens", {})
        gen = gens.get(int(seed))
        if gen is None:
            gen = gens[int(seed)] = ChunkGenerator(self, int(seed))
        return RangeCursor(key, gen.cursor_ranges(key), int(seed))

    def key_sample_counts(self) -> dict[MixtureKey, int]:
        keys = self.component_keys()
        return {k: int(n) for k, n in zip(keys, self._counts)}

    def total_samples(self) -> int:
        return int(self.n_samples)

    def __contains__(self, key) -> bool:
        return key in set(self.component_keys())

    def __len__(self) -> int:  # an empty index is falsy, like an empty row list
        return int(self.n_intervals)

    def __eq__(self, other) -> bool:
        mine = self._nested_index()
        theirs = getattr(other, "_index", None)
        if theirs is None:
            return False
        if isinstance(other, ChunkerIndex):
            return self.table() == other.table()
        conv = {MixtureKey(tuple(getattr(k, "entries", k))): v for k, v in theirs.items()}
        return mine == conv

    __hash__ = None


class RangeCursor:
    """One key's remaining samples as ranges in the seeded order
    (``index.py:118-189``): ``take(n)``, ``depleted``, ``state_dict`` /
    ``load_state``; ``_ranges`` is the device-computed layout."""

    def __init__(self, key: MixtureKey, ranges: list[tuple[int, int, int, int]], seed: int):
        self.key = key
        self.seed = seed
        self._ranges = list(ranges)
        self._pos = 0
        self._offset = 0
        self.remaining_total = sum(e - s for _, _, s, e in self._ranges)

    def take(self, n: int) -> list[tuple[int, int, int, int]]:
        if n < 1:
            raise ValueError("take() needs n >= 1")
        out = []
        need = n
        while need > 0 and self._pos < len(self._ranges):
            ds, fid, start, end = self._ranges[self._pos]
            cur = start + self._offset
            if end - cur <= need:
                out.append((ds, fid, cur, end))
                need -= end - cur
                self._pos += 1
                self._offset = 0
            else:
                out.append((ds, fid, cur, cur + need))
                self._offset += need
                need = 0
        self.remaining_total -= n - need
        return out

    @property
    def depleted(self) -> bool:
        return self.remaining_total == 0

    def state_dict(self) -> dict:
        return {"pos": self._pos, "offset": self._offset}

    def load_state(self, state) -> None:
        self._pos = int(state["pos"])
        self._offset = int(state["offset"])
        consumed = sum(e - s for _, _, s, e in self._ranges[: self._pos]) + self._offset
        self.remaining_total = sum(e - s for _, _, s, e in self._ranges) - consumed


class RowsCodec:
    """Key codec of an index built from explicit rows (``build_index``): one
    field holding the key's 1-based rank in ``sort_key`` order, so the packed
    order is the key order; the keys themselves are the caller's objects
    (reference ``MixtureKey``s under the drop-in)."""

    props = ["\0key"]

    def __init__(self, keys: list):
        self.keys = keys
        self.key_bits = max(1, len(keys).bit_length())
        if self.key_bits > 31:
            raise NotImplementedError(f"{len(keys)} distinct keys (> 2^31 - 1)")
        self.shift, self.width = [0], [self.key_bits]
        self._memo = {}

    def decode(self, packed: int):
        return self.keys[int(packed) - 1]

    def key_strings(self):
        hit = self._memo.get("strings")
        if hit is None:
            blobs = [k.canonical_string().encode("utf-8") for k in self.keys]
            off = np.zeros(len(blobs) + 1, dtype=np.int64)
            off[1:] = np.cumsum([len(b) for b in blobs]) if blobs else []
            hit = self._memo["strings"] = (b"".join(blobs), off, np.zeros(1, np.int32))
        return hit

    def allow_table(self, mkeys):
        """Bit r of mixture key m = component key rank r matches m
        (``mixtures.py:100-109``); bit 0 (no key) is never held."""
        key = ("allow", tuple(tuple(getattr(k, "entries", ())) for k in mkeys))
        hit = self._memo.get(key)
        if hit is None:
            words = (len(self.keys) + 1 + 31) // 32
            bits = np.zeros((len(mkeys), words * 32), dtype=bool)
            for m, mk in enumerate(mkeys):
                bits[m, 1:len(self.keys) + 1] = [mk.matches(k) for k in self.keys]
            table = np.packbits(bits.reshape(len(mkeys), words, 32)[:, :, ::-1], axis=2).view(">u4")
            hit = (table.reshape(len(mkeys), words).astype(np.uint32), np.zeros(1, np.int32), words)
            if len(self._memo) > 256:
                self._memo.clear()
            self._memo[key] = hit
        return hit


class _RowsSource:
    """The "catalog" of a rows-built index: its file table and codec."""

    def __init__(self, codec: RowsCodec, file_ds: np.ndarray, file_ids: np.ndarray, device):
        self.codec = codec
        self.file_ds = file_ds
        self.file_ids = file_ids
        self.device = device


def build_index(rows, workers: int = 1, stream=None) -> ChunkerIndex:
    """``build_index(rows, workers)`` (``index.py:88-115``) on the GPU.

    ``rows`` are ``IntervalRow``-like objects (``dataset_id, file_id, key,
    start, end``) or a device ``ChunkerIndex`` (returned as is: the catalog
    seam already built it). Rows are packed into flat arrays (the one host
    pass over the caller's Python objects), then sorted by (key, file,
    start), checked (empty / overlapping -> ``IndexBuildError``) and merged
    on the device. ``workers`` is accepted for signature parity; the result
    never depends on it (nor on the row order)."""
    import torch

    if isinstance(rows, ChunkerIndex):
        return rows
    rows = list(rows)
    keyset = {}
    for r in rows:
        keyset.setdefault(r.key, None)
    keys = sorted(keyset, key=MixtureKey.sort_key)
    rank = {k: i + 1 for i, k in enumerate(keys)}
    n = len(rows)
    ds = np.fromiter((r.dataset_id for r in rows), dtype=np.int64, count=n)
    fid = np.fromiter((r.file_id for r in rows), dtype=np.int64, count=n)
    st = np.fromiter((r.start for r in rows), dtype=np.int64, count=n)
    en = np.fromiter((r.end for r in rows), dtype=np.int64, count=n)
    kr = np.fromiter((rank[r.key] for r in rows), dtype=np.uint32, count=n)
    if n and (min(st.min(), en.min()) < 0 or max(st.max(), en.max()) >= 1 << 32):
        raise NotImplementedError("interval bounds outside [0, 2^32)")
    if n and (ds.min() < -(1 << 31) or ds.max() >= 1 << 31):
        raise NotImplementedError("dataset ids outside int32")
    pairs = np.unique(np.stack([ds, fid], axis=1), axis=0) if n else np.zeros((0, 2), np.int64)
    file_ix = np.zeros(n, dtype=np.uint32)
    if n:  # index of (ds, fid) in the (ds, fid)-sorted file table
        order = np.lexsort((fid, ds))
        brk = np.ones(n, dtype=bool)
        brk[1:] = (ds[order][1:] != ds[order][:-1]) | (fid[order][1:] != fid[order][:-1])
        file_ix[order] = (np.cumsum(brk) - 1).astype(np.uint32)
    codec = RowsCodec(keys)
    f_ds = np.ascontiguousarray(pairs[:, 0], dtype=np.int32)
    f_ids = np.ascontiguousarray(pairs[:, 1], dtype=np.int64)
    blob, soff, _ = codec.key_strings()
    keep = dict(k=kr, f=file_ix, s=np.ascontiguousarray(st, np.uint32), e=np.ascontiguousarray(en, np.uint32),
                blob=np.frombuffer(blob, dtype=np.uint8).copy() if blob else np.zeros(1, np.uint8), soff=soff)
    P = C.POINTER
    d = _lib.RowsDesc()
    d.n_rows = n
    d.key = keep["k"].ctypes.data_as(P(C.c_uint32))
    d.file = keep["f"].ctypes.data_as(P(C.c_uint32))
    d.start = keep["s"].ctypes.data_as(P(C.c_uint32))
    d.end = keep["e"].ctypes.data_as(P(C.c_uint32))
    d.n_files = len(f_ds)
    d.file_ds = f_ds.ctypes.data_as(P(C.c_int32))
    d.file_ids = f_ids.ctypes.data_as(P(C.c_int64))
    d.n_keys = len(keys)
    d.key_bits = codec.key_bits
    d.key_strings = keep["blob"].ctypes.data_as(P(C.c_uint8))
    d.key_string_offsets = keep["soff"].ctypes.data_as(P(C.c_int64))
    L = _lib.lib()
    out = C.c_void_p()
    _lib.check(L.mx_index_build_rows(C.byref(d), C.c_void_p(_lib.stream_ptr(stream)), C.byref(out)))
    src = _RowsSource(codec, f_ds, f_ids, torch.device("cuda", torch.cuda.current_device()))
    return ChunkerIndex(out.value, src, stream)


def build_index_from_catalog(catalog, predicates: Sequence = (), stream=None) -> ChunkerIndex:
    """Fused filter + intervals + index on the GPU.

    ``catalog`` is a ``DeviceCatalog``, a ``ColumnarCatalog`` (uploaded), or a
    reference ``MetadataCatalog`` (adapted then uploaded). Errors follow the
    reference: unknown property / empty catalog / un-keyable sample ->
    ``QueryError``.
    """
    if not isinstance(catalog, DeviceCatalog):
        if not isinstance(catalog, ColumnarCatalog):
            if not getattr(catalog, "_files", None):
                raise QueryError("catalog is empty")
            catalog = ColumnarCatalog.from_reference(catalog)
        catalog = DeviceCatalog(catalog)
    if catalog.host.n_files == 0:
        raise QueryError("catalog is empty")
    preds = catalog.host.validated(predicates)
    desc, keep = catalog.descriptor(preds)
    L = _lib.lib()
    out = C.c_void_p()
    _lib.check(L.mx_index_build(C.byref(desc), C.c_void_p(_lib.stream_ptr(stream)), C.byref(out)))
    return ChunkerIndex(out.value, catalog, stream)
