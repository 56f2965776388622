"""Chunk generation behind the reference's ``ChunkGenerator`` API.

``ChunkGenerator(index, seed)`` lays out every component's RangeCursor and the
seeded component order on the GPU (``csrc/cursor.cu``); ``generate(spec)``
returns exactly the chunk the reference's ``ChunkGenerator.generate``
(``chunks.py:194-230``) returns for the same index, seed and call sequence.

Chunks are planned and cut on the device in batches (``csrc/stage2.cu``).
Because generation is a deterministic function of (cursor state, spec), a
generator may plan ahead while the caller keeps passing the same spec; the
spec is still re-read on every call: a different spec, or a
checkpoint request, rewinds the device cursors to the last handed-out chunk
by re-planning exactly that many chunks from the batch start.
"""

from __future__ import annotations

import ctypes as C
from typing import Mapping

import numpy as np

from . import _lib
from .errors import MixtureError
from .index import ChunkerIndex
from .mixtures import MixtureKey, MixtureSpec, sorted_keys
from .seeding import canonical_json_bytes, derive_seed, hash_message

_CHUNK_VERSION = 1

RangeMap = dict  # MixtureKey -> {ds: {fid: [(start, end)]}}


class _ChunkBase:
    """Placeholder base: ``dropin.install`` swaps it for the reference's
    ``Chunk`` (a class whose only base is ``object`` cannot be re-based)."""


class Chunk(_ChunkBase):
    """Sample pointers of one chunk + its mixture snapshot (``chunks.py:26-106``).

    A chunk handed out of a device batch is LAZY: ``data`` (the nested
    key -> ds -> fid -> ranges dict) is built from the batch's host arrays
    only when someone reads it, and ``serialize()`` returns the canonical
    bytes built on the device -- the server (``server.py:143-163``) only
    ever calls ``serialize()``, so serving a chunk costs no Python dicts."""

    def __init__(self, chunk_id: int, data: RangeMap, seed: int, mixture: MixtureSpec | None = None):
        self.chunk_id = chunk_id
        self._data = data
        self._src = None  # (batch, index) of a lazy chunk
        self.seed = seed
        self.mixture = mixture
        self._device_bytes = None

    @property
    def data(self) -> RangeMap:
        if self._data is None and self._src is not None:
            batch, i = self._src
            self._data = batch._chunk_data(i)
            dev = self._device_bytes
            if dev is not None and dev[1] is None:
                self._device_bytes = (dev[0], self._data, dev[2])
        return self._data

    @data.setter
    def data(self, value: RangeMap) -> None:
        self._data = value
        self._src = None

    def samples_per_key(self) -> dict[MixtureKey, int]:
        return {
            k: sum(e - s for files in ds.values() for rs in files.values() for s, e in rs)
            for k, ds in self.data.items()
        }

    def total_samples(self) -> int:
        return sum(self.samples_per_key().values())

    def to_json(self) -> dict:
        body = {}
        for key in sorted_keys(self.data):
            datasets = self.data[key]
            body[key.canonical_string()] = {
                str(ds): {str(fid): [[s, e] for s, e in rs] for fid, rs in sorted(files.items())}
                for ds, files in sorted(datasets.items())
            }
        return {
            "version": _CHUNK_VERSION,
            "chunk_id": self.chunk_id,
            "seed": self.seed,
            "mixture": self.mixture.to_json() if self.mixture else None,
            "data": body,
        }

    @staticmethod
    def from_json(payload: Mapping) -> "Chunk":
        if payload.get("version") != _CHUNK_VERSION:
            raise MixtureError(f"unsupported chunk version {payload.get('version')!r}")
        data: RangeMap = {}
        for ks, datasets in payload["data"].items():
            data[MixtureKey.parse(ks)] = {
                int(ds): {int(fid): [(int(s), int(e)) for s, e in rs] for fid, rs in files.items()}
                for ds, files in datasets.items()
            }
        mix = payload.get("mixture")
        return Chunk(int(payload["chunk_id"]), data, int(payload["seed"]),
                     MixtureSpec.from_json(mix) if mix else None)

    def serialize(self) -> bytes:
        # bytes produced on the device for a planned batch (csrc/serialize.cu),
        # valid while data (still lazy, or the object built from the same
        # arrays) and mixture are the ones they were built from
        dev = self._device_bytes
        if dev is not None and dev[2] is self.mixture and (
                (self._data is None and self._src is not None) or dev[1] is self._data):
            return dev[0]
        return canonical_json_bytes(self.to_json())

    @staticmethod
    def deserialize(blob: bytes) -> "Chunk":
        import json

        return Chunk.from_json(json.loads(blob.decode("utf-8")))

    def __eq__(self, other) -> bool:
        return hasattr(other, "serialize") and self.serialize() == other.serialize()

    __hash__ = None

    def __repr__(self) -> str:
        return f"Chunk(id={self.chunk_id}, samples={ {str(k): n for k, n in self.samples_per_key().items()} })"


def redistribute_best_effort(remaining, shortfall_key, progress_keys, weights):
    """Host form of the reference helper (``chunks.py:109-130``); the device
    planner performs the same step inside ``plan_kernel``."""
    from .mixtures import apportion

    shortfall = remaining.get(shortfall_key, 0)
    targets = sorted_keys(k for k in progress_keys if k != shortfall_key)
    if not targets:
        raise MixtureError("no keys left to absorb the shortfall")
    if shortfall > 0:
        for k, extra in apportion({k: weights[k] for k in targets}, shortfall).items():
            remaining[k] = remaining.get(k, 0) + extra
    remaining[shortfall_key] = 0
    return remaining


_TORCH_OF = {np.int64: "int64", np.uint64: "uint64", np.int32: "int32", np.uint32: "uint32"}


def _pinned(n: int, dtype) -> np.ndarray:
    """Host array in page-locked memory (torch's caching host allocator), so
    the result read-back is a direct DMA instead of a staged pageable copy."""
    import torch

    if n < 4096:
        return np.zeros(n, dtype)
    t = torch.empty(n, dtype=getattr(torch, _TORCH_OF[dtype]), pin_memory=True)
    return t.numpy()


def _pinned_bytes(n: int) -> np.ndarray:
    import torch

    if n < 4096:
        return np.zeros(max(n, 1), np.uint8)
    return torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()


class ChunkBatch:
    """Device CSR of consecutive chunks (valid until the generator plans again)."""

    def __init__(self, gen: "ChunkGenerator", n_chunks: int, n_ranges: int, mkeys, spec, arbitrary_size):
        self.n_chunks = n_chunks
        self.n_ranges = n_ranges
        self.mkeys = mkeys
        self.spec = spec
        self.arbitrary_size = arbitrary_size
        self.arbitrary = arbitrary_size is not None
        self.exhausted = False
        self.report = None
        self._gen = gen
        self._host = None

    def to_host(self) -> dict[str, np.ndarray]:
        if self._host is None:
            n, r = self.n_chunks, self.n_ranges
            h = dict(off=_pinned(n + 1, np.int64), ids=_pinned(n, np.int64), seeds=_pinned(n, np.uint64),
                     mkey=_pinned(r, np.uint32), ds=_pinned(r, np.int32), fid=_pinned(r, np.int64),
                     start=_pinned(r, np.uint32), end=_pinned(r, np.uint32))
            _lib.check(_lib.lib().mx_gen_result_copy(
                self._gen._h, *(_lib.ptr(h[x]) for x in ("off", "ids", "seeds", "mkey", "ds", "fid", "start", "end"))))
            self._host = h
        return self._host

    def serialize_all(self) -> tuple[bytes, np.ndarray]:
        """Canonical bytes of every chunk of the batch, built on the device
        (``csrc/serialize.cu``): one blob + offsets [n_chunks + 1]; chunk i is
        ``blob[off[i]:off[i+1]]`` == ``self.chunk(i).serialize()``."""
        import json

        L = _lib.lib()
        keys = self._gen.index.component_keys() if self.arbitrary else list(self.mkeys)
        strs = [k.canonical_string() for k in keys]
        kj = [json.dumps(x, ensure_ascii=True).encode("ascii") for x in strs]
        koff = np.zeros(len(kj) + 1, np.int64)
        koff[1:] = np.cumsum([len(b) for b in kj])
        order = sorted(range(len(strs)), key=strs.__getitem__)
        krank = np.zeros(len(strs), np.uint32)
        krank[order] = np.arange(len(strs), dtype=np.uint32)
        mix = b"null" if self.arbitrary or self.spec is None else canonical_json_bytes(self.spec.to_json())
        frank = self._gen.index.file_string_ranks()
        blob_k = np.frombuffer(b"".join(kj) or b"\0", dtype=np.uint8)
        blob_m = np.frombuffer(mix, dtype=np.uint8)
        d = _lib.JsonDesc()
        P = C.POINTER
        d.n_keys = len(kj)
        d.key_json = blob_k.ctypes.data_as(P(C.c_uint8))
        d.key_json_off = koff.ctypes.data_as(P(C.c_int64))
        d.key_rank = krank.ctypes.data_as(P(C.c_uint32))
        d.file_rank = frank.ctypes.data_as(P(C.c_uint32))
        d.mixture_json = blob_m.ctypes.data_as(P(C.c_uint8))
        d.mixture_len = len(mix)
        total = C.c_int64()
        _lib.check(L.mx_gen_result_json(self._gen._h, C.byref(d), C.byref(total), 0))
        off = _pinned(self.n_chunks + 1, np.int64)
        buf = _pinned_bytes(total.value)
        _lib.check(L.mx_gen_result_json_copy(self._gen._h, _lib.ptr(buf), _lib.ptr(off)))
        return buf[: total.value].tobytes(), off

    DEVICE_JSON_MIN = 64  # batches at least this large serialise on the device

    def chunk(self, i: int, mixture=None) -> Chunk:
        """Chunk i of the batch; ``mixture`` (the spec in force) defaults to the
        batch's spec. Large batches carry device-built canonical bytes and a
        lazy ``data``."""
        h = self.to_host()
        c = Chunk(int(h["ids"][i]), None, int(h["seeds"][i]), None if self.arbitrary else self.spec)
        c._src = (self, i)
        if mixture is not None:
            c.mixture = mixture
        if self.n_chunks >= self.DEVICE_JSON_MIN and self._json_ok() and (self.arbitrary or c.mixture is self.spec):
            if getattr(self, "_json", None) is None:
                self._json = self.serialize_all()
            blob, off = self._json
            c._device_bytes = (blob[int(off[i]):int(off[i + 1])], None, c.mixture)
        return c

    JSON_MAX_RANGES = 2048  # csrc/serialize.cu JS_CAP: larger chunks sort beyond shared memory

    def _json_ok(self) -> bool:
        """Device JSON ranks keys in 16 bits and sorts a chunk's ranges in
        shared memory (csrc/serialize.cu); wider key sets or chunks of more
        than JSON_MAX_RANGES ranges serialise on the host."""
        ok = getattr(self, "_json_ok_v", None)
        if ok is None:
            n = len(self._gen.index.component_keys()) if self.arbitrary else len(self.mkeys)
            off = self.to_host()["off"]
            ok = n < 65536 and (self.n_chunks == 0 or int(np.diff(off).max()) <= self.JSON_MAX_RANGES)
            self._json_ok_v = ok
        return ok

    def _chunk(self, i: int) -> Chunk:
        c = self.chunk(i)
        c.data  # materialise
        return c

    def _chunk_data(self, i: int) -> RangeMap:
        h = self.to_host()
        a, b = int(h["off"][i]), int(h["off"][i + 1])
        data: RangeMap = {}
        keys = self._gen.index.component_keys() if self.arbitrary else self.mkeys
        for m, d, f, s, e in zip(h["mkey"][a:b].tolist(), h["ds"][a:b].tolist(), h["fid"][a:b].tolist(),
                                 h["start"][a:b].tolist(), h["end"][a:b].tolist()):
            data.setdefault(keys[m], {}).setdefault(d, {}).setdefault(f, []).append((s, e))
        return data


class ChunkGenerator:
    """Device-backed generator with the reference's interface (``chunks.py:133-272``)."""

    MAX_BATCH = 1 << 16

    def __init__(self, index: ChunkerIndex, seed: int, stream=None):
        self.index = index
        self.seed = int(seed)
        self.stream = stream
        L = _lib.lib()
        cur = hash_message(self.seed, "cursor")
        chk = hash_message(self.seed, "chunk")
        out = C.c_void_p()
        _lib.check(L.mx_gen_create(index.handle, cur, len(cur), chk, len(chk),
                                   derive_seed(self.seed, "component-order"),
                                   C.c_void_p(_lib.stream_ptr(stream)), C.byref(out)))
        self._h = out
        if getattr(index, "partition", None) is not None:  # collective: block offsets from the key owners
            from .parallel import attach_partition

            attach_partition(self)
        self.last_report: dict | None = None
        self._batch: ChunkBatch | None = None  # planned ahead, not all handed out
        self._served = 0
        self._batch_start_state = None
        self._batch_start_id = 0
        self._look_ahead = 1
        self._next_id = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._handle is not None:
            _lib._handle.mx_gen_free(h)
            self._h = None

    # ---------------------------------------------------------- properties
    @property
    def next_chunk_id(self) -> int:
        return self._next_id

    @next_chunk_id.setter
    def next_chunk_id(self, v: int) -> None:
        self._rewind()
        self._next_id = int(v)
        _lib.check(_lib.lib().mx_gen_set_next_chunk_id(self._h, self._next_id))

    @property
    def _component_order(self) -> list[MixtureKey]:
        keys = self.index.component_keys()
        order = np.zeros(len(keys), dtype=np.uint32)
        if len(keys):
            _lib.check(_lib.lib().mx_gen_component_order(self._h, _lib.ptr(order)))
        return [keys[i] for i in order.tolist()]

    def cursor_ranges(self, key: MixtureKey) -> list[tuple[int, int, int, int]]:
        """RangeCursor._ranges of one component key (index.py:134-144)."""
        r = self.index.component_keys().index(key)
        n = C.c_int64()
        L = _lib.lib()
        _lib.check(L.mx_gen_cursor_ranges(self._h, r, C.byref(n), 0, 0, 0, 0, 0))
        ds, fid = np.zeros(n.value, np.int32), np.zeros(n.value, np.int64)
        s, e = np.zeros(n.value, np.uint32), np.zeros(n.value, np.uint32)
        _lib.check(L.mx_gen_cursor_ranges(self._h, r, C.byref(n), _lib.ptr(ds), _lib.ptr(fid), _lib.ptr(s),
                                          _lib.ptr(e), n.value))
        return list(zip(ds.tolist(), fid.tolist(), s.tolist(), e.tolist()))

    # ---------------------------------------------------------- planning
    def _mixture_desc(self, spec: MixtureSpec):
        mkeys = spec.keys()
        sig = tuple(k.entries for k in mkeys)
        cached = getattr(self, "_allow_cache", None)
        if cached is None or cached[0] != sig:  # ADO re-plans with new weights, same keys
            cached = (sig, *self.index.codec.allow_table(mkeys))
            self._allow_cache = cached
        _, allow, base, words = cached
        w = np.array([spec.weights[k] for k in mkeys], dtype=np.float64)
        keep = (np.ascontiguousarray(allow), np.ascontiguousarray(base), w)
        d = _lib.MixtureDesc()
        P = C.POINTER
        d.n_mkeys = len(mkeys)
        d.allow = keep[0].ctypes.data_as(P(C.c_uint32))
        d.allow_words = words
        d.allow_base = keep[1].ctypes.data_as(P(C.c_int32))
        d.weights = keep[2].ctypes.data_as(P(C.c_double))
        d.chunk_size = spec.chunk_size
        d.strict = int(spec.strict)
        return d, keep, mkeys

    def _cursor_state(self):
        if getattr(self.index, "partition", None) is not None:
            raise NotImplementedError("cursor checkpoints of a key-partitioned generator (use the file-sharded "
                                      "index, parallel.build_sharded_index, for reference-format states)")
        k = self.index.n_keys
        pos, off = np.zeros(k, np.int64), np.zeros(k, np.int64)
        if k:
            _lib.check(_lib.lib().mx_gen_get_cursors(self._h, _lib.ptr(pos), _lib.ptr(off)))
        sh = getattr(self.index, "shard", None)
        if sh is not None:  # a frontier inside another rank's block is answered by its owner
            from .parallel import _max_allreduce

            both = _max_allreduce(np.concatenate([pos, off]), sh.group, self.index.catalog.device)
            pos, off = both[:k], both[k:]
        return pos, off

    def _set_cursor_state(self, pos, off) -> None:
        if getattr(self.index, "partition", None) is not None:
            raise NotImplementedError("cursor checkpoints of a key-partitioned generator")
        if not self.index.n_keys:
            return
        L = _lib.lib()
        pos = np.ascontiguousarray(pos, np.int64)
        off = np.ascontiguousarray(off, np.int64)
        sh = getattr(self.index, "shard", None)
        if sh is None:
            _lib.check(L.mx_gen_set_cursors(self._h, _lib.ptr(pos), _lib.ptr(off)))
            return
        from .parallel import _max_allreduce

        used = np.zeros(self.index.n_keys, np.int64)
        _lib.check(L.mx_gen_cursor_to_consumed(self._h, _lib.ptr(pos), _lib.ptr(off), _lib.ptr(used)))
        used = np.ascontiguousarray(_max_allreduce(used, sh.group, self.index.catalog.device))
        _lib.check(L.mx_gen_set_consumed(self._h, _lib.ptr(used)))

    def _plan(self, spec, max_chunks: int, arbitrary_size: int | None = None) -> tuple[int, bool, list | None]:
        L = _lib.lib()
        n = C.c_int64()
        if arbitrary_size is not None:
            rc = _lib.check(L.mx_gen_plan_arbitrary(self._h, int(arbitrary_size), int(max_chunks), C.byref(n)))
            mkeys = None
        else:
            d, keep, mkeys = self._mixture_desc(spec)
            rc = _lib.check(L.mx_gen_plan(self._h, C.byref(d), int(max_chunks), C.byref(n)))
            del keep
        report = None
        if rc == _lib.MX_EXHAUSTED and mkeys is not None:
            rem = np.zeros(len(mkeys), np.int64)
            _lib.check(L.mx_gen_report(self._h, _lib.ptr(rem)))
            report = {k: int(v) for k, v in zip(mkeys, rem.tolist()) if v > 0}
        return n.value, rc == _lib.MX_EXHAUSTED, (mkeys, report)

    def _result(self, spec, mkeys, arbitrary_size) -> "ChunkBatch":
        nc, nr = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().mx_gen_result_sizes(self._h, C.byref(nc), C.byref(nr)))
        batch = ChunkBatch(self, nc.value, nr.value, mkeys, spec, arbitrary_size)
        if getattr(self.index, "shard", None) is not None or getattr(self.index, "partition", None) is not None:
            # collective: interleave every rank's pieces
            from .parallel import merge_batch

            batch = merge_batch(self, batch, self.stream)
        return batch

    def plan_batch(self, spec: MixtureSpec | None, max_chunks: int, arbitrary_size: int | None = None) -> "ChunkBatch":
        """Plan + emit up to ``max_chunks`` chunks on the device (bulk API).

        Equivalent to that many ``generate(spec)`` (or ``generate_arbitrary``)
        calls; the CSR result stays on the device (``ChunkBatch``)."""
        self._rewind()
        n, exhausted, (mkeys, report) = self._plan(spec, max_chunks, arbitrary_size)
        self._next_id += n
        batch = self._result(spec, mkeys, arbitrary_size)
        batch.exhausted, batch.report = exhausted, report
        if exhausted:
            self.last_report = report
        return batch

    def _rewind(self) -> None:
        """Bring the device cursors back to the last handed-out chunk."""
        b = self._batch
        self._batch = None
        if b is None or (self._served >= b.n_chunks and not b.exhausted):
            return
        _lib.check(_lib.lib().mx_gen_reset_to_mark(self._h))  # cursors + chunk id at the batch start
        if self._served > 0:
            self._plan(b.spec, self._served, b.arbitrary_size)

    def _serve(self, spec, arbitrary_size):
        b = self._batch
        same = b is not None and b.arbitrary_size == arbitrary_size and (
            arbitrary_size is not None or b.spec == spec)
        if same and self._served < b.n_chunks:
            c = b.chunk(self._served, mixture=spec if arbitrary_size is None else None)
            self._served += 1
            self._next_id += 1
            return c
        if same and b.exhausted:  # the call after the batch's last chunk returns None
            self.last_report = b.report
            self._batch = None  # device state already includes that failed attempt
            return None
        if same:  # fully served, same request: look further ahead
            self._look_ahead = min(self._look_ahead * 2, self.MAX_BATCH)
            self._batch = None
        else:
            self._rewind()
            self._look_ahead = 1
        _lib.check(_lib.lib().mx_gen_mark(self._h))  # device-side snapshot for a later rewind
        n, exhausted, (mkeys, report) = self._plan(spec, self._look_ahead, arbitrary_size)
        batch = self._result(spec, mkeys, arbitrary_size)
        batch.exhausted, batch.report = exhausted, report
        self._batch = batch
        self._served = 0
        return self._serve(spec, arbitrary_size)

    # ---------------------------------------------------------- reference API
    def generate(self, spec: MixtureSpec) -> Chunk | None:
        self.last_report = None
        if spec.strict and spec.chunk_size < len(spec.weights):
            spec.counts()  # raises the reference's MixtureError
        return self._serve(spec, None)

    def generate_arbitrary(self, chunk_size: int) -> Chunk | None:
        if chunk_size <= 0:
            raise MixtureError("chunk_size must be positive")
        self.last_report = None
        return self._serve(None, int(chunk_size))

    def state_dict(self) -> dict:
        self._rewind()
        pos, off = self._cursor_state()
        keys = self.index.component_keys()
        return {
            "next_chunk_id": self._next_id,
            "cursors": {k.canonical_string(): {"pos": int(p), "offset": int(o)}
                        for k, p, o in zip(keys, pos.tolist(), off.tolist())},
        }

    def load_state(self, state: Mapping) -> None:
        self._rewind()
        self._next_id = int(state["next_chunk_id"])
        _lib.check(_lib.lib().mx_gen_set_next_chunk_id(self._h, self._next_id))
        pos, off = self._cursor_state()
        saved = state["cursors"]
        for i, k in enumerate(self.index.component_keys()):
            e = saved.get(k.canonical_string())
            if e is not None:
                pos[i], off[i] = int(e["pos"]), int(e["offset"])
        self._set_cursor_state(pos, off)
