"""Order-preserving packed component keys and their device tables.

A component key (the full non-null property map of a run, ``catalog.py:590``)
is packed into one u32 whose NUMERIC order equals ``MixtureKey.sort_key``
(``mixtures.py:111-116``: #properties, then property names, then value
tuples, compared as Python strings/tuples). Fields, most significant first:

    [present count]   only if some property can be null
    [absent bits]     one per nullable property, in name order, 1 = absent
    [rank fields]     one per property, in name order, 1-based rank of the
                      held value tuple among the property's sorted value
                      tuples, 0 = null

Why this is the reference order: keys with more properties sort later; for
equal counts, comparing the sorted property-name tuples of two keys equals
finding the first property (in name order) held by exactly one of them -- the
key that holds it sorts first, i.e. has a 0 absent bit there; for equal
property sets, the value tuples compare field by field in name order. Hence
sorting by the packed integer IS sorting by sort_key, and the dense key rank
falls out of the stage-1 radix sort without any host round trip.

Per sample the packed key is a SUM over properties of per-(property, code)
LUT entries (the present count accumulates, the other fields are disjoint);
bit 31 of an entry marks a code that fails the conjunctive filter
(``catalog.py:459-511``), OR-ed separately by the kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .catalog import ColumnarCatalog, FilterPredicate
from .errors import MixtureError
from .mixtures import MixtureKey, _escape

FAIL = np.uint32(0x80000000)


def _as_tuple(v) -> tuple:
    return tuple(v) if isinstance(v, (tuple, list)) else (v,)


@dataclass
class KeyCodec:
    props: list[str]  # name order
    sorted_values: list[list[tuple]]  # per prop: rank-1 -> value tuple
    code_rank: list[np.ndarray]  # per prop: code -> rank (>= 1)
    nullable: list[bool]
    shift: list[int]
    width: list[int]
    absent_bit: list[int]  # -1 if not nullable
    count_shift: int  # -1 if no nullable property
    key_bits: int
    rank_mask: int
    # derived tables, computed once per codec (a catalog serves many jobs)
    _memo: dict = field(default_factory=dict, repr=False, compare=False)

    _built = None  # class-level cache of build(): signature -> KeyCodec

    @staticmethod
    def build(vocab: dict, nullable: dict) -> "KeyCodec":
        props = sorted(vocab)
        sig = (tuple((p, tuple(_as_tuple(v) for v in vocab[p])) for p in props),
               tuple(bool(nullable.get(p, True)) for p in props))
        if KeyCodec._built is None:
            KeyCodec._built = {}
        hit = KeyCodec._built.get(sig)
        if hit is not None:
            return hit
        codec = KeyCodec._build(vocab, nullable)
        if len(KeyCodec._built) > 64:
            KeyCodec._built.clear()
        KeyCodec._built[sig] = codec
        return codec

    @staticmethod
    def _build(vocab: dict, nullable: dict) -> "KeyCodec":
        props = sorted(vocab)
        sorted_values, code_rank = [], []
        for p in props:
            tuples = [_as_tuple(v) for v in vocab[p]]
            order = sorted(range(len(tuples)), key=lambda i: tuples[i])
            rank = np.zeros(len(tuples), dtype=np.int64)
            for r, i in enumerate(order):
                rank[i] = r + 1
            sorted_values.append([tuples[i] for i in order])
            code_rank.append(rank)
        nullable_l = [bool(nullable.get(p, True)) for p in props]
        widths = [max(1, len(sv).bit_length()) for sv in sorted_values]
        # assign from the least significant end: rank fields (last prop lowest)
        shift = [0] * len(props)
        at = 0
        for j in reversed(range(len(props))):
            shift[j] = at
            at += widths[j]
        absent = [-1] * len(props)
        for j in reversed(range(len(props))):
            if nullable_l[j]:
                absent[j] = at
                at += 1
        count_shift = -1
        if any(nullable_l):
            count_shift = at
            at += max(1, len(props).bit_length())
        if at > 31:
            raise NotImplementedError(f"packed component key needs {at} bits (> 31 supported)")
        rank_mask = 0
        for j in range(len(props)):
            rank_mask |= ((1 << widths[j]) - 1) << shift[j]
        return KeyCodec(props, sorted_values, code_rank, nullable_l, shift, widths, absent,
                        count_shift, at, rank_mask)

    # ---------------------------------------------------------------- LUTs
    def luts(self, cat: ColumnarCatalog, preds: list[FilterPredicate]) -> tuple[np.ndarray, np.ndarray]:
        """Concatenated per-property LUT (entry code+1) and its offsets."""
        key = ("luts", tuple(preds), tuple(sorted(cat.multiple.items())))
        hit = self._memo.get(key)
        if hit is None:
            hit = self._luts(cat, preds)
            self._memo[key] = hit
        return hit

    def _luts(self, cat: ColumnarCatalog, preds: list[FilterPredicate]) -> tuple[np.ndarray, np.ndarray]:
        parts, offs = [], [0]
        for j, p in enumerate(self.props):
            ok = cat.pass_table(p, preds)
            card = len(self.code_rank[j])
            e = np.zeros(card + 1, dtype=np.uint64)
            e[1:] = self.code_rank[j].astype(np.uint64) << np.uint64(self.shift[j])
            if self.count_shift >= 0:
                e[1:] += np.uint64(1 << self.count_shift)
            if self.absent_bit[j] >= 0:
                e[0] = np.uint64(1 << self.absent_bit[j])
            e = e.astype(np.uint32)
            e[~ok] |= FAIL
            parts.append(e)
            offs.append(offs[-1] + card + 1)
        return np.concatenate(parts).astype(np.uint32), np.array(offs, dtype=np.int32)

    def tuple_luts(self, cat: ColumnarCatalog, preds: list[FilterPredicate],
                   table: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """LUT over row-tuple codes (``encode_row_tuples``): entry (t+1) is the
        sum of row tuple t's per-property entries (its whole packed key) with
        FAIL set when any of its property codes fails the filter -- exactly
        what the per-property scan computes for a row holding those codes."""
        lut, off = self.luts(cat, preds)
        t = np.asarray(table, dtype=np.int64)
        key = np.zeros(len(t), dtype=np.uint64)
        fail = np.zeros(len(t), dtype=bool)
        for j in range(len(self.props)):
            e = lut[off[j] + t[:, j] + 1]
            key += (e & ~FAIL).astype(np.uint64)
            fail |= (e & FAIL) != 0
        out = np.empty(len(t) + 1, dtype=np.uint32)
        out[0] = FAIL  # no row holds code -1
        out[1:] = key.astype(np.uint32) | np.where(fail, FAIL, np.uint32(0)).astype(np.uint32)
        return out, np.array([0, len(out)], dtype=np.int32)

    # ---------------------------------------------------------------- keys
    def rank_of(self, packed: int, j: int) -> int:
        return (int(packed) >> self.shift[j]) & ((1 << self.width[j]) - 1)

    def decode(self, packed: int) -> MixtureKey:
        entries = []
        for j, p in enumerate(self.props):
            r = self.rank_of(packed, j)
            if r:
                entries.append((p, self.sorted_values[j][r - 1]))
        return MixtureKey(tuple(entries))

    def key_strings(self) -> tuple[bytes, np.ndarray, np.ndarray]:
        """Canonical-string pieces "esc(prop):esc(v1),esc(v2)" per (prop, rank)."""
        hit = self._memo.get("key_strings")
        if hit is None:
            hit = self._key_strings()
            self._memo["key_strings"] = hit
        return hit

    def _key_strings(self) -> tuple[bytes, np.ndarray, np.ndarray]:
        blobs, offs, base = [], [0], []
        for j, p in enumerate(self.props):
            base.append(len(blobs))
            for vals in self.sorted_values[j]:
                b = (_escape(p) + ":" + ",".join(_escape(v) for v in vals)).encode("utf-8")
                blobs.append(b)
                offs.append(offs[-1] + len(b))
        return b"".join(blobs), np.array(offs, dtype=np.int64), np.array(base, dtype=np.int32)

    # ---------------------------------------------------------- mixtures
    def allow_table(self, mkeys: list[MixtureKey]) -> tuple[np.ndarray, np.ndarray, int]:
        """Per mixture key, per property, bit r = a component holding value
        rank r there matches on that property (rank 0 = null -> property not
        shared -> vacuously true; ``mixtures.py:100-109``)."""
        key = ("allow", tuple(k.entries for k in mkeys))
        hit = self._memo.get(key)
        if hit is None:
            hit = self._allow_table(mkeys)
            if len(self._memo) > 256:
                self._memo.clear()
            self._memo[key] = hit
        return hit

    def _allow_table(self, mkeys: list[MixtureKey]) -> tuple[np.ndarray, np.ndarray, int]:
        base, at = [], 0
        for j in range(len(self.props)):
            base.append(at)
            at += len(self.sorted_values[j]) + 1
        words = (at + 31) // 32
        table = np.zeros((len(mkeys), words), dtype=np.uint32)
        bits = np.zeros((len(mkeys), words * 32), dtype=bool)
        for m, key in enumerate(mkeys):
            held = dict(key.entries)
            for j, p in enumerate(self.props):
                lo = base[j]
                n = len(self.sorted_values[j])
                if p not in held:
                    bits[m, lo : lo + n + 1] = True
                    continue
                want = set(held[p])
                bits[m, lo] = True
                for r, vals in enumerate(self.sorted_values[j], start=1):
                    bits[m, lo + r] = not want.isdisjoint(vals)
        for m in range(len(mkeys)):
            packed = np.packbits(bits[m].reshape(-1, 32)[:, ::-1], axis=1).view(">u4").reshape(-1)
            table[m] = packed.astype(np.uint32)
        return table, np.array(base, dtype=np.int32), words


def mixture_arrays(codec: KeyCodec, weights: dict) -> tuple[list[MixtureKey], np.ndarray]:
    keys = sorted(weights, key=MixtureKey.sort_key)
    w = np.array([float(weights[k]) for k in keys], dtype=np.float64)
    if len(keys) == 0:
        raise MixtureError("mixture has no keys")
    return keys, w
