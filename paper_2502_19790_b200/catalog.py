"""Columnar metadata: the stage-1 input of the hot path.

The reference keeps, per registered file, one int32 code column per
single-valued property (-1 = null; codes interned per property in first-seen
order, categorical vocab pre-seeded) plus a ragged tuple column per
multi-valued property (``catalog.py:265-275, 370-415``). File ids are 1-based
in registration order, dataset ids 0-based (``catalog.py:390, 425-429``).

``ColumnarCatalog`` is the same information laid out for HBM: every property
is ONE int32 column over all samples of all files concatenated in ascending
file-id order, files delimited by ``file_offsets``. Multi-valued columns hold
an interned tuple id (equality of tuple ids <=> equality of the held value
sets, which is what the reference's per-file tuple interning compares at
``catalog.py:566-582``). A property absent from a dataset's schema is stored
as null: the reference's filter treats it exactly like null (positive ops
reject, negative ops keep, ``catalog.py:491-504``) and it never enters a key.

Registration / JSON parsing is out of scope; catalogs come
from ``from_reference`` (drop-in: read a live reference ``MetadataCatalog``) or
from ``synth.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .errors import QueryError

_OPS = ("==", "!=", "in", "not-in")


@dataclass(frozen=True)
class FilterPredicate:
    """``(property, op, operand)`` conjunct (``catalog.py:122-157``)."""

    property: str
    op: str
    operand: str | tuple[str, ...]

    def __post_init__(self):
        if self.op not in _OPS:
            raise QueryError(f"unknown filter op {self.op!r}; expected one of {_OPS}")
        single = self.op in ("==", "!=")
        if single and not isinstance(self.operand, str):
            raise QueryError(f"{self.op} takes a single value, got {self.operand!r}")
        if not single and (isinstance(self.operand, str) or not self.operand):
            raise QueryError(f"{self.op} takes a non-empty value list")

    @staticmethod
    def of(item) -> "FilterPredicate":
        if isinstance(item, FilterPredicate):
            return item
        if hasattr(item, "property") and hasattr(item, "op") and hasattr(item, "operand"):
            return FilterPredicate(item.property, item.op, item.operand)  # reference type
        prop, op, operand = item
        if op in ("in", "not-in") and not isinstance(operand, tuple):
            operand = tuple(operand)
        return FilterPredicate(prop, op, operand)

    @property
    def positive(self) -> bool:
        return self.op in ("==", "in")

    def operand_values(self) -> tuple[str, ...]:
        return (self.operand,) if isinstance(self.operand, str) else tuple(self.operand)

    def to_json(self) -> list:
        return [self.property, self.op, list(self.operand_values())]

    @staticmethod
    def from_json(data: Sequence) -> "FilterPredicate":
        prop, op, values = data
        return FilterPredicate(prop, op, values[0] if op in ("==", "!=") else tuple(values))


@dataclass
class ColumnarCatalog:
    """All files' metadata as flat columns (host numpy; see module doc)."""

    columns: dict[str, np.ndarray]  # prop -> int32[N], -1 = null
    vocab: dict[str, list]  # prop -> code -> str (single) | tuple[str, ...] (multi)
    multiple: dict[str, bool]
    file_ids: np.ndarray  # int64[F], ascending, 1-based
    file_ds: np.ndarray  # int32[F]
    file_offsets: np.ndarray  # int64[F+1]
    dataset_names: list[str] = field(default_factory=list)
    file_paths: dict[int, str] = field(default_factory=dict)

    def __post_init__(self):
        if getattr(self, "_meta_only", False):
            return
        self.file_ids = np.asarray(self.file_ids, dtype=np.int64)
        self.file_ds = np.asarray(self.file_ds, dtype=np.int32)
        self.file_offsets = np.asarray(self.file_offsets, dtype=np.int64)
        for p in list(self.columns):
            self.columns[p] = np.ascontiguousarray(self.columns[p], dtype=np.int32)
        n = int(self.file_offsets[-1]) if len(self.file_offsets) else 0
        if len(self.file_offsets) != len(self.file_ids) + 1 or len(self.file_ds) != len(self.file_ids):
            raise ValueError("file table lengths disagree")
        for p, col in self.columns.items():
            if col.shape != (n,):
                raise ValueError(f"column {p!r} has {col.shape[0]} rows, expected {n}")
        if np.any(np.diff(self.file_ids) <= 0):
            raise ValueError("file ids must be strictly ascending")
        if not self.dataset_names:
            nds = int(self.file_ds.max()) + 1 if len(self.file_ds) else 0
            self.dataset_names = [f"ds{i}" for i in range(nds)]

    @property
    def n_samples(self) -> int:
        return int(self.file_offsets[-1]) if len(self.file_offsets) else 0

    @property
    def n_files(self) -> int:
        return len(self.file_ids)

    def properties(self) -> list[str]:
        return sorted(self.columns)

    def validated(self, predicates: Sequence) -> list[FilterPredicate]:
        """``_validated`` (``catalog.py:506-511``): unknown property -> QueryError."""
        preds = [FilterPredicate.of(p) for p in predicates]
        for p in preds:
            if p.property not in self.columns:
                raise QueryError(f"unknown property {p.property!r}")
        return preds

    def code_of(self, prop: str, value: str) -> int | None:
        idx = self._index(prop)
        return idx.get(value)

    def _index(self, prop: str) -> dict:
        cache = self.__dict__.setdefault("_vocab_idx", {})
        if prop not in cache:
            if self.multiple.get(prop):
                cache[prop] = {}
            else:
                cache[prop] = {v: i for i, v in enumerate(self.vocab[prop])}
        return cache[prop]

    def pass_table(self, prop: str, preds: Sequence[FilterPredicate]) -> np.ndarray:
        """bool[card+1]: does code (index code+1; 0 = null) pass every predicate
        on ``prop`` (``_single_mask``/``_multi_mask``, ``catalog.py:459-489``)."""
        card = len(self.vocab[prop])
        ok = np.ones(card + 1, dtype=bool)
        for pred in preds:
            if pred.property != prop:
                continue
            wanted = set(pred.operand_values())
            if self.multiple.get(prop):
                hit = np.array([False] + [bool(wanted & set(t)) for t in self.vocab[prop]])
            else:
                hit = np.zeros(card + 1, dtype=bool)
                for v in wanted:
                    c = self.code_of(prop, v)
                    if c is not None:
                        hit[c + 1] = True
            ok &= hit if pred.positive else ~hit
        return ok

    @staticmethod
    def meta_only(vocab, file_sizes, file_ds=None, file_ids=None, multiple=None) -> "ColumnarCatalog":
        """Catalog metadata without host columns (the columns live only in HBM,
        e.g. expanded on the device by bench.py)."""
        sizes = np.asarray(file_sizes, dtype=np.int64)
        offsets = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        obj = ColumnarCatalog.__new__(ColumnarCatalog)
        obj._meta_only = True
        obj.columns = {p: None for p in vocab}
        obj.vocab = {k: list(v) for k, v in vocab.items()}
        obj.multiple = {p: bool((multiple or {}).get(p, False)) for p in vocab}
        obj.file_ids = np.arange(1, len(sizes) + 1, dtype=np.int64) if file_ids is None else np.asarray(file_ids, np.int64)
        obj.file_ds = np.zeros(len(sizes), np.int32) if file_ds is None else np.asarray(file_ds, np.int32)
        obj.file_offsets = offsets
        obj.dataset_names = [f"ds{i}" for i in range(int(obj.file_ds.max()) + 1 if len(sizes) else 0)]
        obj.file_paths = {}
        return obj

    # ------------------------------------------------------------ adapters
    @staticmethod
    def from_reference(cat) -> "ColumnarCatalog":
        """Read a reference ``MetadataCatalog`` (duck-typed, ``catalog.py:287-296``).

        Single-valued code columns are concatenated as-is; multi-valued ragged
        columns are interned into tuple ids (value tuples sorted, as stored).
        """
        fids = sorted(cat._files)
        props = dict(cat._props)
        sizes = [cat._files[f].n_samples for f in fids]
        offsets = np.zeros(len(fids) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        n = int(offsets[-1])
        columns: dict[str, np.ndarray] = {}
        vocab: dict[str, list] = {}
        multiple: dict[str, bool] = {}
        for name, pdef in props.items():
            col = np.full(n, -1, dtype=np.int32)
            multiple[name] = bool(pdef.multiple)
            if pdef.multiple:
                tuples: dict[tuple, int] = {}
                names = cat._vocab.get(name, [])
                for i, f in enumerate(fids):
                    store = cat._files[f]
                    rag = store.multi.get(name)
                    if rag is None:
                        continue
                    out = col[offsets[i] : offsets[i + 1]]
                    for j, held in enumerate(rag):
                        if held is None:
                            continue
                        t = tuple(sorted(names[c] for c in held))
                        out[j] = tuples.setdefault(t, len(tuples))
                vocab[name] = list(tuples)
            else:
                for i, f in enumerate(fids):
                    arr = cat._files[f].codes.get(name)
                    if arr is not None:
                        col[offsets[i] : offsets[i + 1]] = arr
                vocab[name] = list(cat._vocab.get(name, []))
            columns[name] = col
        return ColumnarCatalog(
            columns=columns,
            vocab=vocab,
            multiple=multiple,
            file_ids=np.array(fids, dtype=np.int64),
            file_ds=np.array([cat._files[f].dataset_id for f in fids], dtype=np.int32),
            file_offsets=offsets,
            dataset_names=list(cat._dataset_names),
            file_paths={f: cat._files[f].path for f in fids},
        )

    @staticmethod
    def from_arrays(
        columns: Mapping[str, np.ndarray],
        vocab: Mapping[str, Sequence],
        file_sizes: Sequence[int],
        file_ds: Sequence[int] | None = None,
        file_ids: Sequence[int] | None = None,
        multiple: Mapping[str, bool] | None = None,
    ) -> "ColumnarCatalog":
        sizes = np.asarray(file_sizes, dtype=np.int64)
        offsets = np.zeros(len(sizes) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offsets[1:])
        f = len(sizes)
        return ColumnarCatalog(
            columns=dict(columns),
            vocab={k: list(v) for k, v in vocab.items()},
            multiple={p: bool((multiple or {}).get(p, False)) for p in columns},
            file_ids=np.arange(1, f + 1) if file_ids is None else np.asarray(file_ids),
            file_ds=np.zeros(f, dtype=np.int32) if file_ds is None else np.asarray(file_ds),
            file_offsets=offsets,
        )


def _tuple_radix(cards: Sequence[int]) -> list[int]:
    """Mixed-radix place values for (code + 1) digits, last property fastest."""
    mult, m = [], 1
    for c in reversed(cards):
        mult.append(m)
        m *= int(c) + 1
    if m >= 1 << 62:
        raise ValueError("row-tuple space exceeds 2^62; keep the per-property column layout")
    return mult[::-1]


def row_tuple_table(radix_values: np.ndarray, cards: Sequence[int]) -> np.ndarray:
    """int32[T, P] property codes of the distinct row tuples (ascending radix)."""
    mult = _tuple_radix(cards)
    u = np.asarray(radix_values, dtype=np.int64)
    return np.stack([(u // m) % (int(c) + 1) - 1 for m, c in zip(mult, cards)], axis=1).astype(np.int32)


def encode_row_tuples(columns: Sequence[np.ndarray], cards: Sequence[int]) -> tuple[np.ndarray, np.ndarray]:
    """Dictionary-encode the rows of per-property code columns (property-name
    order, -1 = null) into ONE int32 row-tuple code column + the tuple table.

    Registration-time layout choice of this implementation (the reference
    interns each property's values into per-file code columns,
    ``catalog.py:370-415``; interning the whole row tuple is the same step one
    level up). Stage 1 then reads 4 bytes per sample instead of 4 per property,
    and per query the codec folds the filter and key packing of every tuple
    into one LUT (``KeyCodec.tuple_luts``)."""
    mult = _tuple_radix(cards)
    n = len(columns[0]) if columns else 0
    r = np.zeros(n, dtype=np.int64)
    for col, m in zip(columns, mult):
        r += (np.asarray(col, dtype=np.int64) + 1) * m
    u, inv = np.unique(r, return_inverse=True)
    if len(u) >= 1 << 31:
        raise ValueError("more than 2^31 distinct row tuples")
    return inv.astype(np.int32).reshape(n), row_tuple_table(u, cards)


def narrow_codes(codes: np.ndarray, n_tuples: int) -> np.ndarray:
    """u16 view of row-tuple codes when the dictionary has <= 65,536 tuples
    (stored as int16 bits, ``column_bytes`` 2 at the C-ABI), else unchanged."""
    if n_tuples > 1 << 16:
        return codes
    return np.asarray(codes).astype(np.uint16).view(np.int16)

