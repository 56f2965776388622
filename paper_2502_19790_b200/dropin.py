"""Install the B200 hot path into a running reference ``mixplane`` (drop-in).

This is the reference-side integration a maintainer adds.
The server's hot-path seams are module-level names (``server.py:23,31``
imports, ``_Job.__init__`` at ``server.py:112-117``):

* ``catalog.filter_intervals(preds)`` -> a ``DeviceRows`` sequence: the
  fused filter + intervals + grouping ran on the GPU
  (``build_index_from_catalog``); it behaves as the reference's
  ``list[IntervalRow]`` (rows are materialised only if someone iterates it)
  and carries the device ``ChunkerIndex``, which ``build_index`` passes
  through;
* ``build_index(rows, workers)`` -> the device build from explicit rows
  (``index.build_index``: sort, empty / overlap checks, merge on the GPU);
* ``ChunkGenerator`` -> the device generator (same methods, same bytes);
* ``AdoSource`` / ``AdoState`` -> device ADO state (pi within 1e-5 rel).

``install`` also re-bases this package's exception classes onto the
reference's (``errors.rebase_onto``), so the server's ``except
MixplaneError`` frames carry the reference's ``kind`` strings. Everything
else (TCP, distribution cache, checkpoints, client) is unchanged.
``install`` returns an ``uninstall`` callable.
"""

from __future__ import annotations

from collections.abc import Sequence

from . import errors
from .ado import AdoSource, AdoState
from .chunks import ChunkGenerator
from .index import ChunkerIndex, build_index, build_index_from_catalog


def _catalog_version(catalog) -> tuple:
    """Changes whenever a dataset is registered (files are only ever added;
    a re-registration with other content raises, ``catalog.py:437-451``)."""
    files = catalog._files
    return (len(files), sum(f.n_samples for f in files.values()))


def _device_catalog(catalog):
    """The catalog's DeviceCatalog, rebuilt when the catalog changed since
    the last job (new datasets registered on a live catalog)."""
    from .index import DeviceCatalog

    if not getattr(catalog, "_files", None):
        raise errors.QueryError("catalog is empty")
    ver = _catalog_version(catalog)
    hit = catalog.__dict__.get("_mx_device")
    if hit is None or hit[0] != ver:
        hit = (ver, DeviceCatalog.from_reference(catalog))
        catalog.__dict__["_mx_device"] = hit
    return hit[1]


class DeviceRows(Sequence):
    """``filter_intervals``' result on the device: a lazy ``list[IntervalRow]``
    (``catalog.py:549-605``) holding the ``ChunkerIndex`` built from it.
    ``len`` / truthiness need no host rows; indexing / iteration / equality
    materialise the reference's ``IntervalRow`` objects once, in the
    reference's order (file id, then start)."""

    def __init__(self, index: ChunkerIndex, row_cls):
        self.index = index
        self._row_cls = row_cls
        self._rows = None

    def _materialise(self) -> list:
        if self._rows is None:
            import numpy as np

            t = self.index.interval_table()
            keys = self.index.component_keys()
            order = np.lexsort((t["start"], t["fid"]))
            self._rows = [
                self._row_cls(int(t["ds"][i]), int(t["fid"][i]), keys[int(t["key"][i])], int(t["start"][i]),
                              int(t["end"][i]))
                for i in order.tolist()
            ]
        return self._rows

    def __len__(self) -> int:
        return int(self.index.n_intervals)

    def __getitem__(self, i):
        return self._materialise()[i]

    def __iter__(self):
        return iter(self._materialise())

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    __hash__ = None

    def __repr__(self) -> str:
        return f"DeviceRows({len(self)} intervals)"


def _filter_intervals(catalog, predicates, row_cls):
    return DeviceRows(build_index_from_catalog(_device_catalog(catalog), predicates), row_cls)


def gpu_catalog(catalog):
    """Make ONE catalog's ``filter_intervals`` run on the GPU (instance
    patch); ``install(..., catalogs=True)`` does it for every catalog."""
    import sys

    row_cls = sys.modules[type(catalog).__module__].IntervalRow
    catalog.filter_intervals = lambda predicates: _filter_intervals(catalog, predicates, row_cls)
    return catalog


def _device_build_index(rows, workers: int = 1):
    if isinstance(rows, DeviceRows):
        return rows.index
    return build_index(rows, workers)


def install(mixplane, catalogs: bool = False) -> callable:
    """Swap the reference's hot-path seams for the device ones. With
    ``catalogs`` every ``MetadataCatalog.filter_intervals`` runs on the GPU
    (class patch) and the library-level names (``mixplane.index.build_index``,
    ``mixplane.chunks.ChunkGenerator``, ...) are swapped too, so code that
    imports them after ``install`` gets the device path."""
    import importlib

    errors.rebase_onto(importlib.import_module(mixplane.__name__ + ".errors"))
    # device chunks are instances of the reference's Chunk too (its __eq__
    # requires isinstance, chunks.py:97-98); our methods come first in the MRO
    from . import chunks as our_chunks

    ref_chunk = importlib.import_module(mixplane.__name__ + ".chunks").Chunk
    chunk_bases = our_chunks.Chunk.__bases__
    if ref_chunk not in our_chunks.Chunk.__mro__:
        our_chunks.Chunk.__bases__ = (ref_chunk,)
    targets = [(mixplane.server, n) for n in ("build_index", "ChunkGenerator", "AdoSource", "AdoState")]
    if catalogs:
        idx_mod = importlib.import_module(mixplane.__name__ + ".index")
        chk_mod = importlib.import_module(mixplane.__name__ + ".chunks")
        ado_mod = importlib.import_module(mixplane.__name__ + ".ado")
        targets += [(idx_mod, "build_index"), (chk_mod, "ChunkGenerator"), (ado_mod, "AdoSource"),
                    (ado_mod, "AdoState")]
        targets += [(mixplane, n) for n in ("build_index", "ChunkGenerator", "AdoSource", "AdoState")
                    if hasattr(mixplane, n)]
    repl = {"build_index": _device_build_index, "ChunkGenerator": ChunkGenerator, "AdoSource": AdoSource,
            "AdoState": AdoState}
    saved = [(mod, n, getattr(mod, n)) for mod, n in targets]
    for mod, n in targets:
        setattr(mod, n, repl[n])
    cat_cls = saved_filter = None
    if catalogs:
        cat_mod = importlib.import_module(mixplane.__name__ + ".catalog")
        cat_cls, row_cls = cat_mod.MetadataCatalog, cat_mod.IntervalRow
        saved_filter = cat_cls.filter_intervals

        def filter_intervals(self, predicates):
            return _filter_intervals(self, predicates, row_cls)

        cat_cls.filter_intervals = filter_intervals

    def uninstall():
        our_chunks.Chunk.__bases__ = chunk_bases
        for mod, n, v in saved:
            setattr(mod, n, v)
        if cat_cls is not None:
            cat_cls.filter_intervals = saved_filter

    return uninstall
