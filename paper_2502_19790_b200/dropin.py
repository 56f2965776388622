"""Install the B200 hot path into a running reference ``mixplane`` (drop-in).

This is the reference-side integration a maintainer adds:
the server's three hot-path seams are module-level names
(``server.py:23,31`` imports, ``_Job.__init__`` at ``server.py:112-117``):

* ``catalog.filter_intervals(preds)`` -> returns a device ``ChunkerIndex``
  built by ``build_index_from_catalog`` (filter + intervals + grouping on the
  GPU; no Python ``IntervalRow`` objects), which ``build_index`` passes through;
* ``ChunkGenerator`` -> the device generator (same methods, same bytes);
* ``AdoSource`` / ``AdoState`` -> device ADO state (pi within 1e-5 rel).

Everything else (TCP, distribution cache, checkpoints, client) is unchanged.
``install`` returns an ``uninstall`` callable.
"""

from __future__ import annotations

from .ado import AdoSource, AdoState
from .chunks import ChunkGenerator
from .index import ChunkerIndex, build_index_from_catalog


def gpu_catalog(catalog):
    """Make ``catalog.filter_intervals`` return a device ChunkerIndex (the
    reference's columnar store is uploaded once and cached)."""
    state = {}

    def filter_intervals(predicates):
        from .index import DeviceCatalog

        if "dev" not in state:
            if not getattr(catalog, "_files", None):
                from .errors import QueryError

                raise QueryError("catalog is empty")
            state["dev"] = DeviceCatalog.from_reference(catalog)
        return build_index_from_catalog(state["dev"], predicates)

    catalog.filter_intervals = filter_intervals
    return catalog


def install(mixplane) -> callable:
    server = mixplane.server
    saved = {n: getattr(server, n) for n in ("build_index", "ChunkGenerator", "AdoSource", "AdoState")}
    ref_build = saved["build_index"]

    def build_index(rows, workers: int = 1):
        return rows if isinstance(rows, ChunkerIndex) else ref_build(rows, workers)

    server.build_index = build_index
    server.ChunkGenerator = ChunkGenerator
    server.AdoSource = AdoSource
    server.AdoState = AdoState

    def uninstall():
        for n, v in saved.items():
            setattr(server, n, v)

    return uninstall
