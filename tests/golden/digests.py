"""Size-independent digests of a full job, shared by the digest generator
(``make_digests.py``, runs the pinned CPU oracle) and the GPU parity tests
(``tests/test_gpu_parity_scale.py``). TEST INFRASTRUCTURE ONLY.

* index digest: sha256 over the interval table in index order, as
  little-endian int64 arrays (key rank, ds, fid, start, end), plus the
  canonical key strings in key order;
* chunk digest: blake2b-128 over the canonical serialized bytes
  (``Chunk.serialize``, ``chunks.py:92-93`` / ``seeding.py:36-42``) of
  ``BLOCK`` consecutive chunks, one hex digest per block, so a mismatch
  localises to one block of chunks.
"""

from __future__ import annotations

import hashlib

import numpy as np

BLOCK = 1024


def index_digest(key_strings, rank, ds, fid, start, end) -> str:
    h = hashlib.sha256()
    h.update("\n".join(key_strings).encode("utf-8"))
    for a in (rank, ds, fid, start, end):
        h.update(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes())
    return h.hexdigest()


class ChunkDigest:
    """Feed serialized chunks in order; ``blocks`` = one hex digest per BLOCK."""

    def __init__(self):
        self.blocks: list[str] = []
        self.n = 0
        self._h = hashlib.blake2b(digest_size=16)

    def add(self, blob: bytes) -> None:
        self._h.update(len(blob).to_bytes(8, "little"))
        self._h.update(blob)
        self.n += 1
        if self.n % BLOCK == 0:
            self.blocks.append(self._h.hexdigest())
            self._h = hashlib.blake2b(digest_size=16)

    def finish(self) -> list[str]:
        if self.n % BLOCK:
            self.blocks.append(self._h.hexdigest())
            self._h = hashlib.blake2b(digest_size=16)
        return self.blocks


def blob_digest(blob: bytes, off) -> list[str]:
    """Digests of a device-serialized batch (one blob + chunk offsets)."""
    d = ChunkDigest()
    off = np.asarray(off, dtype=np.int64)
    mv = memoryview(blob)
    for i in range(len(off) - 1):
        d.add(bytes(mv[int(off[i]):int(off[i + 1])]))
    return d.finish()
