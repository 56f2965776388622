"""Seeds and canonical JSON, bit-compatible with the reference.

``stable_hash`` follows ``seeding.py:18-28``: BLAKE2b with a 16-byte digest
over length-prefixed parts (8-byte big-endian length, then the UTF-8 bytes of
``str(part)``), first 8 digest bytes read big-endian and masked to 63 bits.
The CUDA path recomputes the same function on device for per-key cursor seeds
and per-chunk seeds (``csrc/blake2b.cuh``); this host copy seeds the job and
checks the device one.
"""

from __future__ import annotations

import hashlib
import json
from typing import Any

SEED_MASK = (1 << 63) - 1


def _encode(part: object) -> bytes:
    return part if isinstance(part, bytes) else str(part).encode("utf-8")


def hash_message(*parts: object) -> bytes:
    """The exact byte string BLAKE2b consumes for ``parts``."""
    out = bytearray()
    for part in parts:
        data = _encode(part)
        out += len(data).to_bytes(8, "big")
        out += data
    return bytes(out)


def stable_hash(*parts: object) -> int:
    digest = hashlib.blake2b(hash_message(*parts), digest_size=16).digest()
    return int.from_bytes(digest[:8], "big") & SEED_MASK


def derive_seed(base_seed: int, *context: object) -> int:
    return stable_hash(base_seed, *context)


def canonical_json(obj: Any) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=True)


def canonical_json_bytes(obj: Any) -> bytes:
    return canonical_json(obj).encode("ascii")


def content_id(data: bytes, length: int = 16) -> str:
    return hashlib.blake2b(data, digest_size=length).hexdigest()[: 2 * length]
