"""Client tokenized mode on the GPU.

``TokenStore.build(paths, text_field, tokenizer)`` tokenizes the text field
of every record of a set of JSON-lines files once, on the device
(``csrc/tokenize.cu``), into one int32 token array in HBM with per-record
offsets; ``tokenized(chunk, store, sequence_length)`` then produces exactly
the ``TokenBatchItem`` stream of the reference's
``ChunkStreamer.tokenized`` (``client.py:451-506``) for one chunk -- the
same tokens in the same order -- as two device tensors: tokens
``int32[n, L]`` and per-token tags ``int32[n, L]`` (the index of the token's
mixture key, stage 3's domain id for ``per_domain_loss``).

Order semantics (restated, control data only): the chunk's keys in
``sorted_keys`` order; each key's ``ActiveIterator`` walks its files in the
order ``Random(derive_seed(chunk.seed, "iter", key)).shuffle`` gives the
(dataset, file) pairs, ranges ascending (``client.py:296-325``); the window
counts are ``apportion`` of the chunk's mixture (live keys, normalised) over
the window (``_window_counts``, ``client.py:401-413``); keys are visited in
``Random(derive_seed(chunk.seed, "tokenized")).shuffle`` order. A key's
stream is cut into L-token sequences across sample boundaries (empty samples
contribute nothing); windows are emitted while every key with a count can
fill its sequences -- W = min over those keys of floor(floor(T_key / L) /
count) -- and the partial window is dropped, as the reference's loop does.
The token data path (gathering every token of every sequence) is one kernel.
"""

from __future__ import annotations

import ctypes as C
import json
from random import Random
from typing import Mapping

import numpy as np

from . import _lib
from .errors import QueryError
from .mixtures import apportion, sorted_keys
from .register import load_jsonl
from .seeding import derive_seed, stable_hash

TOKENIZERS = {"byte": 0, "whitespace": 1}


def host_tokenize(name: str, text, vocab_size: int) -> list[int]:
    """ByteTokenizer / WhitespaceTokenizer (``tokenizers.py:20-40``) for the
    records the device path hands back (same exceptions on bad input)."""
    if name == "byte":
        return list(text.encode("utf-8"))
    return [stable_hash("tok", piece) % vocab_size for piece in text.split()]


class TokenStore:
    """Tokens of every record's text field in HBM (records in file order,
    files in the given order = the catalog's file-id order)."""

    def __init__(self, tokens, offsets, file_base: dict, tokenizer: str, text_field: str):
        self.tokens = tokens          # device int32 [total]
        self.offsets = offsets        # device int64 [n_records + 1]
        self.file_base = file_base    # file id -> first global record index
        self.tokenizer = tokenizer
        self.text_field = text_field

    @staticmethod
    def build(paths, file_ids=None, text_field: str = "text", tokenizer: str = "whitespace",
              vocab_size: int = 32768, device=None) -> "TokenStore":
        import torch

        if tokenizer not in TOKENIZERS:
            raise ValueError(f"unknown tokenizer {tokenizer!r}; available: {sorted(TOKENIZERS)}")
        dev = torch.device(device or "cuda")
        paths = [str(p) for p in paths]
        file_ids = list(file_ids) if file_ids is not None else list(range(1, len(paths) + 1))
        lf = load_jsonl(paths, dev)
        R = lf.n_records
        L = _lib.lib()
        stream = C.c_void_p(_lib.stream_ptr())
        fld = torch.from_numpy(np.frombuffer(text_field.encode("utf-8") or b"\0", np.uint8).copy()).to(dev)
        counts = torch.zeros(R + 1, dtype=torch.int64, device=dev)
        host = torch.zeros(max(R, 1), dtype=torch.uint8, device=dev)
        kind = TOKENIZERS[tokenizer]
        _lib.check(L.mx_jsonl_tokenize(lf.buf.data_ptr(), lf.rs.data_ptr(), lf.re.data_ptr(), R, fld.data_ptr(),
                                       len(text_field.encode("utf-8")), kind, vocab_size, None, counts.data_ptr(),
                                       None, host.data_ptr(), stream))
        # records the device hands back: the reference's payload handling
        # (client.py:466-472) and tokenizer on the host
        back = torch.nonzero(host[:R]).flatten().cpu().numpy().tolist()
        host_tokens = {}
        if back:
            rs, re = lf.rs.cpu().numpy(), lf.re.cpu().numpy()
            for r in back:
                payload = json.loads(bytes(lf.host[int(rs[r]):int(re[r])]))
                text = payload.get(text_field, "") if isinstance(payload, Mapping) else str(payload)
                host_tokens[r] = host_tokenize(tokenizer, text, vocab_size)
            idx = torch.tensor(back, device=dev)
            counts[idx] = torch.tensor([len(host_tokens[r]) for r in back], dtype=torch.int64, device=dev)
        offsets = torch.zeros(R + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts[:R], 0, out=offsets[1:])
        total = int(offsets[R].item()) if R else 0
        tokens = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        _lib.check(L.mx_jsonl_tokenize(lf.buf.data_ptr(), lf.rs.data_ptr(), lf.re.data_ptr(), R, fld.data_ptr(),
                                       len(text_field.encode("utf-8")), kind, vocab_size, offsets.data_ptr(), None,
                                       tokens.data_ptr(), host.data_ptr(), stream))
        if back:
            off_h = offsets.cpu().numpy()
            for r, tk in host_tokens.items():
                if tk:
                    tokens[int(off_h[r]):int(off_h[r]) + len(tk)] = torch.tensor(tk, dtype=torch.int32, device=dev)
        rec_file = np.searchsorted(lf.starts[:-1], lf.rs.cpu().numpy(), side="right") - 1
        per_file = np.bincount(rec_file, minlength=len(paths))
        base = np.concatenate([[0], np.cumsum(per_file)[:-1]])
        store = TokenStore(tokens[:total], offsets, {int(f): int(b) for f, b in zip(file_ids, base)}, tokenizer,
                           text_field)
        store.n_records = R
        store.host_records = len(back)
        return store


def _window_counts(chunk, keys, window_size: int) -> dict:
    """``ChunkStreamer._window_counts`` (``client.py:401-413``)."""
    live = set(keys)
    weights = {k: w for k, w in chunk.mixture.weights.items() if k in live} if chunk.mixture is not None else {}
    if not weights:
        per_key = chunk.samples_per_key()
        weights = {k: float(n) for k, n in per_key.items() if n > 0}
    total = sum(weights.values())
    weights = {k: w / total for k, w in weights.items()}
    return apportion(weights, window_size)


def tokenized(chunk, store: TokenStore, sequence_length: int, window_size: int | None = None, key_tags=None):
    """The chunk's tokenized-mode sequences on the device: (tokens int32[n, L],
    tags int32[n, L], keys) with tags = index into ``keys`` (the chunk's
    mixture keys in sorted_keys order) or ``key_tags[key]`` when given."""
    import torch

    L = int(sequence_length)
    if L < 1:
        raise QueryError("tokenized mode needs sequence_length >= 1")
    if chunk.mixture is not None:
        cs = chunk.mixture.chunk_size
        if window_size is not None and window_size != cs:
            raise QueryError(f"tokenized mode requires window_size == chunk_size ({window_size} != {cs})")
        window_size = cs
    elif window_size is None:
        raise QueryError("tokenized mode on mixture-less chunks needs window_size")
    data = chunk.data
    keys = sorted_keys(data)
    counts = _window_counts(chunk, keys, window_size)
    order = list(keys)
    Random(derive_seed(chunk.seed, "tokenized")).shuffle(order)
    # iterator order of every key's samples (ActiveIterator, client.py:296-325)
    segs, key_off = [], [0]
    for key in keys:
        rng = Random(derive_seed(chunk.seed, "iter", key.canonical_string()))
        work = [(ds, fid) for ds in sorted(data[key]) for fid in sorted(data[key][ds])]
        rng.shuffle(work)
        n = 0
        for ds, fid in work:
            base = store.file_base[fid]
            for s, e in sorted(data[key][ds][fid]):
                segs.append((base + s, base + e))
                n += e - s
        key_off.append(key_off[-1] + n)
    dev = store.tokens.device
    if segs:
        seg = torch.tensor(segs, dtype=torch.int64, device=dev)
        lens = seg[:, 1] - seg[:, 0]
        samples = torch.repeat_interleave(seg[:, 0], lens) + (
            torch.arange(int(lens.sum().item()), device=dev) -
            torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens))
    else:
        samples = torch.zeros(0, dtype=torch.int64, device=dev)
    ntok = store.offsets[samples + 1] - store.offsets[samples]
    koff = torch.tensor(key_off, dtype=torch.int64, device=dev)
    incl = torch.cumsum(ntok, 0)
    key_start = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), incl])[koff[:-1]]
    sprefix = incl - ntok - torch.repeat_interleave(key_start, koff[1:] - koff[:-1])
    key_tokens = (torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), incl])[koff[1:]] - key_start).cpu().numpy()
    cnt = [int(counts.get(k, 0)) for k in keys]
    live = [i for i, c in enumerate(cnt) if c > 0]
    W = min((int(key_tokens[i]) // L) // cnt[i] for i in live) if live else 0
    kidx = {k: i for i, k in enumerate(keys)}
    slot_key = [kidx[k] for k in order]
    slot_first = [0]
    for k in order:
        slot_first.append(slot_first[-1] + int(counts.get(k, 0)))
    S = slot_first[-1]
    tags = [int(key_tags[k]) if key_tags is not None else i for i, k in enumerate(keys)]
    out_t = torch.empty((W * S, L), dtype=torch.int32, device=dev)
    out_g = torch.empty((W * S, L), dtype=torch.int32, device=dev)
    if W * S:
        i32 = lambda x: torch.tensor(x, dtype=torch.int32, device=dev)  # noqa: E731
        sk, sf, kc, kt = i32(slot_key), i32(slot_first), i32(cnt), i32(tags)
        _lib.check(_lib.lib().mx_pack_tokens(W, L, len(order), sk.data_ptr(), sf.data_ptr(), kc.data_ptr(),
                                             koff.data_ptr(), samples.data_ptr(), sprefix.data_ptr(),
                                             store.offsets.data_ptr(), store.tokens.data_ptr(), kt.data_ptr(), S,
                                             out_t.data_ptr(), out_g.data_ptr(), C.c_void_p(_lib.stream_ptr())))
    return out_t, out_g, keys
