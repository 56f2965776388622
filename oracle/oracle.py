"""CPU ORACLE for the Mixtera hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline. The product (``paper_2502_19790_b200``) never imports
it; the CUDA path fails loudly when its extension is missing.

This is an independent restatement, in flat numpy arrays rather than the
reference's nested dicts and per-row Python objects, of:

* stage 1: ``MetadataCatalog.filter_intervals`` (``catalog.py:549-605``, filter
  semantics ``:459-511``) + ``build_index`` (``index.py:88-115``, merge rule
  ``:32-47``) + ``RangeCursor`` layout (``index.py:126-147``);
* stage 2: ``ChunkGenerator`` (``chunks.py:133-272``) with ``apportion``
  (``mixtures.py:158-184``) and ``redistribute_best_effort``
  (``chunks.py:109-130``), replayed at count level over per-component consumed
  offsets, then cut by binary search in cursor prefix
  sums and normalised per (mixture key, dataset, file);
* stage 3: ``per_domain_loss`` (``client.py:582-598``), ``fit_power_law`` /
  ``_loglinear`` (``ado.py:93-168``), ``AdoState`` (``ado.py:179-319``).

Randomness and hashing use exactly the stdlib the reference uses
(``random.Random`` MT19937 shuffles, ``hashlib.blake2b``, ``json``), so seeds,
shuffles and serialized chunk bytes are comparable bit for bit.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (importable
in the build container) on seeded catalogs and commits its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this oracle against
every one of them before any GPU result is compared with it.
"""

from __future__ import annotations

import hashlib
import json
import math
import random
import sys
from bisect import bisect_right

import numpy as np

TOL = 1e-9
_ESC = set("\\;:,")


class OracleError(Exception):
    """Raised where the reference raises (QueryError / MixtureError / ...)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------- keys / seeds


def seed_of(*parts) -> int:
    """``seeding.stable_hash`` (``seeding.py:18-28``)."""
    h = hashlib.blake2b(digest_size=16)
    for part in parts:
        b = part if isinstance(part, bytes) else str(part).encode("utf-8")
        h.update(len(b).to_bytes(8, "big") + b)
    return int.from_bytes(h.digest()[:8], "big") & ((1 << 63) - 1)


def make_key(pairs) -> tuple:
    """Canonical key: ((prop, (sorted unique values...)), ...) sorted by prop."""
    out = []
    for p, vals in sorted(pairs, key=lambda pv: pv[0]):
        if isinstance(vals, str):
            vals = (vals,)
        out.append((str(p), tuple(sorted(set(map(str, vals))))))
    return tuple(out)


def key_order(k) -> tuple:
    """``MixtureKey.sort_key`` (``mixtures.py:111-116``)."""
    return (len(k), tuple(p for p, _ in k), tuple(v for _, v in k))


def key_string(k) -> str:
    esc = lambda s: "".join("\\" + c if c in _ESC else c for c in s)  # noqa: E731
    return ";".join(esc(p) + ":" + ",".join(esc(v) for v in vs) for p, vs in k)


def keys_match(a, b) -> bool:
    da = dict(a)
    return all(set(da[p]) & set(v) for p, v in b if p in da)


def as_key(obj) -> tuple:
    """Accept a product/reference MixtureKey (``.entries``) or a raw tuple."""
    return tuple(getattr(obj, "entries", obj))


# ------------------------------------------------------------------- stage 1


def _pass_table(cat, prop, preds) -> np.ndarray:
    vocab = cat.vocab[prop]
    multi = bool(cat.multiple.get(prop))
    ok = np.ones(len(vocab) + 1, dtype=bool)
    for p_name, op, operand in preds:
        if p_name != prop:
            continue
        want = {operand} if isinstance(operand, str) else set(operand)
        hit = np.zeros(len(vocab) + 1, dtype=bool)
        for c, v in enumerate(vocab):
            hit[c + 1] = bool(want & set(v)) if multi else (v in want)
        ok &= hit if op in ("==", "in") else ~hit
    return ok


def filter_intervals(cat, predicates):
    """Flat interval table in (file, start) order.

    Returns dict of arrays: ``ds``, ``fid``, ``key`` (index into ``keys``),
    ``start``, ``end`` plus the list ``keys``. A run breaks on a sample-id gap
    after filtering, a file change, or any change of the full code signature.
    """
    props = sorted(cat.columns)
    preds = []
    for p in predicates:
        if hasattr(p, "property"):
            p = (p.property, p.op, p.operand)
        if p[0] not in cat.columns:
            raise OracleError("QueryError", f"unknown property {p[0]!r}")
        preds.append(tuple(p))
    n = int(cat.file_offsets[-1]) if len(cat.file_offsets) else 0
    if cat.n_files == 0:
        raise OracleError("QueryError", "catalog is empty")
    mask = np.ones(n, dtype=bool)
    for prop in {p[0] for p in preds}:
        mask &= _pass_table(cat, prop, preds)[cat.columns[prop].astype(np.int64) + 1]
    idx = np.flatnonzero(mask)
    empty = dict(ds=np.zeros(0, np.int64), fid=np.zeros(0, np.int64), key=np.zeros(0, np.int64),
                 start=np.zeros(0, np.int64), end=np.zeros(0, np.int64), keys=[])
    if idx.size == 0:
        return empty
    fidx = np.searchsorted(cat.file_offsets, idx, side="right") - 1
    sig = np.stack([cat.columns[p][idx] for p in props]) if props else np.zeros((0, idx.size))
    brk = np.ones(idx.size, dtype=bool)
    brk[1:] = (np.diff(idx) != 1) | (np.diff(fidx) != 0)
    if props:
        brk[1:] |= np.any(np.diff(sig, axis=1) != 0, axis=0)
    first = np.flatnonzero(brk)
    last = np.append(first[1:], idx.size) - 1
    rows = sig[:, first].T
    uniq, inv = np.unique(rows, axis=0, return_inverse=True)
    keys = []
    for row in uniq:
        pairs = []
        for p, c in zip(props, row):
            if c >= 0:
                v = cat.vocab[p][c]
                pairs.append((p, v if isinstance(v, (tuple, list)) else (v,)))
        if not pairs:
            bad = np.flatnonzero(np.all(rows == row, axis=1))[0]
            g = idx[first[bad]]
            f = int(fidx[first[bad]])
            raise OracleError(
                "QueryError",
                f"sample {int(g - cat.file_offsets[f])} of file {int(cat.file_ids[f])} "
                "has no non-null properties",
            )
        keys.append(make_key(pairs))
    f_of = fidx[first]
    return dict(
        ds=cat.file_ds[f_of].astype(np.int64),
        fid=cat.file_ids[f_of].astype(np.int64),
        key=inv.reshape(-1).astype(np.int64),
        start=(idx[first] - cat.file_offsets[f_of]).astype(np.int64),
        end=(idx[last] + 1 - cat.file_offsets[f_of]).astype(np.int64),
        keys=keys,
    )


class OracleIndex:
    """Key-major interval table: rows sorted by (key order, ds, fid, start),
    adjacent same-(key, file) intervals merged, overlaps rejected
    (``index.py:32-47, 88-115``)."""

    def __init__(self, iv):
        keys = iv["keys"]
        order_of_key = sorted(range(len(keys)), key=lambda i: key_order(keys[i]))
        rank = np.empty(len(keys), dtype=np.int64)
        rank[order_of_key] = np.arange(len(keys))
        self.keys = [keys[i] for i in order_of_key]
        kr = rank[iv["key"]] if len(keys) else np.zeros(0, np.int64)
        o = np.lexsort((iv["start"], iv["fid"], iv["ds"], kr))
        kr, ds, fid, s, e = kr[o], iv["ds"][o], iv["fid"][o], iv["start"][o], iv["end"][o]
        if np.any(e <= s):
            raise OracleError("IndexBuildError", "empty interval")
        same = np.zeros(len(s), dtype=bool)
        same[1:] = (kr[1:] == kr[:-1]) & (ds[1:] == ds[:-1]) & (fid[1:] == fid[:-1])
        if np.any(same[1:] & (s[1:] < e[:-1])):
            raise OracleError("IndexBuildError", "overlapping intervals")
        join = np.zeros(len(s), dtype=bool)
        join[1:] = same[1:] & (s[1:] == e[:-1])
        if join.any():  # never produced by filter_intervals, kept for build_index parity
            head = np.flatnonzero(~join)
            tail = np.append(head[1:], len(s)) - 1
            kr, ds, fid, s, e = kr[head], ds[head], fid[head], s[head], e[tail]
        self.rank, self.ds, self.fid, self.start, self.end = kr, ds, fid, s, e
        self.key_bounds = np.searchsorted(kr, np.arange(len(self.keys) + 1))

    def table(self):
        """[(key_string, ds, fid, start, end)] in index order (the parity form)."""
        ks = [key_string(k) for k in self.keys]
        return [
            (ks[r], int(d), int(f), int(a), int(b))
            for r, d, f, a, b in zip(self.rank, self.ds, self.fid, self.start, self.end)
        ]

    def key_sample_counts(self):
        lens = self.end - self.start
        return {k: int(lens[self.key_bounds[i] : self.key_bounds[i + 1]].sum())
                for i, k in enumerate(self.keys)}

    def cursor_ranges(self, r: int, seed: int):
        """RangeCursor layout of key ``r`` (``index.py:126-147``): shuffle the
        sorted dataset ids, then each dataset's sorted file ids, with ONE
        ``random.Random(derive_seed(seed, "cursor", key string))``."""
        lo, hi = self.key_bounds[r], self.key_bounds[r + 1]
        ds, fid = self.ds[lo:hi], self.fid[lo:hi]
        rng = random.Random(seed_of(seed, "cursor", key_string(self.keys[r])))
        # rows are sorted by (ds, fid, start): group boundaries by run starts
        brk = np.ones(len(fid), dtype=bool)
        brk[1:] = (fid[1:] != fid[:-1]) | (ds[1:] != ds[:-1])
        heads = np.flatnonzero(brk)
        tails = np.append(heads[1:], len(fid))
        by_ds: dict = {}
        for h, t in zip(heads.tolist(), tails.tolist()):
            by_ds.setdefault(int(ds[h]), []).append((int(fid[h]), h, t))
        datasets = sorted(by_ds)
        rng.shuffle(datasets)
        out = []
        s, e = self.start[lo:hi].tolist(), self.end[lo:hi].tolist()
        for d in datasets:
            files = sorted(by_ds[d])
            order = [f for f, _, _ in files]
            rng.shuffle(order)
            span = {f: (h, t) for f, h, t in files}
            for f in order:
                h, t = span[f]
                out.extend((d, f, s[i], e[i]) for i in range(h, t))
        return out


def build_index(cat, predicates) -> OracleIndex:
    return OracleIndex(filter_intervals(cat, predicates))


# ------------------------------------------------------------------- stage 2


def neumaier_sum(xs) -> float:
    """CPython 3.12 builtin ``sum`` over floats (compensated)."""
    s = 0.0
    c = 0.0
    for x in xs:
        x = float(x)
        t = s + x
        if abs(s) >= abs(x):
            c += (s - t) + x
        else:
            c += (x - t) + s
        s = t
    return s + c if c != 0.0 else s


def apportion(weights: dict, total: int) -> dict:
    """Largest remainders over keys in key order (``mixtures.py:158-184``)."""
    if total < 0:
        raise OracleError("MixtureError", "total must be nonnegative")
    ks = sorted(weights, key=key_order)
    wsum = neumaier_sum(weights[k] for k in ks)
    if wsum <= 0:
        raise OracleError("MixtureError", "weights must sum to a positive value")
    base, frac = {}, []
    for i, k in enumerate(ks):
        share = weights[k] / wsum * total
        b = int(share + TOL)
        base[k] = b
        frac.append((-max(0.0, share - b), i))
    left = total - sum(base.values())
    for _, i in sorted(frac)[:left]:
        base[ks[i]] += 1
    return base


def apportion_vec(w: np.ndarray, total: int) -> np.ndarray:
    """``apportion`` over weights already in key order, vectorised: the same
    IEEE operations element by element (``share = w / wsum * total``,
    ``int(share + 1e-9)``, ``max(0, share - base)``) and the same
    (-frac, key order) leftover order; ``wsum`` is CPython's compensated
    ``sum`` (the builtin on 3.12+, ``neumaier_sum`` otherwise)."""
    if total < 0:
        raise OracleError("MixtureError", "total must be nonnegative")
    wl = w.tolist()
    wsum = float(sum(wl)) if sys.version_info >= (3, 12) else neumaier_sum(wl)
    if wsum <= 0:
        raise OracleError("MixtureError", "weights must sum to a positive value")
    share = w / wsum * float(total)
    base = np.trunc(share + TOL)
    frac = np.maximum(share - base, 0.0)
    out = base.astype(np.int64)
    left = int(total - int(out.sum()))
    if left > 0:
        order = np.lexsort((np.arange(len(w)), -frac))
        out[order[:left]] += 1
    return out


class OracleGenerator:
    """``ChunkGenerator`` replayed over per-component consumed offsets."""

    def __init__(self, index: OracleIndex, seed: int):
        self.index = index
        self.seed = seed
        n = len(index.keys)
        order = list(range(n))  # ranks == sorted component keys
        random.Random(seed_of(seed, "component-order")).shuffle(order)
        self.order = order
        self.ranges = [index.cursor_ranges(r, seed) for r in range(n)]
        self.cum = []
        for rg in self.ranges:
            lens = np.array([e - s for _, _, s, e in rg], dtype=np.int64)
            self.cum.append(np.concatenate(([0], np.cumsum(lens))))
        self.total = np.array([c[-1] for c in self.cum], dtype=np.int64)
        self.used = np.zeros(n, dtype=np.int64)
        self.next_chunk_id = 0
        self.last_report = None
        self._match_cache = {}

    # -- cursor primitives
    def _cut(self, r, lo, hi):
        """Ranges of component r's stream offsets [lo, hi)."""
        cum, rg, out = self.cum[r], self.ranges[r], []
        i = bisect_right(cum, lo) - 1
        while lo < hi:
            d, f, s, e = rg[i]
            a = int(s + (lo - cum[i]))
            b = int(min(e, s + (hi - cum[i])))
            out.append((d, f, a, b))
            lo += b - a
            i += 1
        return out

    def _matching(self, m):
        got = self._match_cache.get(m)
        if got is None:
            got = [r for r in self.order if keys_match(m, self.index.keys[r])]
            self._match_cache[m] = got
        return got

    # -- generation
    def _chunk(self, data, weights, chunk_size, strict):
        for files in data.values():
            for d in files:
                for f, rs in files[d].items():
                    rs.sort()
                    merged = []
                    for s, e in rs:
                        if merged and merged[-1][1] == s:
                            merged[-1] = (merged[-1][0], e)
                        else:
                            merged.append((s, e))
                    files[d][f] = merged
        cid = self.next_chunk_id
        self.next_chunk_id += 1
        return OracleChunk(cid, data, seed_of(self.seed, "chunk", cid), weights, chunk_size, strict)

    def generate(self, weights: dict, chunk_size: int, strict: bool = False):
        """``ChunkGenerator.generate`` (``chunks.py:194-230``) with the per-key
        state in arrays indexed by mixture-key order (``sorted_keys``), so
        10k-key mixtures (cfg 5) replay in reasonable time. Same passes, same
        death / redistribution order (``redistribute_best_effort``,
        ``chunks.py:109-130``: the shortfall is apportioned over every
        not-yet-dead key, in key order, by the original weights)."""
        weights = {as_key(k): float(v) for k, v in weights.items()}
        if strict and chunk_size < len(weights):
            raise OracleError("MixtureError", "chunk size below the number of mixture keys")
        mkeys = sorted(weights, key=key_order)
        w = np.array([weights[k] for k in mkeys], dtype=np.float64)
        remaining = apportion_vec(w, chunk_size)
        dead = np.zeros(len(mkeys), dtype=bool)
        data: dict = {}
        self.last_report = None
        while (remaining > 0).any():
            found = {}
            for i in np.flatnonzero(remaining > 0).tolist():
                m = mkeys[i]
                need = int(remaining[i])
                got = 0
                for r in self._matching(m):
                    if need <= 0:
                        break
                    free = self.total[r] - self.used[r]
                    if free <= 0:
                        continue
                    t = int(min(need, free))
                    lo = int(self.used[r])
                    self.used[r] = lo + t
                    for d, f, a, b in self._cut(r, lo, lo + t):
                        data.setdefault(m, {}).setdefault(d, {}).setdefault(f, []).append((a, b))
                    got += t
                    need -= t
                found[i] = got
                remaining[i] -= got
            newly = sorted(i for i, g in found.items() if g == 0 and remaining[i] > 0)
            if not newly:
                continue
            if strict:
                self.last_report = {mkeys[i]: int(remaining[i]) for i in np.flatnonzero(remaining > 0)}
                return None
            for i in newly:
                dead[i] = True
                alive = np.flatnonzero(~dead)
                if len(alive) == 0:
                    self.last_report = {mkeys[j]: int(remaining[j]) for j in np.flatnonzero(remaining > 0)}
                    return None
                short = int(remaining[i])
                if short > 0:
                    remaining[alive] += apportion_vec(w[alive], short)
                remaining[i] = 0
        return self._chunk(data, weights, chunk_size, strict)

    def generate_arbitrary(self, chunk_size: int):
        if chunk_size <= 0:
            raise OracleError("MixtureError", "chunk_size must be positive")
        data: dict = {}
        need = chunk_size
        for r in self.order:
            if need <= 0:
                break
            free = self.total[r] - self.used[r]
            if free <= 0:
                continue
            t = int(min(need, free))
            lo = int(self.used[r])
            self.used[r] = lo + t
            k = self.index.keys[r]
            for d, f, a, b in self._cut(r, lo, lo + t):
                data.setdefault(k, {}).setdefault(d, {}).setdefault(f, []).append((a, b))
            need -= t
        if not data:
            return None
        return self._chunk(data, None, None, None)

    # -- checkpoint form (``chunks.py:257-272``, ``index.py:180-189``)
    def state_dict(self):
        cur = {}
        for r, k in enumerate(self.index.keys):
            ends = self.cum[r][1:]
            pos = int(np.searchsorted(ends, self.used[r], side="right"))
            off = int(self.used[r] - self.cum[r][pos])
            cur[key_string(k)] = {"pos": pos, "offset": off}
        return {"next_chunk_id": self.next_chunk_id, "cursors": cur}

    def load_state(self, state):
        self.next_chunk_id = int(state["next_chunk_id"])
        for r, k in enumerate(self.index.keys):
            e = state["cursors"].get(key_string(k))
            if e is not None:
                self.used[r] = self.cum[r][int(e["pos"])] + int(e["offset"])


class OracleChunk:
    def __init__(self, cid, data, seed, weights, chunk_size, strict):
        self.chunk_id, self.data, self.seed = cid, data, seed
        self.weights, self.chunk_size, self.strict = weights, chunk_size, strict

    def samples_per_key(self):
        return {key_string(k): sum(e - s for fs in ds.values() for rs in fs.values() for s, e in rs)
                for k, ds in self.data.items()}

    def to_json(self):
        mix = None
        if self.weights is not None:
            mix = {
                "weights": {key_string(k): self.weights[k] for k in sorted(self.weights, key=key_order)},
                "chunk_size": self.chunk_size,
                "strict": self.strict,
            }
        return {
            "version": 1,
            "chunk_id": self.chunk_id,
            "seed": self.seed,
            "mixture": mix,
            "data": {
                key_string(k): {
                    str(d): {str(f): [[s, e] for s, e in rs] for f, rs in sorted(fs.items())}
                    for d, fs in sorted(ds.items())
                }
                for k, ds in sorted(self.data.items(), key=lambda kv: key_order(kv[0]))
            },
        }

    def serialize(self) -> bytes:
        return json.dumps(self.to_json(), sort_keys=True, separators=(",", ":"),
                          ensure_ascii=True).encode("ascii")


# ------------------------------------------------------------------- stage 3


def per_domain_loss(losses, tags, n_domains: int):
    """Sequential f64 sums and counts per tag (``client.py:582-598``)."""
    if len(losses) != len(tags):
        raise OracleError("DataReadError", f"{len(losses)} losses for {len(tags)} tags")
    sums = [0.0] * n_domains
    counts = [0] * n_domains
    for x, t in zip(np.asarray(losses, dtype=np.float32).tolist(), np.asarray(tags).tolist()):
        sums[t] += float(x)
        counts[t] += 1
    return np.array(sums), np.array(counts, dtype=np.int64)


def per_domain_loss_np(losses, tags, n_domains: int):
    """Vectorised form of the same reduction (pairwise f64; for large T)."""
    t = np.asarray(tags, dtype=np.int64)
    x = np.asarray(losses, dtype=np.float32).astype(np.float64)
    return np.bincount(t, weights=x, minlength=n_domains), np.bincount(t, minlength=n_domains)


def _loglinear(eps, n, loss):
    resid = loss - eps
    if np.any(resid <= 0):
        return None
    y = np.log(resid)
    x = np.log(n)
    xm, ym = x.mean(), y.mean()
    sxx = float(((x - xm) ** 2).sum())
    if sxx == 0:
        return None
    slope = float(((x - xm) * (y - ym)).sum()) / sxx
    if slope >= 0:
        return None
    alpha = -slope
    beta = math.exp(ym - slope * xm)
    sse = float(((eps + beta * n ** -alpha - loss) ** 2).sum())
    return alpha, beta, sse


def fit_power_law(points):
    """(eps, beta, alpha, fallback) by eps grid + one linear refinement
    (``ado.py:121-168``)."""
    if len(points) < 8:
        raise OracleError("MixtureError", "need at least 8 points to fit a power law")
    n = np.array([p[0] for p in points], dtype=float)
    loss = np.array([p[1] for p in points], dtype=float)
    hi = 0.999 * float(loss.min())
    grid = {0.0}
    if hi > 0:
        grid.update(float(hi * (1.0 - g)) for g in np.geomspace(1e-6, 1.0, 49))
    grid = sorted(grid)
    best = None
    for eps in grid:
        r = _loglinear(eps, n, loss)
        if r is not None and (best is None or r[2] < best[0]):
            best = (r[2], eps, r[0], r[1])
    if best is None:
        e = float(loss.min())
        return (e, max(float(loss[0]) - e, 1e-12), 1e-6, True)
    i = grid.index(best[1])
    lo, hi2 = grid[max(0, i - 1)], grid[min(len(grid) - 1, i + 1)]
    if hi2 > lo:
        for eps in np.linspace(lo, hi2, 201):
            r = _loglinear(float(eps), n, loss)
            if r is not None and r[2] < best[0]:
                best = (r[2], float(eps), r[0], r[1])
    return (best[1], best[3], best[2], False)


class OracleAdo:
    """``AdoState`` + ``AdoSource`` over domain indices 0..K-1 in key order."""

    def __init__(self, prior, fit_start_step=1000, refit_every=1000, subsample_every=10,
                 discard_first=500, p_min=None, smoothing=0.5, credit_rate=0.1,
                 samples_per_step=1):
        self.K = len(prior)
        self.mu = [float(p) for p in prior]
        self.cfg = dict(fit_start_step=fit_start_step, refit_every=refit_every,
                        subsample_every=subsample_every, discard_first=discard_first,
                        smoothing=smoothing, credit_rate=credit_rate,
                        samples_per_step=samples_per_step)
        self.p_min = 0.1 / self.K if p_min is None else p_min
        self.t = 0
        self.cum = 0
        self.cum_at = []
        self.hist = [[] for _ in range(self.K)]
        self.last = [None] * self.K
        self.law = [None] * self.K
        self.credit = list(self.mu)
        self.pi = list(self.mu)
        self.pi_bar = list(self.mu)
        self.pi_bar_count = 1
        self.fit_steps = []

    def observe(self, step, sums, counts):
        means = {k: float(sums[k]) / int(counts[k]) for k in range(self.K) if int(counts[k]) > 0}
        total = int(sum(int(c) for c in counts))
        self.record(step, means, total or None)

    def record(self, step, means, num):
        if step != self.t + 1:
            raise OracleError("FeedbackError", f"expected step {self.t + 1}, got {step}")
        self.t = step
        self.cum += self.cfg["samples_per_step"] if num is None else int(num)
        self.cum_at.append(self.cum)
        for k in range(self.K):
            if k in means:
                self.last[k] = float(means[k])
                self.hist[k].append((step, self.last[k]))
            elif self.last[k] is not None:
                self.hist[k].append((step, self.last[k]))
        d = self.cfg["credit_rate"]
        self.credit = [(1 - d) * c + d * p for c, p in zip(self.credit, self.pi)]
        if step >= self.cfg["fit_start_step"] and step % self.cfg["refit_every"] == 0:
            for k in range(self.K):
                pts = [(self._n(s), v) for s, v in self.hist[k]
                       if s > self.cfg["discard_first"] and s % self.cfg["subsample_every"] == 0]
                if len(pts) >= 8:
                    self.law[k] = fit_power_law(pts)
            self.fit_steps.append(step)

    def _n(self, step):
        tot = self.cum_at[step - 1] if 1 <= step <= len(self.cum_at) else self.cum
        return max(tot / self.K, 1.0)

    def _floor(self, dist):
        out = [float(x) for x in dist]
        fixed = set()
        while True:
            low = [k for k in range(self.K) if k not in fixed and out[k] < self.p_min]
            if not low:
                return out
            fixed.update(low)
            free = [k for k in range(self.K) if k not in fixed]
            if not free:
                return [1.0 / self.K] * self.K
            budget = 1.0 - self.p_min * len(fixed)
            mass = neumaier_sum(out[k] for k in free)
            for k in fixed:
                out[k] = self.p_min
            for k in free:
                out[k] = out[k] / mass * budget if mass > 0 else budget / len(free)

    def compute_pi(self):
        if not self.fit_steps:
            return list(self.mu)
        n = self._n(self.t)
        score = []
        for k in range(self.K):
            law = self.law[k]
            speed = law[2] * law[1] * n ** -(law[2] + 1.0) if law is not None else 0.0
            score.append(self.mu[k] * self.credit[k] * speed)
        total = neumaier_sum(score)
        if total <= 0:
            pi = self._floor(self.mu)
        else:
            s = self.cfg["smoothing"]
            pi = self._floor([(1 - s) * (v / total) + s * b for v, b in zip(score, self.pi_bar)])
        self.pi = pi
        c = self.pi_bar_count
        self.pi_bar = [(b * c + p) / (c + 1) for b, p in zip(self.pi_bar, pi)]
        self.pi_bar_count = c + 1
        return list(pi)
