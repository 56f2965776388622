"""Seeded synthetic metadata, identical bytes for the CUDA
path and the CPU oracle.

A corpus is generated as a *run table*: the global sample stream is cut into
runs of Geometric(1/R) length (R=1 -> every run is one sample, the iid
layout) and additionally at every file boundary; each run draws one full
property tuple (independent uniform codes, or one Zipf-distributed joint key).
``expand_numpy`` materialises the int32 code columns on the host;
``bench.py`` expands the same run table on the device.

Vocabularies are registered in a seeded *shuffled* order, so interned codes
differ from the string order the key order is defined on -- this exercises the
code -> rank remapping of ``codec.py`` exactly like a first-seen interning
would.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .catalog import ColumnarCatalog

CFG1_PROPS = {
    "language": ["de", "en", "es", "fr"],
    "source": ["arxiv", "books", "code", "web", "wiki"],
}


def numbered_props(cards, names=None) -> dict[str, list[str]]:
    names = names or [f"p{j}" for j in range(len(cards))]
    return {n: [f"v{i:05d}" for i in range(c)] for n, c in zip(names, cards)}


CFG2_PROPS = numbered_props((4, 5, 5, 4, 5))
CFG5_PROPS = numbered_props((20, 20, 25), ["caption_len", "dataset", "resolution"])


@dataclass
class RunTable:
    n_samples: int
    file_sizes: np.ndarray  # int64[F]
    run_starts: np.ndarray  # int64[R] global sample index
    run_codes: dict[str, np.ndarray]  # prop -> int32[R]
    vocab: dict[str, list[str]]

    def run_lengths(self) -> np.ndarray:
        ends = np.append(self.run_starts[1:], self.n_samples)
        return ends - self.run_starts


def make_runs(
    n_samples: int,
    n_files: int,
    props: dict[str, list[str]],
    mean_run: float,
    seed: int,
    zipf: float | None = None,
    null_frac: float = 0.0,
) -> RunTable:
    rng = np.random.Generator(np.random.PCG64(seed))
    base, extra = divmod(n_samples, n_files)
    sizes = np.full(n_files, base, dtype=np.int64)
    sizes[:extra] += 1
    # run boundaries: geometric lengths over the whole stream, plus file starts
    chunks, covered = [], 0
    while covered < n_samples:
        m = max(1024, int((n_samples - covered) / max(mean_run, 1.0) * 1.1) + 16)
        lens = rng.geometric(1.0 / mean_run, size=m) if mean_run > 1 else np.ones(m, np.int64)
        chunks.append(lens)
        covered += int(lens.sum())
    lens = np.concatenate(chunks)
    starts = np.concatenate(([0], np.cumsum(lens)[:-1]))
    starts = starts[starts < n_samples]
    file_starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    file_starts = file_starts[file_starts < n_samples]
    run_starts = np.union1d(starts, file_starts).astype(np.int64)
    # every geometric run owns a tuple; pieces split at file starts inherit it
    owner = np.searchsorted(starts, run_starts, side="right") - 1
    n_runs = len(starts)
    names = sorted(props)
    codes: dict[str, np.ndarray] = {}
    vocab: dict[str, list[str]] = {}
    perm = {p: rng.permutation(len(props[p])) for p in names}
    for p in names:
        vocab[p] = [props[p][i] for i in perm[p]]  # shuffled registration order
    if zipf is None:
        for p in names:
            draw = rng.integers(0, len(props[p]), size=n_runs)
            codes[p] = np.argsort(perm[p])[draw].astype(np.int32)
    else:
        cards = [len(props[p]) for p in names]
        space = int(np.prod(cards))
        order = rng.permutation(space)  # shuffled key order for the Zipf ranks
        prob = 1.0 / np.arange(1, space + 1, dtype=np.float64) ** zipf
        cdf = np.cumsum(prob / prob.sum())
        ranks = np.minimum(np.searchsorted(cdf, rng.random(n_runs), side="right"), space - 1)
        joint = order[ranks]
        for j, p in enumerate(reversed(names)):
            draw = joint % cards[-1 - j]
            joint = joint // cards[-1 - j]
            codes[p] = np.argsort(perm[p])[draw].astype(np.int32)
    if null_frac > 0:
        for p in names:
            codes[p][rng.random(n_runs) < null_frac] = -1
        allnull = np.all(np.stack([codes[p] for p in names]) < 0, axis=0)
        codes[names[0]][allnull] = 0  # keep every run keyable
    run_codes = {p: codes[p][owner] for p in names}
    return RunTable(n_samples, sizes, run_starts, run_codes, vocab)


def expand_numpy(rt: RunTable) -> ColumnarCatalog:
    lens = rt.run_lengths()
    cols = {p: np.repeat(c, lens).astype(np.int32) for p, c in rt.run_codes.items()}
    return ColumnarCatalog.from_arrays(cols, rt.vocab, rt.file_sizes)


def config(name: str, scale: float = 1.0, layout_r: float | None = None) -> RunTable:
    """Named synthetic workloads of SURVEY.md §8(d); generator seed = config no."""
    if name == "cfg1":
        n, f = int(1_000_000 * scale), max(1, int(1000 * scale))
        return make_runs(n, f, CFG1_PROPS, layout_r or 64, seed=1)
    if name == "cfg2":
        n, f = int(100_000_000 * scale), max(1, int(10_000 * scale))
        return make_runs(n, f, CFG2_PROPS, layout_r or 64, seed=2)
    if name == "cfg3":
        n, f = int(1_000_000_000 * scale), max(1, int(100_000 * scale))
        return make_runs(n, f, CFG2_PROPS, layout_r or 64, seed=3)
    if name == "cfg5":
        n, f = int(100_000_000 * scale), max(1, int(10_000 * scale))
        return make_runs(n, f, CFG5_PROPS, layout_r or 16, seed=5, zipf=1.1)
    raise KeyError(name)


def cfg1_mixtures():
    from .mixtures import MixtureKey as K, MixtureSpec

    disjoint = {K.of({"language": "en"}): 0.5, K.of({"language": ["de", "es", "fr"]}): 0.5}
    overlap = {K.of({"language": "en"}): 0.5, K.of({"source": "web"}): 0.5}
    return {
        "disjoint": MixtureSpec(disjoint, 1024),
        "overlap": MixtureSpec(overlap, 1024),
        "disjoint_strict": MixtureSpec(disjoint, 1024, strict=True),
        "overlap_strict": MixtureSpec(overlap, 1024, strict=True),
    }


def cfg2_mixture(chunk_size: int = 1024):
    from .mixtures import MixtureKey as K, MixtureSpec

    return MixtureSpec(
        {
            K.of({"p0": "v00000"}): 0.4,
            K.of({"p0": "v00001"}): 0.3,
            K.of({"p0": "v00002", "p1": ["v00000", "v00001"]}): 0.2,
            K.of({"p0": "v00003"}): 0.1,
        },
        chunk_size,
    )


def cfg5_mixture(keys, chunk_size: int = 1024):
    """cfg 5's static best-effort mixture: every realized key,
    weights proportional to Zipf(0.8) ranks in a seeded shuffled order, so
    weights differ from the data shares and keys deplete one by one. ``keys``
    are the index's component keys in key order."""
    from .mixtures import MixtureSpec

    rng = np.random.Generator(np.random.PCG64(5))
    w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
    w = w[rng.permutation(len(keys))]
    w = w / w.sum()
    return MixtureSpec({k: float(x) for k, x in zip(keys, w)}, chunk_size)


def write_jsonl_corpus(rt: RunTable, directory, text_len: int = 48) -> list:
    """The run table as JSON-lines files (one per file of the table): every
    record is {"id": i, <prop>: value, ..., "text": "..."} with the run's
    property values, the registration input of SURVEY.md §8f-3 (the
    reference's JsonFieldParser reads the property fields)."""
    from pathlib import Path

    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    props = sorted(rt.run_codes)
    lens = rt.run_lengths()
    ends = np.cumsum(rt.file_sizes)
    filler = "x" * text_len
    paths, buf, f = [], [], 0
    for r in range(len(rt.run_starts)):
        pre = "{" + ", ".join(f'"{p}": "{rt.vocab[p][rt.run_codes[p][r]]}"' for p in props) + ', "id": '
        s = int(rt.run_starts[r])
        for i in range(s, s + int(lens[r])):
            buf.append(f'{pre}{i}, "text": "{filler}"}}')
            if i + 1 == ends[f]:
                path = directory / f"part{f:05d}.jsonl"
                path.write_text("\n".join(buf) + "\n")
                paths.append(path)
                buf, f = [], f + 1
    return paths
