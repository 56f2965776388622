"""Full-size parity digests from the pinned CPU oracle (run in the build
container; the GPU box only reads the committed ``digests.json``):

    python tests/golden/make_digests.py [case ...]

Cases (SURVEY.md §8d workloads, generator seed = config number):

* ``cfg2``       100M samples, 10k files, 5 props, R=64, the cfg 2 mixture,
                 EVERY chunk of the job (the bench workload);
* ``cfg2_iid``   the iid (R=1) variant on a 10M-sample slice (1,000 files),
                 every chunk;
* ``cfg5``       100M samples, Zipf joint keys (10k keys), R=16, the cfg 5
                 best-effort mixture over all keys, first ``CFG5_CHUNKS``;
* ``cfg3``       the 1B-sample, 100k-file catalog on ONE device (north-star
                 job), every chunk of the cfg 2 mixture.

The oracle (``oracle/oracle.py``) is pinned to the reference by
``tests/test_oracle_golden.py``; these digests extend that pin to sizes the
reference itself cannot run in reasonable time. See ``digests.py``.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE))

from digests import ChunkDigest, index_digest  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2502_19790_b200 import synth  # noqa: E402

OUT = HERE / "digests.json"
CFG5_CHUNKS = 2000


def catalog(case):
    if case == "cfg2":
        return synth.config("cfg2")
    if case == "cfg2_iid":
        return synth.make_runs(10_000_000, 1000, synth.CFG2_PROPS, 1, seed=2)
    if case == "cfg5":
        return synth.config("cfg5")
    if case == "cfg3":
        return synth.config("cfg3")
    raise KeyError(case)


def spec_for(case, keys):
    if case == "cfg5":
        from paper_2502_19790_b200.mixtures import MixtureKey

        mk = [MixtureKey.parse(orc.key_string(k)) for k in keys]
        return synth.cfg5_mixture(mk), CFG5_CHUNKS
    return synth.cfg2_mixture(), None


def chunked_intervals(rt, block=100_000_000):
    """``oracle.filter_intervals`` over file blocks of ~``block`` samples
    (intervals never cross files, ``catalog.py:559-604``), concatenated with
    one key table: the 1B-sample catalog does not fit the host as one
    expansion."""
    import numpy as np

    from paper_2502_19790_b200.catalog import ColumnarCatalog

    sizes = rt.file_sizes
    off = np.concatenate(([0], np.cumsum(sizes)))
    ends = np.append(rt.run_starts[1:], rt.n_samples)
    keys, key_of, parts = [], {}, []
    f0 = 0
    while f0 < len(sizes):
        f1 = int(np.searchsorted(off, off[f0] + block, side="right")) - 1
        f1 = max(f1, f0 + 1)
        a, b = int(off[f0]), int(off[f1])
        r0 = int(np.searchsorted(rt.run_starts, a, side="right")) - 1
        r1 = int(np.searchsorted(rt.run_starts, b, side="left"))
        lens = np.minimum(ends[r0:r1], b) - np.maximum(rt.run_starts[r0:r1], a)
        cols = {p: np.repeat(c[r0:r1], lens).astype(np.int32) for p, c in rt.run_codes.items()}
        sub = ColumnarCatalog.from_arrays(cols, rt.vocab, sizes[f0:f1], file_ids=np.arange(f0 + 1, f1 + 1))
        iv = orc.filter_intervals(sub, [])
        remap = np.empty(len(iv["keys"]), dtype=np.int64)
        for j, k in enumerate(iv["keys"]):
            if k not in key_of:
                key_of[k] = len(keys)
                keys.append(k)
            remap[j] = key_of[k]
        iv["key"] = remap[iv["key"]] if len(remap) else iv["key"]
        parts.append(iv)
        print("  block", f0, f1, len(iv["start"]), "intervals", flush=True)
        f0 = f1
    out = {x: np.concatenate([p[x] for p in parts]) for x in ("ds", "fid", "key", "start", "end")}
    out["keys"] = keys
    return out


def run(case):
    t0 = time.time()
    if case == "cfg3":
        idx = orc.OracleIndex(chunked_intervals(catalog(case)))
    else:
        cc = synth.expand_numpy(catalog(case))
        idx = orc.build_index(cc, [])
        del cc
    ks = [orc.key_string(k) for k in idx.keys]
    out = {"samples": int((idx.end - idx.start).sum()), "intervals": int(len(idx.start)), "keys": len(ks),
           "index_sha256": index_digest(ks, idx.rank, idx.ds, idx.fid, idx.start, idx.end)}
    print(case, "index", round(time.time() - t0, 1), "s", out["intervals"], "intervals", flush=True)
    spec, limit = spec_for(case, idx.keys)
    w = {orc.as_key(k): v for k, v in spec.weights.items()}
    gen = orc.OracleGenerator(idx, 42)
    dig = ChunkDigest()
    ranges = 0
    while limit is None or dig.n < limit:
        c = gen.generate(w, spec.chunk_size, spec.strict)
        if c is None:
            out["report"] = {orc.key_string(k): int(v) for k, v in (gen.last_report or {}).items()}
            break
        ranges += sum(len(rs) for ds in c.data.values() for fs in ds.values() for rs in fs.values())
        dig.add(c.serialize())
        if dig.n % 20000 == 0:
            print(case, dig.n, "chunks", round(time.time() - t0, 1), "s", flush=True)
    out.update(chunks=dig.n, ranges=ranges, exhausted=limit is None, chunk_blocks=dig.finish(),
               final_state_sha256=__import__("hashlib").sha256(
                   json.dumps(gen.state_dict(), sort_keys=True).encode()).hexdigest())
    print(case, "done", round(time.time() - t0, 1), "s", out["chunks"], "chunks", flush=True)
    return out


def main(cases):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for case in cases:
        data[case] = run(case)
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg2_iid", "cfg5"])
