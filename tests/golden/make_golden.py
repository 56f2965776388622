"""Generate golden vectors by running the REAL reference (mixplane, pure
Python) on seeded synthetic catalogs. Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (read-only), injects
the same int32 code columns the CUDA path consumes into a reference
``MetadataCatalog`` (its columnar layout, ``catalog.py:265-296``), and records:

* the ChunkerIndex interval table (``build_index(filter_intervals(...))._index``),
* every key's RangeCursor order and the component order (job seed 42),
* chunk sequences under static / strict / overlapping / inferred / arbitrary
  mixtures (serialized bytes), shortfall reports, generator states,
* ``per_domain_loss`` sums, ``fit_power_law`` laws and ADO pi trajectories.

Inputs are stored next to the outputs (``<case>.npz``) so the GPU box never
needs the reference. Output: ``tests/golden/<case>.json.gz`` + ``.npz``.
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mixplane import catalog as rcat  # noqa: E402
from mixplane.ado import AdoConfig, AdoSource, AdoState, fit_power_law  # noqa: E402
from mixplane.chunks import ChunkGenerator  # noqa: E402
from mixplane.client import per_domain_loss  # noqa: E402
from mixplane.index import build_index  # noqa: E402
from mixplane.mixtures import MixtureKey, MixtureSpec, infer_mixture  # noqa: E402

from paper_2502_19790_b200 import synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402

JOB_SEED = 42


def inject(cc: ColumnarCatalog, schemas: dict[int, list[str]] | None = None):
    """Build a reference MetadataCatalog holding exactly ``cc``'s columns."""
    cat = rcat.MetadataCatalog()
    props = sorted(cc.columns)
    nds = int(cc.file_ds.max()) + 1
    schemas = schemas or {d: props for d in range(nds)}
    vocab, vidx = {}, {}
    for p in props:
        if cc.multiple.get(p):
            vals = sorted({v for t in cc.vocab[p] for v in t})
            vocab[p] = vals
        else:
            vocab[p] = list(cc.vocab[p])
        vidx[p] = {v: i for i, v in enumerate(vocab[p])}
    cat._props = {p: rcat.PropertyDef(p, "string", True, bool(cc.multiple.get(p))) for p in props}
    cat._vocab, cat._vocab_idx = vocab, vidx
    cat._dataset_names = [f"ds{d}" for d in range(nds)]
    cat._dataset_schemas = {d: rcat.PropertySchema([cat._props[p] for p in schemas[d]]) for d in range(nds)}
    cat._dataset_files = {d: [] for d in range(nds)}
    for i, fid in enumerate(cc.file_ids.tolist()):
        ds = int(cc.file_ds[i])
        a, b = int(cc.file_offsets[i]), int(cc.file_offsets[i + 1])
        store = rcat._FileStore(path=f"/synthetic/{fid}.jsonl", dataset_id=ds, n_samples=b - a,
                                content_hash="0" * 32)
        for p in schemas[ds]:
            col = cc.columns[p][a:b]
            if cc.multiple.get(p):
                store.multi[p] = [None if c < 0 else tuple(vidx[p][v] for v in cc.vocab[p][c]) for c in col]
            else:
                store.codes[p] = col.astype(np.int32).copy()
        cat._files[fid] = store
        cat._dataset_files[ds].append(fid)
    return cat


def index_table(index):
    out = []
    for k in index.component_keys():
        for ds in sorted(index.entries(k)):
            for fid in sorted(index.entries(k)[ds]):
                for s, e in index.entries(k)[ds][fid]:
                    out.append([k.canonical_string(), ds, fid, s, e])
    return out


def run_chunks(index, spec_fn, limit, arbitrary=None):
    gen = ChunkGenerator(index, JOB_SEED)
    chunks, states = [], {}
    exhausted = False
    for i in range(limit):
        if i in (1, 3):
            states[str(i)] = gen.state_dict()
        c = gen.generate_arbitrary(arbitrary) if arbitrary else gen.generate(spec_fn())
        if c is None:
            exhausted = True
            break
        chunks.append(c.serialize().decode("ascii"))
    report = None
    if gen.last_report is not None:
        report = {k.canonical_string(): v for k, v in gen.last_report.items()}
    return {"chunks": chunks, "report": report, "states": states, "final_state": gen.state_dict(),
            "exhausted": exhausted}


def spec_json(spec: MixtureSpec):
    return spec.to_json()


def save(name, cc: ColumnarCatalog, payload: dict):
    np.savez_compressed(
        HERE / f"{name}.npz",
        file_ids=cc.file_ids, file_ds=cc.file_ds, file_offsets=cc.file_offsets,
        **{f"col_{p}": c for p, c in cc.columns.items()},
    )
    payload["vocab"] = {p: [list(v) if isinstance(v, tuple) else v for v in cc.vocab[p]] for p in cc.vocab}
    payload["multiple"] = {p: bool(v) for p, v in cc.multiple.items()}
    with gzip.open(HERE / f"{name}.json.gz", "wt") as f:
        json.dump(payload, f)
    print(f"{name}: {len(payload.get('index', []))} intervals, "
          f"{sum(len(v['chunks']) for v in payload.get('runs', {}).values())} chunks")


def stage12_case(name, cc, predicates, mixtures, limit=400, schemas=None, arbitrary=(), infer=()):
    cat = inject(cc, schemas)
    rows = cat.filter_intervals(predicates)
    index = build_index(rows)
    gen = ChunkGenerator(index, JOB_SEED)
    payload = {
        "predicates": [list(p[:2]) + [p[2] if isinstance(p[2], str) else list(p[2])] for p in predicates],
        "job_seed": JOB_SEED,
        "index": index_table(index),
        "component_order": [k.canonical_string() for k in gen._component_order],
        "cursors": {k.canonical_string(): [list(r) for r in gen._cursors[k]._ranges]
                    for k in index.component_keys()},
        "mixtures": {},
        "runs": {},
    }
    for mname, spec in mixtures.items():
        payload["mixtures"][mname] = spec_json(spec)
        payload["runs"][mname] = run_chunks(index, lambda s=spec: s, limit)
    for size in arbitrary:
        payload["runs"][f"arbitrary{size}"] = run_chunks(index, None, limit, arbitrary=size)
    for size in infer:
        spec = infer_mixture(index, size)
        payload["mixtures"][f"infer{size}"] = spec_json(spec)
        payload["runs"][f"infer{size}"] = run_chunks(index, lambda s=spec: s, limit)
    save(name, cc, payload)


def K(d):
    return MixtureKey.of(d)


def main():
    # A/B: cfg1 shape at reduced size, iid and clustered
    for r, n, f in ((1, 20_000, 20), (64, 60_000, 60)):
        cc = synth.expand_numpy(synth.make_runs(n, f, synth.CFG1_PROPS, r, seed=1))
        dis = {K({"language": "en"}): 0.5, K({"language": ["de", "es", "fr"]}): 0.5}
        ovl = {K({"language": "en"}): 0.5, K({"source": "web"}): 0.5}
        stage12_case(
            f"cfg1_r{r}", cc, [],
            {"disjoint": MixtureSpec(dis, 1024), "overlap": MixtureSpec(ovl, 1024),
             "disjoint_strict": MixtureSpec(dis, 1024, True), "overlap_strict": MixtureSpec(ovl, 1024, True),
             "three_way": MixtureSpec({K({"language": "en"}): 0.25, K({"source": ["code", "web"]}): 0.5,
                                       K({"language": "fr", "source": "wiki"}): 0.25}, 333)},
            arbitrary=(1000,), infer=(256,),
        )
    # C: cfg2 shape, small
    cc = synth.expand_numpy(synth.make_runs(200_000, 20, synth.CFG2_PROPS, 64, seed=2))
    stage12_case("cfg2_small", cc, [], {"cfg2": synth_cfg2()}, limit=400)
    # D: nulls, two datasets, a property absent from one schema, filters
    rt = synth.make_runs(30_000, 24, synth.numbered_props((3, 4, 3)), 3, seed=7, null_frac=0.15)
    cc = synth.expand_numpy(rt)
    cc.file_ds[12:] = 1
    cc.columns["p2"][cc.file_offsets[12]:] = -1  # dataset 1 has no p2 in its schema
    stage12_case(
        "filters_nulls", cc,
        [("p0", "in", ("v00000", "v00002", "nope")), ("p1", "!=", "v00003")],
        {"sub": MixtureSpec({K({"p0": "v00000"}): 0.6, K({"p2": "v00001"}): 0.4}, 200)},
        schemas={0: ["p0", "p1", "p2"], 1: ["p0", "p1"]}, arbitrary=(500,), infer=(128,),
    )
    # E: multi-valued property registered through the reference's own parser
    stage12_case_multi()
    # F: depletion / redistribution (acceptance 04 shape) and a 3-key strict stop
    cols = np.repeat(np.array([0, 1, 2], np.int32), [500, 40, 500])
    cc = ColumnarCatalog.from_arrays({"domain": cols}, {"domain": ["a", "b", "c"]}, [500, 40, 500])
    stage12_case(
        "depletion", cc, [],
        {"best_effort": MixtureSpec({K({"domain": "a"}): 0.5, K({"domain": "b"}): 0.2, K({"domain": "c"}): 0.3}, 100),
         "strict": MixtureSpec({K({"domain": "a"}): 0.5, K({"domain": "b"}): 0.2, K({"domain": "c"}): 0.3}, 100, True)},
    )
    # G: cfg5 shape (Zipf joint key, many keys, heavy redistribution), small
    rt = synth.make_runs(60_000, 12, synth.numbered_props((5, 5, 6), ["caption_len", "dataset", "resolution"]),
                         16, seed=5, zipf=1.1)
    cc = synth.expand_numpy(rt)
    cat = inject(cc)
    keys = build_index(cat.filter_intervals([])).component_keys()
    rng = np.random.Generator(np.random.PCG64(55))
    w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
    w = w[rng.permutation(len(keys))]
    w = w / w.sum()
    weights = {k: float(x) for k, x in zip(keys, w)}
    weights = normalize_weights(weights)
    stage12_case("cfg5_small", cc, [], {"zipf": MixtureSpec(weights, 1024)}, limit=80)
    # H: more mixture keys than the serial planner keeps on chip (> 256), Zipf
    # weights, uniform weights (exact share ties) and a Zipf subset
    rt = synth.make_runs(150_000, 16, synth.numbered_props((8, 9, 10), ["caption_len", "dataset", "resolution"]),
                         16, seed=8, zipf=1.05)
    cc = synth.expand_numpy(rt)
    keys = build_index(inject(cc).filter_intervals([])).component_keys()
    rng = np.random.Generator(np.random.PCG64(56))
    w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
    w = w[rng.permutation(len(keys))]
    zipf = normalize_weights({k: float(x) for k, x in zip(keys, w)})
    uniform = normalize_weights({k: 1.0 for k in keys})
    sub = normalize_weights({k: float(x) for k, x in list(zip(keys, w))[: 300]})
    stage12_case("cfg5_wide", cc, [], {"zipf": MixtureSpec(zipf, 1024), "uniform": MixtureSpec(uniform, 4096),
                                       "subset": MixtureSpec(sub, 700)}, limit=80)
    stage3()


def normalize_weights(weights):
    s = sum(weights.values())
    out = {k: v / s for k, v in weights.items()}
    if abs(sum(out.values()) - 1.0) > 1e-9:
        raise RuntimeError("weights do not normalize")
    return out


def synth_cfg2():
    return MixtureSpec(
        {K({"p0": "v00000"}): 0.4, K({"p0": "v00001"}): 0.3,
         K({"p0": "v00002", "p1": ["v00000", "v00001"]}): 0.2, K({"p0": "v00003"}): 0.1}, 1024)


def stage12_case_multi():
    from mixplane.formats import write_jsonl

    rng = np.random.Generator(np.random.PCG64(11))
    tags = ["ml", "nlp", "cv", "rl"]
    langs = ["python", "go", "rust"]
    with tempfile.TemporaryDirectory() as tmp:
        files = []
        for i in range(6):
            recs = []
            n = int(rng.integers(50, 120))
            cur = None
            for j in range(n):
                if cur is None or rng.random() < 0.2:
                    k = int(rng.integers(0, 3))
                    t = sorted(set(rng.choice(tags, size=k).tolist())) if k else None
                    cur = (t, str(rng.choice(langs)))
                rec = {"text": "x", "language": cur[1]}
                if cur[0] is not None:
                    rec["tags"] = cur[0]
                recs.append(rec)
            path = Path(tmp) / f"f{i}.jsonl"
            write_jsonl(path, recs)
            files.append(path)
        cat = rcat.MetadataCatalog()
        schema = rcat.PropertySchema([rcat.PropertyDef("language"), rcat.PropertyDef("tags", multiple=True)])
        cat.register_dataset("tagged", files, rcat.JsonFieldParser.for_properties(["language", "tags"]), schema)
        cc = ColumnarCatalog.from_reference(cat)
        preds = [("tags", "in", ("ml", "cv")), ("language", "not-in", ("go",))]
        rows = cat.filter_intervals(preds)
        index = build_index(rows)
        gen = ChunkGenerator(index, JOB_SEED)
        spec = MixtureSpec({K({"tags": "ml"}): 0.5, K({"language": "python"}): 0.5}, 20)
        payload = {
            "predicates": [list(p[:2]) + [list(p[2])] for p in preds],
            "job_seed": JOB_SEED,
            "index": index_table(index),
            "component_order": [k.canonical_string() for k in gen._component_order],
            "cursors": {k.canonical_string(): [list(r) for r in gen._cursors[k]._ranges]
                        for k in index.component_keys()},
            "mixtures": {"tagmix": spec_json(spec)},
            "runs": {"tagmix": run_chunks(index, lambda: spec, 200)},
        }
        save("multi_tags", cc, payload)


def stage3():
    out = {}
    rng = np.random.Generator(np.random.PCG64(4))
    # per_domain_loss: sequential f64 sums of f32 token losses
    K_dom = 7
    losses = rng.gamma(50.0, 1 / 50.0, size=20_000).astype(np.float32) * 2.5
    tags = rng.integers(0, K_dom, size=20_000).astype(np.int32)
    keys = [K({"domain": f"d{i}"}) for i in range(K_dom)]
    got = per_domain_loss(losses.tolist(), [keys[t] for t in tags.tolist()])
    out["per_domain_loss"] = {
        "losses": losses.tolist(), "tags": tags.tolist(),
        "sums": [got[keys[i]][0] for i in range(K_dom)], "counts": [got[keys[i]][1] for i in range(K_dom)],
    }
    # fit_power_law known answers
    fits = []
    for eps, beta, alpha, noise in ((2.0, 10.0, 0.35, 0.0), (1.5, 3.0, 0.2, 0.0), (0.8, 20.0, 0.6, 0.0),
                                    (2.0, 10.0, 0.35, 0.01), (1.2, 5.0, 0.5, 0.003)):
        ns = np.arange(510, 5001, 10, dtype=float)
        ys = eps + beta * ns ** -alpha + (rng.normal(0, noise, ns.size) if noise else 0.0)
        pts = [(float(a), float(b)) for a, b in zip(ns, ys)]
        law = fit_power_law(pts)
        fits.append({"points": pts, "law": [law.epsilon, law.beta, law.alpha, law.fallback]})
    pts = [(float(n), 1.0 + 0.001 * n) for n in range(100, 1000, 50)]
    law = fit_power_law(pts)
    fits.append({"points": pts, "law": [law.epsilon, law.beta, law.alpha, law.fallback]})
    out["fits"] = fits
    # ADO trajectory: 6 domains, hidden laws, Gamma noise, 2 refits
    D = 6
    dom = [K({"domain": f"x{i}"}) for i in range(D)]
    prior = rng.dirichlet(np.ones(D))
    prior = prior / prior.sum()
    prior_map = {k: float(p) for k, p in zip(dom, prior)}
    drift = 1.0 - sum(prior_map.values())
    prior_map[dom[0]] += drift
    hid = [(float(rng.uniform(1.5, 2.5)), float(rng.uniform(2, 10)), float(rng.uniform(0.2, 0.5))) for _ in range(D)]
    cfg = AdoConfig()
    src = AdoSource(AdoState(cfg, prior_map), chunk_size=1024)
    tokens_per_step = 4096
    cum = np.zeros(D)
    steps = []
    for step in range(1, 2101):
        spec = src.current_spec()
        pi = np.array([spec.weights.get(k, 0.0) for k in dom])
        seqs = rng.choice(D, size=tokens_per_step // 64, p=pi / pi.sum())
        counts = np.bincount(seqs, minlength=D) * 64
        cum += counts
        feedback = {}
        for i in range(D):
            if counts[i] == 0:
                continue
            e, b, a = hid[i]
            mean = e + b * cum[i] ** -a
            noise = rng.gamma(50.0, 1 / 50.0, size=int(counts[i])).astype(np.float32)
            tl = (mean * noise).astype(np.float32)
            s, c = per_domain_loss(tl.tolist(), [dom[i]] * len(tl))[dom[i]]
            feedback[dom[i]] = (s, c)
        steps.append({
            "pi": pi.tolist(),
            "feedback": {str(i): list(feedback[dom[i]]) for i in range(D) if dom[i] in feedback},
        })
        src.observe_feedback(step, feedback)
    out["ado"] = {
        "prior": [prior_map[k] for k in dom],
        "steps": steps,
        "fit_steps": list(src.state.fit_steps),
        "laws": [[t.law.epsilon, t.law.beta, t.law.alpha, t.law.fallback] if t.law else None
                 for t in (src.state.tracks[k] for k in dom)],
    }
    with gzip.open(HERE / "stage3.json.gz", "wt") as f:
        json.dump(out, f)
    print("stage3: ado steps", len(steps), "fits", out["ado"]["fit_steps"])


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
