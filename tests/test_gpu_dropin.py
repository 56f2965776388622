"""Drop-in integration: the reference's OWN server (mixplane, installed under
baseline/_ref) run twice in one process -- stock CPU path vs the same server
with the B200 index / generator / ADO installed by ``dropin.install`` -- must
hand every (group, node, worker) identical chunk bytes, survive checkpoint /
restore identically, and track the same ADO mixture."""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def mixplane():
    if not (REF / "mixplane").exists():
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, str(REF))
    import mixplane as mp

    return mp


def _corpus(mp, tmp_path, seed=3, files=8, props=("language", "license")):
    from mixplane.formats import write_jsonl

    rng = np.random.default_rng(seed)
    vals = {"language": ["python", "go", "rust", "c"], "license": ["mit", "apache", "gpl"]}
    paths = []
    for f in range(files):
        recs, cur = [], None
        for i in range(int(rng.integers(150, 400))):
            if cur is None or rng.random() < 0.08:
                cur = {p: str(rng.choice(vals[p])) for p in props}
            recs.append({"text": f"f{f} s{i}", **cur})
        path = tmp_path / f"part{f}.jsonl"
        write_jsonl(path, recs)
        paths.append(path)
    cat = mp.MetadataCatalog()
    cat.register_dataset("code", paths, mp.JsonFieldParser.for_properties(list(props)),
                         mp.PropertySchema([mp.PropertyDef(p) for p in props]))
    return cat


def _stream(server, job, args):
    out = {}
    for g in range(args.dp_groups):
        for n in range(args.nodes_per_group):
            for w in range(max(1, args.num_workers)):
                pos, blobs = 0, []
                while (b := server.next_chunk(job, g, n, w, pos)) is not None:
                    blobs.append(b)
                    pos += 1
                out[(g, n, w)] = blobs
    return out


def _both(mp, catalog_factory, query, args):
    from paper_2502_19790_b200 import dropin

    stock = mp.MixplaneServer(catalog_factory())
    stock.submit_query(query, args)
    ref = _stream(stock, query.job_id, args)
    undo = dropin.install(mp)
    try:
        gpu = mp.MixplaneServer(dropin.gpu_catalog(catalog_factory()))
        gpu.submit_query(query, args)
        got = _stream(gpu, query.job_id, args)
    finally:
        undo()
    return ref, got


@pytest.mark.parametrize("mixture_kind", ["static", "strict", "inferring", "arbitrary", "hierarchical"])
def test_server_streams_identical_bytes(mixplane, tmp_path, mixture_kind):
    mp = mixplane
    cat = _corpus(mp, tmp_path)
    K = mp.MixtureKey.of
    mixtures = {
        "static": mp.MixtureSpec({K({"language": "python"}): 0.5, K({"license": ["mit", "gpl"]}): 0.5}, 64),
        "strict": mp.MixtureSpec({K({"language": "go"}): 0.3, K({"language": "rust"}): 0.7}, 50, strict=True),
        "inferring": mp.query.inferring_mixture(40),
        "arbitrary": mp.query.arbitrary_chunks(100),
        "hierarchical": mp.HierarchicalMixtureSpec(
            mp.HierarchyNode("language", [
                mp.HierarchyBranch(("python",), 0.6, mp.HierarchyNode("license", [
                    mp.HierarchyBranch(("mit",), 0.5), mp.HierarchyBranch(("apache", "gpl"), 0.5)])),
                mp.HierarchyBranch(("go", "c"), 0.4)]), 80),
    }
    query = mp.Query.for_job("j").select(("license", "!=", "apache")) if mixture_kind == "inferring" \
        else mp.Query.for_job("j")
    args = mp.QueryExecutionArgs(mixtures[mixture_kind], dp_groups=2, nodes_per_group=2, num_workers=2, seed=7)
    ref, got = _both(mp, lambda: cat, query, args)
    assert sum(len(v) for v in ref.values()) > 0
    assert got == ref


def test_checkpoint_restore_matches_stock(mixplane, tmp_path):
    from paper_2502_19790_b200 import dropin

    mp = mixplane
    cat = _corpus(mp, tmp_path, seed=5)
    K = mp.MixtureKey.of
    spec = mp.MixtureSpec({K({"language": "python"}): 0.25, K({"language": ["go", "c"]}): 0.75}, 32)
    args = mp.QueryExecutionArgs(spec, dp_groups=1, nodes_per_group=1, num_workers=2, seed=11)
    q = mp.Query.for_job("ck")

    def run(server):
        server.submit_query(q, args)
        first = [server.next_chunk("ck", 0, 0, w, p) for p in range(3) for w in range(2)]
        cid = server.checkpoint("ck")
        server.restore(cid)  # rebuilds the job (stage 1 again) and loads cursor state
        rest = {}
        for w in range(2):
            pos, blobs = server.register("ck", 0, 0, w)["position"], []
            while (b := server.next_chunk("ck", 0, 0, w, pos)) is not None:
                blobs.append(b)
                pos += 1
            rest[w] = blobs
        return first, rest

    ref = run(mp.MixplaneServer(cat))
    undo = dropin.install(mp)
    try:
        got = run(mp.MixplaneServer(dropin.gpu_catalog(cat)))
    finally:
        undo()
    assert got == ref


def test_ado_job_tracks_reference_mixture(mixplane, tmp_path):
    from paper_2502_19790_b200 import dropin

    mp = mixplane
    cat = _corpus(mp, tmp_path, seed=9, files=12)
    prior = {"language:python": 0.4, "language:go": 0.3, "language:rust": 0.2, "language:c": 0.1}
    cfg = {"fit_start_step": 40, "refit_every": 40, "discard_first": 5, "subsample_every": 2}
    args = mp.QueryExecutionArgs(mp.query.ado_mixture(16, prior, cfg), seed=3)
    q = mp.Query.for_job("ado")
    rng = np.random.default_rng(0)
    feedback = [{k: (float(rng.uniform(2, 3) * 64 / (1 + s / 50)), 64) for k in prior} for s in range(120)]

    def run(server):
        server.submit_query(q, args)
        job = server._job("ado")
        pis = []
        for step, fb in enumerate(feedback, start=1):
            server.next_chunk("ado", 0, 0, 0, step - 1)
            server.receive_feedback("ado", step, fb)
            pis.append(dict(job.source.state.pi))
        return pis

    ref = run(mp.MixplaneServer(cat))
    undo = dropin.install(mp)
    try:
        got = run(mp.MixplaneServer(dropin.gpu_catalog(cat)))
    finally:
        undo()
    worst = 0.0
    for a, b in zip(ref, got):
        for k, v in a.items():
            mine = next(x for kk, x in b.items() if kk.canonical_string() == k.canonical_string())
            worst = max(worst, abs(mine - v) / v)
    assert worst < 1e-5, worst
