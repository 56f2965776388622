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


def test_schedule_mixture_switches_mid_look_ahead(mixplane, tmp_path):
    """ScheduleSource (mixtures.py:360-463): the spec changes with training
    feedback while the device generator has planned ahead; every worker must
    still receive the stock server's bytes (the generator rewinds to the
    last handed-out chunk on a spec change, chunks.py here)."""
    from paper_2502_19790_b200 import dropin

    mp = mixplane
    cat = _corpus(mp, tmp_path, seed=13, files=10)
    K = mp.MixtureKey.of
    sched = mp.MixtureSchedule([
        (0, mp.MixtureSpec({K({"language": "python"}): 0.7, K({"language": "go"}): 0.3}, 24)),
        (3, mp.MixtureSpec({K({"license": "mit"}): 0.5, K({"license": ["apache", "gpl"]}): 0.5}, 24)),
        (7, mp.MixtureSpec({K({"language": ["rust", "c"]}): 0.4, K({"language": "python"}): 0.6}, 30)),
    ])
    args = mp.QueryExecutionArgs(sched, dp_groups=1, nodes_per_group=1, num_workers=2, seed=5)
    q = mp.Query.for_job("sched")

    def run(server):
        server.submit_query(q, args)
        got = []
        for step in range(1, 12):
            for w in range(2):
                got.append(server.next_chunk("sched", 0, 0, w, step - 1))
            server.receive_feedback("sched", step, {K({"language": "python"}): (1.0, 1)})
        return got

    ref = run(mp.MixplaneServer(cat))
    undo = dropin.install(mp)
    try:
        got = run(mp.MixplaneServer(dropin.gpu_catalog(cat)))
    finally:
        undo()
    assert len(ref) == len(got) and got == ref


def test_ado_checkpoint_round_trip_through_server(mixplane, tmp_path):
    """ADO job checkpointed mid-run and restored (server.py:244-286): the
    device AdoSource state (fit history, credit, pi, pi_bar, step) survives
    the round trip, and the restored job continues exactly like the job that
    was never interrupted; both track the stock server's pi within 1e-5."""
    from paper_2502_19790_b200 import dropin

    mp = mixplane
    cat = _corpus(mp, tmp_path, seed=21, files=12)
    prior = {"language:python": 0.4, "language:go": 0.3, "language:rust": 0.2, "language:c": 0.1}
    cfg = {"fit_start_step": 20, "refit_every": 20, "discard_first": 2, "subsample_every": 2}
    args = mp.QueryExecutionArgs(mp.query.ado_mixture(16, prior, cfg), seed=4)
    q = mp.Query.for_job("adock")
    rng = np.random.default_rng(1)
    feedback = [{mp.MixtureKey.parse(k): (float(rng.uniform(2, 3) * 64 / (1 + s / 30)), 64) for k in prior}
                for s in range(70)]

    def run(server, restore_at=None):
        server.submit_query(q, args)
        pis = []
        for step, fb in enumerate(feedback, start=1):
            server.next_chunk("adock", 0, 0, 0, step - 1)
            server.receive_feedback("adock", step, fb)
            if step == restore_at:
                cid = server.checkpoint("adock")
                server.restore(cid)
            pis.append({k.canonical_string(): v for k, v in server._job("adock").source.state.pi.items()})
        return pis

    ref = run(mp.MixplaneServer(cat))
    undo = dropin.install(mp)
    try:
        plain = run(mp.MixplaneServer(dropin.gpu_catalog(cat)))
        restored = run(mp.MixplaneServer(dropin.gpu_catalog(cat)), restore_at=33)
    finally:
        undo()
    assert restored == plain  # the round trip is lossless on the device state
    worst = max(abs(b[k] - a[k]) / a[k] for a, b in zip(ref, plain) for k in a)
    assert worst < 1e-5, worst


def test_tcp_error_frames_carry_reference_kinds(mixplane, tmp_path):
    """Through the TCP server (server.py:463-491) with the drop-in, errors the
    device path raises reach the client with the reference's ``kind``:
    an unknown property -> QueryError, a replayed feedback step ->
    FeedbackError (which the client itself treats as an ack,
    client.py:269-272), an un-keyable catalog never reaches 'internal'."""
    from mixplane.protocol import ServerReply

    from paper_2502_19790_b200 import dropin

    mp = mixplane
    cat = _corpus(mp, tmp_path, seed=2)
    undo = dropin.install(mp, catalogs=True)
    server = mp.MixplaneServer(cat)
    host, port = server.start()
    try:
        client = mp.MixplaneClient(host, port, attempts=3)
        K = mp.MixtureKey.of
        spec = mp.MixtureSpec({K({"language": "python"}): 1.0}, 16)
        with pytest.raises(ServerReply) as ei:
            client.submit_query(mp.Query.for_job("bad").select(("colour", "==", "red")),
                                mp.QueryExecutionArgs(spec))
        assert ei.value.kind == "QueryError"
        with pytest.raises(ServerReply) as ei:
            client.submit_query(mp.Query.for_job("none").select(("language", "==", "cobol")),
                                mp.QueryExecutionArgs(spec))
        assert ei.value.kind == "QueryError" and "matches no samples" in str(ei.value)
        prior = {"language:python": 0.5, "language:go": 0.5}
        client.submit_query(mp.Query.for_job("ado"), mp.QueryExecutionArgs(mp.query.ado_mixture(8, prior)))
        fb = {K({"language": "python"}): (3.0, 2)}
        assert client.feedback("ado", 1, fb)["status"] == "ok"
        assert client.feedback("ado", 1, fb)["status"] == "ok"  # replay: FeedbackError -> ack (client.py:269)
        with pytest.raises(ServerReply) as ei:
            client._call(mp.protocol.TASK_FEEDBACK, {"job_id": "ado", "step": 1, "losses": {}})
        assert ei.value.kind == "FeedbackError"
        with pytest.raises(ServerReply) as ei:
            client.feedback("ado", 2, {K({"language": "cobol"}): (1.0, 1)})
        assert ei.value.kind == "FeedbackError"
        assert client.next_chunk("ado", 0, 0, 0, 0) is not None
        client.close()
    finally:
        server.stop()
        undo()
