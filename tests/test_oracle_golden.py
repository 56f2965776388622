"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py). No GPU needed."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import STAGE12_CASES, golden_predicates, load_golden, load_stage3


def _key(orc, s):
    from paper_2502_19790_b200.mixtures import MixtureKey

    return orc.as_key(MixtureKey.parse(s))


@pytest.mark.parametrize("case", STAGE12_CASES)
def test_oracle_index_and_cursors_match_reference(oracle, case):
    cc, g = load_golden(case)
    idx = oracle.build_index(cc, golden_predicates(g))
    assert [list(r) for r in idx.table()] == g["index"]
    gen = oracle.OracleGenerator(idx, g["job_seed"])
    assert [oracle.key_string(idx.keys[r]) for r in gen.order] == g["component_order"]
    for r, k in enumerate(idx.keys):
        assert [list(x) for x in gen.ranges[r]] == g["cursors"][oracle.key_string(k)]


@pytest.mark.parametrize("case", STAGE12_CASES)
def test_oracle_chunks_match_reference(oracle, case):
    cc, g = load_golden(case)
    idx = oracle.build_index(cc, golden_predicates(g))
    for name, run in g["runs"].items():
        gen = oracle.OracleGenerator(idx, g["job_seed"])
        got, states = [], {}
        for i in range(len(run["chunks"]) + int(run.get("exhausted", True))):
            if i in (1, 3):
                states[str(i)] = gen.state_dict()
            if name.startswith("arbitrary"):
                c = gen.generate_arbitrary(int(name[len("arbitrary"):]))
            else:
                m = g["mixtures"][name]
                w = {_key(oracle, k): v for k, v in m["weights"].items()}
                c = gen.generate(w, m["chunk_size"], m["strict"])
            if c is None:
                break
            got.append(c.serialize().decode("ascii"))
        assert len(got) == len(run["chunks"]), name
        for a, b in zip(got, run["chunks"]):
            assert a == b, name
        if run["report"] is not None:
            assert {oracle.key_string(k): v for k, v in gen.last_report.items()} == run["report"]
        for i, st in run["states"].items():
            assert states[i] == st
        assert gen.state_dict() == run["final_state"]


def test_oracle_state_restore_resumes(oracle):
    cc, g = load_golden("cfg1_r64")
    idx = oracle.build_index(cc, [])
    m = g["mixtures"]["disjoint"]
    w = {_key(oracle, k): v for k, v in m["weights"].items()}
    run = g["runs"]["disjoint"]
    gen = oracle.OracleGenerator(idx, g["job_seed"])
    gen.load_state(run["states"]["3"])
    nxt = gen.generate(w, m["chunk_size"], m["strict"])
    assert nxt.serialize().decode() == run["chunks"][3]


def test_oracle_per_domain_loss_exact(oracle):
    g = load_stage3()["per_domain_loss"]
    sums, counts = oracle.per_domain_loss(np.array(g["losses"], np.float32), g["tags"], len(g["sums"]))
    assert sums.tolist() == g["sums"]
    assert counts.tolist() == g["counts"]


def test_oracle_fit_power_law_exact(oracle):
    for case in load_stage3()["fits"]:
        law = oracle.fit_power_law([tuple(p) for p in case["points"]])
        assert list(law) == case["law"]


def test_oracle_ado_trajectory_exact(oracle):
    g = load_stage3()["ado"]
    ado = oracle.OracleAdo(g["prior"])
    D = len(g["prior"])
    for step, rec in enumerate(g["steps"], start=1):
        pi = ado.compute_pi()
        assert pi == rec["pi"], step
        sums = np.zeros(D)
        counts = np.zeros(D, np.int64)
        for i, (s, c) in rec["feedback"].items():
            sums[int(i)], counts[int(i)] = s, c
        ado.observe(step, sums, counts)
    assert ado.fit_steps == g["fit_steps"]
    assert [list(l) if l else None for l in ado.law] == g["laws"]
