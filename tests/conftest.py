"""Shared test plumbing: GPU marker, golden-vector loading, oracle import.

``-m "not gpu"`` tests run on the CPU build container (oracle vs golden
vectors, host logic, C-ABI symbol checks); ``-m gpu`` tests call the CUDA
path through the C-ABI and compare it with the oracle and the goldens.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

STAGE12_CASES = ["cfg1_r1", "cfg1_r64", "cfg2_small", "filters_nulls", "multi_tags", "depletion", "cfg5_small", "cfg5_wide"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running (full-size properties)")


def load_golden(name: str):
    """(ColumnarCatalog, payload) of one committed golden case."""
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    with gzip.open(GOLDEN / f"{name}.json.gz", "rt") as f:
        payload = json.load(f)
    z = np.load(GOLDEN / f"{name}.npz")
    cols = {k[4:]: z[k] for k in z.files if k.startswith("col_")}
    vocab = {p: [tuple(v) if isinstance(v, list) else v for v in vs] for p, vs in payload["vocab"].items()}
    cc = ColumnarCatalog(
        columns=cols, vocab=vocab, multiple=payload["multiple"],
        file_ids=z["file_ids"], file_ds=z["file_ds"], file_offsets=z["file_offsets"],
    )
    return cc, payload


def load_stage3():
    with gzip.open(GOLDEN / "stage3.json.gz", "rt") as f:
        return json.load(f)


def golden_predicates(payload):
    return [(p, op, v if op in ("==", "!=") else tuple(v)) for p, op, v in payload["predicates"]]


def spec_from_json(d):
    from paper_2502_19790_b200.mixtures import MixtureSpec

    return MixtureSpec.from_json(d)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc

    return orc
