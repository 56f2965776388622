"""Break the bench's e2e step (pinned host columns -> chunks on the host) into
its parts: H2D copy, device job, result read-back.

    python tools/e2e_breakdown.py [--scale 1.0]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2502_19790_b200 import synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rt = bench.make_workload(0, args.scale)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    cols = bench.device_columns(rt, dev)
    pinned = {p: c.cpu().pin_memory() for p, c in cols.items()}
    del cols
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    out = {}
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dcols = {p: x.to(dev, non_blocking=True) for p, x in pinned.items()}
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        idx, gen, batch = bench.run_step(bench.device_catalog(meta, dcols), spec)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        h = batch.to_host()
        t3 = time.perf_counter()
        nbytes = sum(x.numel() * 4 for x in pinned.values())
        out = {"h2d_ms": (t1 - t0) * 1e3, "h2d_gbs": nbytes / (t1 - t0) / 1e9, "job_ms": (t2 - t1) * 1e3,
               "to_host_ms": (t3 - t2) * 1e3, "ranges": int(batch.n_ranges)}
        del idx, gen, batch, h, dcols
    print(json.dumps({k: round(v, 3) if isinstance(v, float) else v for k, v in out.items()}))


if __name__ == "__main__":
    main()
