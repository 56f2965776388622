"""Host-side breakdown of one cfg2 job (wall clock per API call, GPU synced).

    python tools/host_profile.py [--scale 1.0] [--reps 3]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, build_index_from_catalog, synth
    from paper_2502_19790_b200.catalog import ColumnarCatalog

    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rt = bench.make_workload(0, a.scale)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    cols = bench.device_columns(rt, torch.device("cuda"))
    spec = synth.cfg2_mixture()
    for rep in range(a.reps):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dcat = DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols})
        torch.cuda.synchronize(); t["catalog"] = time.perf_counter() - t0; t0 = time.perf_counter()
        idx = build_index_from_catalog(dcat, [])
        torch.cuda.synchronize(); t["index"] = time.perf_counter() - t0; t0 = time.perf_counter()
        gen = ChunkGenerator(idx, 42)
        torch.cuda.synchronize(); t["gen"] = time.perf_counter() - t0; t0 = time.perf_counter()
        batch = gen.plan_batch(spec, 1 << 40)
        torch.cuda.synchronize(); t["plan"] = time.perf_counter() - t0; t0 = time.perf_counter()
        del idx, gen, batch
        torch.cuda.synchronize(); t["free"] = time.perf_counter() - t0
        print(rep, {k: round(v * 1e3, 3) for k, v in t.items()}, "total", round(sum(t.values()) * 1e3, 2), "ms")


if __name__ == "__main__":
    main()
