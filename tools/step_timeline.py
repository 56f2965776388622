"""Where a bench step's wall time goes: host wall-clock per API call (with
device syncs) next to the library's per-phase CUDA-event times.

    python tools/step_timeline.py [--scale 1.0] [--reps 5]
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
from paper_2502_19790_b200 import ChunkGenerator, DeviceCatalog, _lib, build_index_from_catalog, synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    rt = bench.make_workload(0, args.scale)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    cols = bench.device_columns(rt, dev)
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    rows = []
    for rep in range(args.reps + 2):
        torch.cuda.synchronize()
        L.mx_profile_reset()
        L.mx_profile_enable(1)
        t = [time.perf_counter()]
        dcat = DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols})
        t.append(time.perf_counter())
        idx = build_index_from_catalog(dcat, [])
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        gen = ChunkGenerator(idx, bench.CFG["job_seed"])
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        batch = gen.plan_batch(spec, 1 << 40)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        del batch, gen, idx
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        L.mx_profile_enable(0)
        ph = {p: round(_lib.profile_read(p)[0], 4) for p in ("scan_runs", "radix_sort", "index_scans",
                                                            "cursor_layout", "cursor_shuffle", "plan", "emit")}
        if rep >= 2:
            ms = [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])]
            rows.append({"catalog_ms": ms[0], "index_ms": ms[1], "gen_ms": ms[2], "plan_emit_ms": ms[3],
                         "free_ms": ms[4], "total_ms": round((t[-1] - t[0]) * 1e3, 3), "phases_ms": ph})
    print(json.dumps(rows[-1]))
    print(json.dumps({k: round(sum(r[k] for r in rows) / len(rows), 3) for k in rows[0] if k != "phases_ms"}))


if __name__ == "__main__":
    main()
