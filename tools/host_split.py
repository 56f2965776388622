"""Host wall time of each public call of one bench step (no profiler):
build_index_from_catalog / ChunkGenerator / plan_batch, each without a sync
(what the host spends issuing it) and the final sync (device tail).

    python tools/host_split.py [--layout tuples|columns]
"""
import argparse
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_19790_b200 import ChunkGenerator, build_index_from_catalog, synth  # noqa: E402
from paper_2502_19790_b200.catalog import ColumnarCatalog  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layout", default="tuples")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rt = bench.make_workload(0, 1.0)
    meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    cols, table = bench.layout_columns(rt, bench.device_columns(rt, dev), args.layout)
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    dcat = bench.device_catalog(meta, cols, table)
    rows = []
    for rep in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx = build_index_from_catalog(dcat, [])
        t1 = time.perf_counter()
        gen = ChunkGenerator(idx, bench.CFG["job_seed"])
        t2 = time.perf_counter()
        batch = gen.plan_batch(spec, 1 << 40)
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        del batch, gen, idx
        rows.append([1e6 * (t1 - t0), 1e6 * (t2 - t1), 1e6 * (t3 - t2), 1e6 * (t4 - t3), 1e6 * (t4 - t0)])
    import statistics
    med = [statistics.median(r[i] for r in rows[2:]) for i in range(5)]
    print("median us: index %.0f  generator %.0f  plan_batch %.0f  tail-sync %.0f  total %.0f" % tuple(med))


if __name__ == "__main__":
    main()
