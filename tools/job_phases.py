"""Phase breakdown (library CUDA-event phases) of one job on a synthetic
catalog: cfg2 (100M) or the cfg3 shape on one GPU (1B), u16 row tuples.

    python tools/job_phases.py [--cfg cfg3] [--reps 3]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2502_19790_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg3")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec = synth.cfg2_mixture(bench.CFG["chunk_size"])
    rt = synth.config(args.cfg) if args.cfg != "cfg2" else bench.make_workload(0, 1.0)
    meta = synth.ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
    codes, table = bench.run_level_tuples(rt, dev)
    cat = bench.device_catalog(meta, {"tuples": codes}, table)
    L = _lib.lib()
    bench.run_step(cat, spec)
    torch.cuda.synchronize()
    L.mx_profile_reset()
    L.mx_profile_enable(1)
    ms = bench._timed_steps(lambda: bench.run_step(cat, spec), args.reps, 0)
    L.mx_profile_enable(0)
    ph = {}
    for p in ("scan_runs", "radix_sort", "index_scans", "cursor_layout", "cursor_shuffle", "plan", "emit"):
        t, n = _lib.profile_read(p)
        ph[p] = round(t / max(n, 1), 3)
    print(json.dumps({"cfg": args.cfg, "samples": rt.n_samples, "ms_per_job": ms, "phases_ms": ph}))


if __name__ == "__main__":
    main()
