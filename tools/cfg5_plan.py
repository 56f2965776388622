import sys; sys.path.insert(0,'.')
import numpy as np, torch, bench
from paper_2502_19790_b200 import DeviceCatalog, MixtureSpec, build_index_from_catalog, synth, ChunkGenerator
from paper_2502_19790_b200.catalog import ColumnarCatalog
rt = synth.config("cfg5")
meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
cols = bench.device_columns(rt, torch.device("cuda", 0))
dcat = DeviceCatalog(meta, columns=cols, nullable={p: False for p in cols})
idx = build_index_from_catalog(dcat, [])
keys = idx.component_keys()
rng = np.random.Generator(np.random.PCG64(5))
w = 1.0 / np.arange(1, len(keys) + 1) ** 0.8
w = w[rng.permutation(len(keys))]; w /= w.sum()
spec = MixtureSpec({k: float(x) for k, x in zip(keys, w)}, 1024)
gen = ChunkGenerator(idx, 42)
import time
t0=time.perf_counter(); b = gen.plan_batch(spec, 200); torch.cuda.synchronize(); print("200 chunks", time.perf_counter()-t0, b.n_chunks)
# CUPTI kernel summary of a 2000-chunk plan
from torch.profiler import ProfilerActivity, profile
gen = ChunkGenerator(idx, 42)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter(); b = gen.plan_batch(spec, 2000); torch.cuda.synchronize(); wall = time.perf_counter() - t0
print("2000 chunks wall", wall, b.n_chunks)
for e in sorted(prof.key_averages(), key=lambda e: -(getattr(e, "device_time_total", 0) or 0))[:12]:
    print(f"{(getattr(e, 'device_time_total', 0) or 0) / 1e3:10.2f} ms dev  {e.cpu_time_total / 1e3:10.2f} ms cpu  x{e.count:5d}  {e.key[:70]}")
