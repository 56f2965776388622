import sys, time, ctypes as C
sys.path.insert(0, '.')
import torch, bench
from paper_2502_19790_b200 import synth, _lib, ChunkGenerator
from paper_2502_19790_b200.index import ChunkerIndex, build_index_from_catalog
from paper_2502_19790_b200.catalog import ColumnarCatalog
from paper_2502_19790_b200.seeding import hash_message, derive_seed
rt = bench.make_workload(0, 1.0)
meta = ColumnarCatalog.meta_only(rt.vocab, rt.file_sizes)
cols = bench.device_columns(rt, torch.device("cuda", 0))
dcat = bench.device_catalog(meta, cols)
spec = synth.cfg2_mixture(1024)
for rep in range(6):
    torch.cuda.synchronize()
    L = _lib.lib()
    t0 = time.perf_counter()
    preds = dcat.host.validated([])
    desc, keep = dcat.descriptor(preds)
    t1 = time.perf_counter()
    out = C.c_void_p()
    _lib.check(L.mx_index_build(C.byref(desc), C.c_void_p(_lib.stream_ptr(None)), C.byref(out)))
    t2 = time.perf_counter()
    idx = ChunkerIndex(out.value, dcat, None)
    t3 = time.perf_counter()
    cur = hash_message(42, "cursor"); chk = hash_message(42, "chunk"); os_ = derive_seed(42, "component-order")
    t4 = time.perf_counter()
    gen = ChunkGenerator(idx, 42)
    t5 = time.perf_counter()
    b = gen.plan_batch(spec, 1 << 40)
    t6 = time.perf_counter()
    del b, gen, idx
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    print(f"desc {1e6*(t1-t0):.0f} build {1e6*(t2-t1):.0f} ChunkerIndex {1e6*(t3-t2):.0f} hashes {1e6*(t4-t3):.0f} gen {1e6*(t5-t4):.0f} plan {1e6*(t6-t5):.0f} free {1e6*(t7-t6):.0f} us")
