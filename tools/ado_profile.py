"""Host profile of the ADO step loop (cfg4 shape): where the per-step
latency goes (python tools/ado_profile.py)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2502_19790_b200 import (AdoConfig, AdoSource, AdoState, ChunkGenerator, DeviceCatalog, MixtureKey,  # noqa
                                   build_index_from_catalog, synth)
from paper_2502_19790_b200.ado import domain_loss_device  # noqa: E402

D = 22
dom = [f"x{i:02d}" for i in range(D)]
cc = synth.expand_numpy(synth.make_runs(10_000_000, 1000, {"domain": dom}, 64, seed=4))
idx = build_index_from_catalog(DeviceCatalog(cc), [])
keys = [MixtureKey.of({"domain": d}) for d in dom]
prior = np.random.Generator(np.random.PCG64(4)).dirichlet(np.ones(D))
src = AdoSource(AdoState(AdoConfig(), dict(zip(keys, prior))), 1024)
gen = ChunkGenerator(idx, 42)
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(4)
losses = torch.rand(131072, device=dev, generator=g) + 1.5
tags = torch.randint(0, D, (131072,), device=dev, generator=g, dtype=torch.int32)


def step(s):
    spec = src.current_spec()
    gen.generate(spec)
    sums, counts = domain_loss_device(losses, tags, D)
    hs, hc = sums.cpu().numpy(), counts.cpu().numpy()
    src.observe_feedback(s, {keys[i]: (float(hs[i]), int(hc[i])) for i in range(D)})


for s in range(1, 50):
    step(s)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for s in range(50, 550):
    step(s)
pr.disable()
print("us/step", (time.perf_counter() - t0) / 500 * 1e6)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
