"""Debug: GPU per-layer residual traces vs the oracle (profiler inputs)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle as O  # noqa: E402
from paper_2506_02006_b200.device import DeviceModel  # noqa: E402
from paper_2506_02006_b200.profiler import GpuProfiler  # noqa: E402

CFG = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024)
PROMPTS = [((np.arange(24, dtype=np.int32) * 37 + 5 * i) % 1024).astype(np.int32) for i in range(3)]
m = O.RefModel(dict(CFG, max_pos=128), 7)
refs = [m.prefill_trace(m.new_seq(64), p) for p in PROMPTS]
m.close()
dev = DeviceModel(CFG, max_batch=4, max_prefill_tokens=64, max_pos=128, arena_pages=512)
dev.weights_synthetic(7)
prof = GpuProfiler(dev, PROMPTS)
gs = prof.traces(set())
for i, (g, r) in enumerate(zip(gs, refs)):
    print(i, [float(np.abs(g[l] - r[l]).max() / np.abs(r[l]).max()) for l in range(CFG["L"] + 1)])
dev.close()
