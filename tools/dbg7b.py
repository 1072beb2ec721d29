"""Debug: 2-layer 7B-shaped decode with one layer swapped to W4 (sanitizer runs)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_02006_b200.device import DeviceModel, layer_pages  # noqa: E402

S = dict(L=2, d=4096, H=32, KVH=32, hd=128, ffn=11008, V=32000)
B, CTX = 64, 256
bps = (CTX + 64) // 16 + 1
kv_pages = B * bps
dev = DeviceModel(S, device=0, max_batch=B, max_prefill_tokens=256, max_pos=CTX + 64,
                  arena_pages=kv_pages + S["L"] * layer_pages(S, 16) + layer_pages(S, 4) + 8)
dev.weights_synthetic(7)
dev.hist_reserve(B, CTX + 64)
dev.kv_attach(0, kv_pages)
table = np.arange(kv_pages, dtype=np.int64).reshape(bps, B).T.copy()
dev.kv_fill_synthetic(table.reshape(-1), seed=11)
slots = np.arange(B, dtype=np.int32)
pos = np.full(B, CTX - 1, dtype=np.int32)
for i in range(2):
    nxt, lg = dev.decode(slots, pos, table, want_logits=True)
    print("step", i, "next", nxt[:8], "logit finite", np.isfinite(lg).all(), "absmax", np.abs(lg).max(), flush=True)
    print("hist", dev.hist_read(0, int(pos[0]) - 1, 3), flush=True)
    pos += 1
dev.sync()
print("bf16 ok", flush=True)
t = dev.swap_begin(1, 4)
dev.swap_wait(t)
dev.swap_commit(t)
for i in range(2):
    dev.decode(slots, pos, table, want_next=False)
    pos += 1
dev.sync()
print("w4 ok", flush=True)
