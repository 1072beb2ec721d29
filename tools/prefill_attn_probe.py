"""Causal prefill attention at the 13B 8k shape, one layer (experiments / ncu).

    python tools/prefill_attn_probe.py [--n 8192] [--H 40] [--reps 5]

Times ms_k_attn_prefill with CUDA events (H=40 heads, hd 128, one layer of
paged KV filled with random bf16); useful flops = 4 * H * hd * sum_q (q + 1).
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_02006_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--H", type=int, default=40)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--layers", type=int, default=1, help="layers per KV page (40 = the 13B serving geometry)")
    a = ap.parse_args()
    n, H, hd, L = a.n, a.H, 128, a.layers
    page_bytes = 16 * L * H * 2 * hd * 2
    nb = (n + 15) // 16
    arena = torch.empty((nb * page_bytes // 2,), dtype=torch.int16, device="cuda")
    for c in arena.split(1 << 28):
        r = torch.randint(-16000, 16000, c.shape, dtype=torch.int16, device="cuda")
        c.copy_((r.view(torch.bfloat16).float().clamp(-1, 1) * 0.5).to(torch.bfloat16).view(torch.int16))
    pages = torch.randperm(nb, dtype=torch.int32, device="cuda")
    q = torch.randn(n * H * hd, dtype=torch.float32, device="cuda")
    out = torch.empty(n * H * hd, dtype=torch.int16, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def run():
        N.check(N.lib().ms_k_attn_prefill(C.c_void_p(q.data_ptr()), C.c_void_p(arena.data_ptr()), page_bytes, L, L // 2,
                                          H, H, hd, C.c_void_p(pages.data_ptr()), n, C.c_void_p(out.data_ptr()), st))
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    flops = 4.0 * H * hd * n * (n + 1) / 2
    print(json.dumps({"n": n, "H": H, "layers_per_page": L, "ms": ms, "tflops": flops / ms / 1e9, "each": [round(t, 4) for t in ts]}))



def timeline():
    """(experiment) MS_LIB_DIR=<lib built with MS_NVCC_EXTRA=-DMS_PATTN_TL>: CTA 0 event timeline."""
    lib = N.lib()
    buf = (C.c_ulonglong * (8 * 128))()
    lib.ms_dbg_pattn_tl(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(8, 128).astype(np.int64)
    t0 = a[a > 0].min()
    names = ["S_A", "S_B", "PV_A", "PV_B", "smA_gotS", "smB_gotS", "smA_P", "smB_P"]
    for kt in range(128):
        row = {nm: int(a[e, kt] - t0) if a[e, kt] else None for e, nm in enumerate(names)}
        if all(v is None for v in row.values()):
            continue
        print(json.dumps({"kt": kt, **row}))


if __name__ == "__main__":
    main()
    if os.environ.get("MS_PATTN_TL"):
        timeline()
