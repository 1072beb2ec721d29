"""Decode attention rate vs KV page geometry (kernel entry ms_k_attn_decode).

    python tools/attn_geom_probe.py

Same rows / context, three head layouts: the Llama-3-8B GQA shape (32/8 heads,
2 MiB pages), the MHA kernel on the same 2 MiB page geometry (8/8 heads), and
the Llama-2-7B MHA shape (32/32, 8 MiB pages).  Prints GB/s of KV bytes per
launch (CUDA events around each call; the entry's page-table D2H read adds a
few us per call).
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_02006_b200 import _native as N  # noqa: E402


def run(H, KVH, rows=64, ctx=2048, L=32, hd=128, iters=10, pad=0, spread=1, perm=False):
    page_bytes = 16 * L * KVH * 2 * hd * 2 + pad  # pad: page stride beyond one block's bytes
    nb = (ctx + 15) // 16
    n_pages = rows * nb
    # spread: the same pages placed every `spread`-th page of a larger arena
    arena = torch.empty(n_pages * spread * page_bytes // 2, dtype=torch.int16, device="cuda").random_(-2000, 2000)
    # interleaved ids as in bench.build_model: row r's block j -> page j * rows + r
    ids = torch.randperm(n_pages, device="cuda").to(torch.int32) if perm else torch.arange(n_pages, dtype=torch.int32,
                                                                                          device="cuda")
    pages = (ids * spread).reshape(nb, rows).t().contiguous()
    q = torch.randn(rows, H, hd, device="cuda")
    d_ctx = torch.full((rows,), ctx, dtype=torch.int32, device="cuda")
    out = torch.empty(rows * H * hd, dtype=torch.int16, device="cuda")
    ws = torch.empty(16 * rows * H * (hd + 2), dtype=torch.float32, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ts = []
    for i in range(iters + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.check(N.lib().ms_k_attn_decode(C.c_void_p(q.data_ptr()), C.c_void_p(arena.data_ptr()), page_bytes, L, 5,
                                         H, KVH, hd, C.c_void_p(pages.data_ptr()), nb, C.c_void_p(d_ctx.data_ptr()),
                                         rows, 1, C.c_void_p(ws.data_ptr()), C.c_void_p(out.data_ptr()), st))
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    us = ts[len(ts) // 2] * 1e3
    kv = rows * ctx * KVH * hd * 4
    del arena
    torch.cuda.empty_cache()
    return {"H": H, "KVH": KVH, "page_MiB": page_bytes / 2**20, "us": round(us, 1), "kv_MB": kv / 1e6,
            "GB_s": round(kv / us / 1e3, 1)}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "tlb":
        # MHA kernel, 2048 items each: the per-layer slice of a page that one
        # 2 MB translation serves (256 KB vs 64 KB) at equal page size
        for H, KVH, rows, L in [(32, 32, 64, 32), (32, 32, 64, 8), (8, 8, 256, 32), (8, 8, 256, 8)]:
            r = run(H, KVH, rows=rows, L=L)
            r.update(rows=rows, L=L, slice_KB=KVH * 2 * 128 * 16 * 2 // 1024)
            print(json.dumps(r), flush=True)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pad":
        # same pages, stride padded: concurrent reads no longer share their offset modulo 2 MiB
        for H, KVH in [(32, 8), (8, 8)]:
            for pad in (0, 8192, 65536, 262144):
                print(json.dumps(dict(run(H, KVH, pad=pad), pad=pad)), flush=True)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "spread":
        # same bytes, pages spread over a 1x / 2x / 4x larger arena, or randomly permuted
        for H, KVH in [(32, 8), (8, 8)]:
            for sp, pm in ((1, False), (2, False), (4, False), (1, True), (4, True)):
                print(json.dumps(dict(run(H, KVH, spread=sp, perm=pm), spread=sp, perm=pm)), flush=True)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "gqa":  # run under MS_ATTN_GQA_MMA=0 / 1
        for rows in (64, 16):
            print(json.dumps(dict(run(32, 8, rows=rows), rows=rows)), flush=True)
        sys.exit(0)
    for H, KVH in [(32, 8), (8, 8), (32, 32)]:
        print(json.dumps(run(H, KVH)), flush=True)
    # 8B GQA with a 4x longer context per row (fewer rows in flight per byte)
    print(json.dumps(run(32, 8, rows=16, ctx=8192)), flush=True)
