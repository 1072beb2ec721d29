"""Kernel microbenchmarks on the B200 (CUDA events, warm, back-to-back launches).

    python tools/bench_kernels.py [--which gemm,attn]

Times the tcgen05 GEMM (BF16 and W4A16) at the Llama-2-7B decode shapes
(M = 64) and the paged attention kernel, reporting algorithmic GB/s.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_02006_b200 import _native as N  # noqa: E402

SHAPES = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008),
          "lm_head": (32000, 4096),
          # Llama-2-13B (BASELINE configs[3] prefill): d 5120, ffn 13824
          "qkv13": (15360, 5120),
          # fixed per-launch cost probes
          "t256": (256, 128), "t4k": (4096, 128), "t4k1k": (4096, 1024), "o13": (5120, 5120), "gate_up13": (27648, 5120), "down13": (5120, 13824)}


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def time_it(fn, iters=50, warm=5):
    """Average device time per call; the calls are replayed from a CUDA graph
    so that host launch cost (ctypes + plan) does not floor small kernels."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def gemm(bits, Nn, K, M, TM, ctas=0):
    """One GEMM shape; the weights rotate over enough copies (> 300 MB) that
    every call streams them from HBM, not from the 126 MB L2."""
    L = N.lib()
    w = torch.randint(-2000, 2000, (Nn * K,), dtype=torch.int16, device="cuda")
    if bits == 16:
        wp = torch.empty_like(w)
        N.check(L.ms_k_pack_bf16(C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), stream()))
        wbytes = Nn * K * 2
    else:
        chunk = 16640 if bits == 8 else 8448
        wp = torch.empty((Nn // 128) * (K // 128) * chunk, dtype=torch.uint8, device="cuda")
        N.check(L.ms_k_quant(bits, C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), None, stream()))
        wbytes = (Nn // 128) * (K // 128) * (chunk - 256) + Nn * K // 128 * 2
    del w
    copies = [wp] + [wp.clone() for _ in range(min(63, max(0, -(-300_000_000 // wp.numel() // wp.element_size()) - 1)))]
    xp = torch.randint(-2000, 2000, (((M + TM - 1) // TM) * TM * K,), dtype=torch.int16, device="cuda")
    out = torch.zeros((160 if M <= 256 else 4) * M * Nn, dtype=torch.float32, device="cuda")
    used = C.c_int()
    i = [0]

    def run():
        w_ = copies[i[0] % len(copies)]
        i[0] += 1
        N.check(L.ms_k_gemm(bits, C.c_void_p(w_.data_ptr()), Nn, K, C.c_void_p(xp.data_ptr()), M, TM, ctas,
                            C.c_void_p(out.data_ptr()), C.byref(used), stream()))
    ms = time_it(run, iters=4 * len(copies) if len(copies) > 12 else 48, warm=len(copies) + 2)
    total = wbytes + M * K * 2 + M * Nn * 4
    tflops = 2.0 * M * Nn * K / (ms * 1e-3) / 1e12
    return {"bits": bits, "N": Nn, "K": K, "M": M, "us": ms * 1e3, "GBps": total / ms / 1e6, "TFLOPs": tflops,
            "slots": used.value, "copies": len(copies)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="gemm")
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--names", default=",".join(SHAPES))
    ap.add_argument("--bits", default="16,4")
    args = ap.parse_args()
    res = []
    if "gemm" in args.which:
        for name in args.names.split(","):
            Nn, K = SHAPES[name]
            for bits in [int(b) for b in args.bits.split(",")]:
                if name == "lm_head" and bits != 16:
                    continue
                r = gemm(bits, Nn, K, args.M, min(256, (args.M + 15) // 16 * 16))
                r["name"] = name
                res.append(r)
                print(json.dumps(r), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "bench_kernels.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
