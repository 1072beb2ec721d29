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
          "lm_head": (32000, 4096)}


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def time_it(fn, iters=50, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def gemm(bits, Nn, K, M, TM, ctas=0):
    L = N.lib()
    w = torch.randint(-2000, 2000, (Nn * K,), dtype=torch.int16, device="cuda")
    if bits == 16:
        wp = torch.empty_like(w)
        N.check(L.ms_k_pack_bf16(C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), stream()))
        wbytes = Nn * K * 2
    else:
        wp = torch.empty((Nn // 128) * (K // 128) * 8448, dtype=torch.uint8, device="cuda")
        N.check(L.ms_k_quant_w4(C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), None, stream()))
        wbytes = Nn * K // 2 + Nn * K // 128 * 2
    xp = torch.randint(-2000, 2000, (((M + TM - 1) // TM) * TM * K,), dtype=torch.int16, device="cuda")
    out = torch.zeros(160 * M * Nn, dtype=torch.float32, device="cuda")
    used = C.c_int()

    def run():
        N.check(L.ms_k_gemm(bits, C.c_void_p(wp.data_ptr()), Nn, K, C.c_void_p(xp.data_ptr()), M, TM, ctas,
                            C.c_void_p(out.data_ptr()), C.byref(used), stream()))
    ms = time_it(run)
    total = wbytes + M * K * 2 + M * Nn * 4
    return {"bits": bits, "N": Nn, "K": K, "M": M, "us": ms * 1e3, "GBps": total / ms / 1e6, "slots": used.value}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="gemm")
    ap.add_argument("--M", type=int, default=64)
    args = ap.parse_args()
    res = []
    if "gemm" in args.which:
        for name, (Nn, K) in SHAPES.items():
            for bits in (16, 4):
                if name == "lm_head" and bits == 4:
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
