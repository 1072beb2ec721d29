"""W4A16 decode GEMM probe (experiments): per-unit timeline of CTA 0.

    MS_GEMM_DEBUG=8 python tools/w4_probe.py [--name qkv] [--M 64]

Runs one W4 GEMM at a 7B decode shape with the kernel's debug timeline on
(MS_GEMM_DEBUG bit 3: CTA 0 stamps %globaltimer per pipeline event) and
prints, per pipeline unit, the time each event happened relative to the
kernel start (ns).  Events: 0 raw issue, 1 dequant got raw, 2 dequant got A
stage, 3 dequant done, 4 MMA start, 5 B issue, 7 MMAs issued.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from bench_kernels import SHAPES, stream  # noqa: E402
from paper_2506_02006_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", default="qkv")
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--bits", type=int, default=4)
    args = ap.parse_args()
    L = N.lib()
    Nn, K = SHAPES[args.name]
    M, TM = args.M, min(256, (args.M + 15) // 16 * 16)
    w = torch.randint(-2000, 2000, (Nn * K,), dtype=torch.int16, device="cuda")
    if args.bits == 4:
        wp = torch.empty((Nn // 128) * (K // 128) * 8448, dtype=torch.uint8, device="cuda")
        N.check(L.ms_k_quant_w4(C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), None, stream()))
    else:
        wp = torch.empty_like(w)
        N.check(L.ms_k_pack_bf16(C.c_void_p(w.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), stream()))
    xp = torch.randint(-2000, 2000, (((M + TM - 1) // TM) * TM * K,), dtype=torch.int16, device="cuda")
    out = torch.zeros(160 * M * Nn, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    used = C.c_int()
    rows = []
    for rep in range(3):
        flush.fill_(rep)
        out.view(-1)[150 * M * Nn:].zero_()
        torch.cuda.synchronize()
        N.check(L.ms_k_gemm(args.bits, C.c_void_p(wp.data_ptr()), Nn, K, C.c_void_p(xp.data_ptr()), M, TM, 0,
                            C.c_void_p(out.data_ptr()), C.byref(used), stream()))
        torch.cuda.synchronize()
    tl = out.view(-1)[150 * M * Nn:150 * M * Nn + 2 * 8 * 64].view(torch.int64).view(8, 64).cpu()
    t0 = int(tl[6, 0])
    for i in range(64):
        ev = [int(tl[e, i]) for e in range(8)]
        if all(v == 0 for v in ev[:6]):
            continue
        rows.append({"unit": i, **{f"e{e}": (ev[e] - t0 if ev[e] else None) for e in range(8) if e != 6}})
    print(json.dumps({"name": args.name, "M": M, "end_ns": int(tl[6, 1]) - t0 if int(tl[6, 1]) else None}))
    if int(os.environ.get("MS_GEMM_DEBUG", "0")) & 64:  # per-CTA start / end (ns from the earliest start)
        ce = out.view(-1)[150 * M * Nn:150 * M * Nn + 2 * (1024 + 2 * 148)].view(torch.int64)[1024:].view(148, 2).cpu()
        ce = ce[ce[:, 1] > 0]
        sm = (ce[:, 0] >> 48).tolist()
        ce[:, 0] &= (1 << 48) - 1
        ce[:, 1] &= (1 << 48) - 1
        s0 = int(ce[:, 0].min())
        st, en = (ce[:, 0] - s0).tolist(), (ce[:, 1] - s0).tolist()
        q = lambda v, f: sorted(v)[int(f * (len(v) - 1))]
        print(json.dumps({"ctas": len(en), "start_ns": [q(st, f) for f in (0, .5, 1)],
                          "end_ns": [q(en, f) for f in (0, .1, .5, .9, 1)]}))
        if os.environ.get("W4_PROBE_SM"):
            rot = int(os.environ.get("MS_GEMM_DEBUG", "0")) >> 8
            work = [(b + rot) % 148 for b in range(len(en))]  # rows are in blockIdx order
            print(json.dumps({"sm_end": dict(zip(sm, [e - s for s, e in zip(st, en)])),
                              "work_end": dict(zip(work, [e - s for s, e in zip(st, en)]))}))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
