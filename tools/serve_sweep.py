"""Serving-load exploration on the B200 (experiment tool).

    python tools/serve_sweep.py --shape 7b --rps 20,30,40 --out 128,256 --seconds 8

Runs the morph-performance and static-full arms of a Gamma-burst trace through
the C++ engine on a DeviceModel (GPU clock) and prints P95 TTFT / TPOT, SLO
violations, swaps, preemptions and wall time per point, to pick bench loads that
put the static arm under memory pressure.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="7b", choices=["7b", "8b"])
    ap.add_argument("--rps", default="20,30")
    ap.add_argument("--out", default="128")
    ap.add_argument("--prompt", type=int, default=0)
    ap.add_argument("--seconds", type=float, default=8.0)
    ap.add_argument("--arms", default="morph-performance,static-full")
    a = ap.parse_args()
    from paper_2506_02006_b200 import serving as S
    from paper_2506_02006_b200.device import LLAMA2_7B, LLAMA3_8B, DeviceModel, layer_pages, page_bytes
    shape = dict(LLAMA2_7B if a.shape == "7b" else LLAMA3_8B)
    prompt = a.prompt or (512 if a.shape == "7b" else 1024)
    max_out = max(int(x) for x in a.out.split(","))
    pb = page_bytes(shape)
    budget_pages = int(24.0 * (1 << 30)) // pb
    dev = DeviceModel(shape, device=0, max_batch=256, max_prefill_tokens=prompt + max_out + 16,
                      max_pos=prompt + max_out + 32, arena_pages=budget_pages + 2 * layer_pages(shape, 16) + 64)
    dev.weights_synthetic(7)
    for out in [int(x) for x in a.out.split(",")]:
        for rps in [float(x) for x in a.rps.split(",")]:
            wl = {"gamma": {"seed": 101, "rps": rps, "shape": 0.25, "total_ms": int(a.seconds * 1000),
                            "prompt_tokens": prompt, "output_tokens": out}}
            cfg = S.device_config(dev, wl, budget_gib=24.0, reserve_gib=4.0)
            for arm in a.arms.split(","):
                t0 = time.time()
                rep, _ = S.serve(dev, cfg, arm, clock="device")
                sm = S.summary(rep)
                print(json.dumps({"shape": a.shape, "rps": rps, "out": out, "arm": arm, "wall_s": round(time.time() - t0, 1),
                                  "p95_ttft_ms": sm["p95_ttft_ms"], "p95_tpot_ms": sm["p95_tpot_ms"],
                                  "slo": sm["slo_violations"], "swaps": sm["swap_events"],
                                  "restores": sm["restore_events"], "peakq": sm["peak_quantized_layers"],
                                  "preempt": sm["preemptions"], "kv_peak": sm["kv_peak_blocks"],
                                  "kv_static": sm["kv_static_blocks"], "decode_tok_s": sm["decode_tok_s"],
                                  "requests": sm["requests"]}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
