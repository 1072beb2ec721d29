"""Offline LIS layer profile of a Llama-shaped model on the B200.

    python tools/gpu_profile.py --shape 7b --prompts 2 --tokens 64 --out configs/sequence_gpu_lis_32.json

Random-init weights (seed 7, as everywhere else), synthetic calibration prompts;
writes the reference sequence-JSON schema (profiler.cpp:198-214) that
morphsim.load_sequence / the engine consume.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="7b", choices=["tiny", "7b", "8b"])
    ap.add_argument("--prompts", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2506_02006_b200 import morphsim as M
    from paper_2506_02006_b200.device import LLAMA2_7B, LLAMA3_8B, TINY, DeviceModel, layer_pages
    from paper_2506_02006_b200.profiler import GpuProfiler
    shape = {"tiny": TINY, "7b": LLAMA2_7B, "8b": LLAMA3_8B}[a.shape]
    pages = shape["L"] * layer_pages(shape, 16) + 2 * layer_pages(shape, 4) + 64
    dev = DeviceModel(shape, max_batch=4, max_prefill_tokens=a.tokens, max_pos=a.tokens + 16, arena_pages=pages)
    dev.weights_synthetic(7)
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, shape["V"], size=a.tokens).astype(np.int32) for _ in range(a.prompts)]
    prof = GpuProfiler(dev, prompts)
    t0 = time.time()
    seq = prof.greedy_sequence()
    wall = time.time() - t0
    prof.close()
    dev.close()
    print(json.dumps({"shape": a.shape, "order": seq["order"], "wall_s": round(wall, 1), "forwards": prof.forwards,
                      "lts": [round(x, 6) for x in seq["lts"]], "lrs": [round(x, 6) for x in seq["lrs"]]}))
    if a.out:
        M.save_sequence(seq, a.out)


if __name__ == "__main__":
    main()
