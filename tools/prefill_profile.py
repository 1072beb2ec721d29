"""TTFT and per-kernel time of one long prefill (BASELINE configs[3] shape by default).

    python tools/prefill_profile.py [--tokens 8192] [--layers 40] [--w4 0,10] [--reps 3]

For each W4 layer count (LIS order of configs/sequence_lis_40.json) prints the
median prefill time (CUDA events around ms_prefill) and the per-category
kernel time of one further prefill (ms_prof_kernels, events between kernels).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--w4", default="0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-prof", action="store_true")
    a = ap.parse_args()
    from paper_2506_02006_b200.device import LLAMA2_13B, DeviceModel, layer_pages
    shape = dict(LLAMA2_13B, L=a.layers)
    n = a.tokens
    nb = (n + 15) // 16
    w4s = [int(x) for x in a.w4.split(",")]
    dev = DeviceModel(shape, max_batch=8, max_prefill_tokens=n, max_pos=n + 32,
                      arena_pages=shape["L"] * layer_pages(shape, 16) + max(w4s) * layer_pages(shape, 4) + nb + 64)
    dev.weights_synthetic(7)
    dev.hist_reserve(1, n + 2)
    dev.kv_attach(0, nb)
    ids = np.arange(nb, dtype=np.int64)
    dev.hist_write(0, 0, np.random.default_rng(5).integers(0, shape["V"], size=n).astype(np.int32))
    order = [int(x) for x in json.load(open(os.path.join(ROOT, "configs", "sequence_lis_40.json")))["order"]]
    order = [l for l in order if l < a.layers]
    done = 0
    for w4 in w4s:
        for l in order[done:w4]:
            t = dev.swap_begin(l, 4)
            dev.swap_wait(t)
            dev.swap_commit(t)
        done = w4
        dev.prefill(0, n, ids)
        dev.sync()
        ms = []
        for _ in range(a.reps):
            dev.prefill(0, n, ids)
            ms.append(dev.last_step_ms())
        out = {"w4_layers": w4, "ttft_ms": float(np.median(ms)), "each": [round(x, 2) for x in ms]}
        if not a.no_prof:
            dev.prof_kernels(True)
            dev.prefill(0, n, ids)
            out["ms_by_kernel"] = {k: [round(v[0], 2), v[1]] for k, v in dev.prof_kernels_read().items()}
            dev.prof_kernels(False)
        print(json.dumps(out), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
