"""Per-kernel time of one long prefill (BASELINE configs[3] shape by default).

    python tools/prefill_profile.py [--tokens 8192] [--layers 40]
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
    a = ap.parse_args()
    from paper_2506_02006_b200.device import LLAMA2_13B, DeviceModel, layer_pages
    shape = dict(LLAMA2_13B, L=a.layers)
    n = a.tokens
    nb = (n + 15) // 16
    dev = DeviceModel(shape, max_batch=8, max_prefill_tokens=n, max_pos=n + 32,
                      arena_pages=shape["L"] * layer_pages(shape, 16) + nb + 64)
    dev.weights_synthetic(7)
    dev.hist_reserve(1, n + 2)
    dev.kv_attach(0, nb)
    ids = np.arange(nb, dtype=np.int64)
    dev.hist_write(0, 0, (np.arange(n) % shape["V"]).astype(np.int32))
    dev.prefill(0, n, ids)
    dev.sync()
    dev.prof_kernels(True)
    dev.prefill(0, n, ids)
    prof = dev.prof_kernels_read()
    print(json.dumps({k: [round(v[0], 2), v[1]] for k, v in prof.items()}))
    dev.close()


if __name__ == "__main__":
    main()
