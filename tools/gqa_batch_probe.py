"""Per-kernel decode time of the Llama-3-8B shape at several batch sizes.

    python tools/gqa_batch_probe.py [--batches 37,64,74] [--steps 20]

Each batch runs in its own child process.  Prints ms per step and the
per-category kernel time (ms_prof_kernels, serialising) so the GQA attention's
time per (row, kv_head) item can be compared across whole and partial waves
(2 CTAs per SM x 148 SMs = 296 items per wave).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(batch, steps):
    import numpy as np

    import bench
    from paper_2506_02006_b200.device import LLAMA3_8B
    bench.SHAPE = dict(LLAMA3_8B)
    bench.BATCH = batch
    dev, table = bench.build_model(0, 1, 64)
    slots = np.arange(batch, dtype=np.int32)
    pos = np.full(batch, bench.CTX - 1, dtype=np.int32)
    for _ in range(8):
        dev.decode(slots, pos, table, want_next=False)
        pos = pos + 1
    dev.sync()
    dev.timer_start()
    for _ in range(steps):
        dev.decode(slots, pos, table, want_next=False)
        pos = pos + 1
    ms = dev.timer_stop() / steps
    dev.prof_kernels(True)
    for _ in range(steps):
        dev.decode(slots, pos, table, want_next=False)
        pos = pos + 1
    us = {k: round(v[0] / steps * 1e3, 1) for k, v in dev.prof_kernels_read().items()}
    dev.prof_kernels(False)
    print(json.dumps({"batch": batch, "ms_per_step": round(ms, 4), "us_by_kernel": us}))
    dev.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="37,64,74")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--child", type=int, default=0)
    a = ap.parse_args()
    if a.child:
        child(a.child, a.steps)
        return
    for b in a.batches.split(","):
        r = subprocess.run([sys.executable, __file__, "--child", b, "--steps", str(a.steps)], capture_output=True,
                           text=True)
        print(r.stdout.strip().splitlines()[-1] if r.returncode == 0 else "batch %s failed: %s" % (b, r.stderr[-800:]),
              flush=True)


if __name__ == "__main__":
    main()
