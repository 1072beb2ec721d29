"""Per-CTA timeline of the fused decode-layer kernel (layer.cu) in the 7B
bench step (experiment tool, B200 only).

    MS_GRAPH=0 MS_LAYER_TL=<layer> python tools/layer_timeline.py [--steps 3]

Builds the bench model (BASELINE configs[1]: B=64, ctx 2048, 8 W4 layers) and
runs eager decode steps; the runtime prints min / median / max over CTAs of
each event (epilogue last tile, grid-barrier pass, row phase done, activation
producer go, first MMA, first weight issue) per phase of that layer's launch.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--w4", type=int, default=8)
    args = ap.parse_args()
    dev, table = bench.build_model(0, 1, args.steps + 4)
    for l in bench.W4_LAYERS[: args.w4]:
        t = dev.swap_begin(l, 4)
        dev.swap_wait(t)
        dev.swap_commit(t)
    slots = np.arange(bench.BATCH, dtype=np.int32)
    pos = np.full(bench.BATCH, bench.CTX - 1, dtype=np.int32)
    for i in range(args.steps):
        print(f"--- step {i}", file=sys.stderr, flush=True)
        dev.decode(slots, pos, table, want_next=False)
        dev.sync()
        pos = pos + 1
    dev.close()


if __name__ == "__main__":
    main()
