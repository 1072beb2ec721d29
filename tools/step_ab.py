"""A/B timing of the BASELINE configs[1] decode step under environment knobs.

    python tools/step_ab.py [--steps 20] [--w4 0,8] [--shape 7b|8b] 'NAME:VAR=V,VAR=V' ...

Each configuration runs in its own child process (the runtime reads its MS_*
knobs once per process); prints ms per step for each W4 layer count and,
with --prof, the per-category kernel time (ms_prof_kernels, serialising).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(steps, w4s, shape, prof, order_kind, reps, bits=4):
    import numpy as np

    import bench
    if bits != 4:
        bench.VARIANTS = (16, bits, 4)
    if shape == "8b":
        from paper_2506_02006_b200.device import LLAMA3_8B
        bench.SHAPE = dict(LLAMA3_8B)
    dev, table = bench.build_model(0, 1, 64)
    slots = np.arange(bench.BATCH, dtype=np.int32)
    if order_kind == "lis":
        order = bench.W4_LAYERS + [l for l in range(32) if l not in bench.W4_LAYERS]
    elif order_kind == "seq":
        order = list(range(32))
    else:
        order = [int(x) for x in order_kind.split(",")]
    cur = set()
    res = {w4: [] for w4 in w4s}
    # configurations interleaved over `reps` rounds (the SM clock drifts down
    # under the power cap during a run, so back-to-back phases are not comparable)
    for _ in range(reps):
        for w4 in w4s:
            want = set(order[:w4])
            for l in sorted(cur - want):
                t = dev.swap_begin(l, 16)
                dev.swap_wait(t)
                dev.swap_commit(t)
            for l in sorted(want - cur):
                t = dev.swap_begin(l, bits)
                dev.swap_wait(t)
                dev.swap_commit(t)
            cur = want
            pos = np.full(bench.BATCH, bench.CTX - 1, dtype=np.int32)
            for _ in range(8):  # graphs of the 3 staging slots are captured on their second sighting
                dev.decode(slots, pos, table, want_next=False)
                pos = pos + 1
            dev.sync()
            dev.timer_start()
            for _ in range(steps):
                dev.decode(slots, pos, table, want_next=False)
                pos = pos + 1
            res[w4].append(dev.timer_stop() / steps)
    out = {w4: {"ms": float(np.mean(v)), "each": [round(x, 4) for x in v]} for w4, v in res.items()}
    if prof:
        dev.prof_kernels(True)
        pos = np.full(bench.BATCH, bench.CTX - 1, dtype=np.int32)
        for _ in range(steps):
            dev.decode(slots, pos, table, want_next=False)
            pos = pos + 1
        out["us_by_kernel"] = {k: round(v[0] / steps * 1e3, 1) for k, v in dev.prof_kernels_read().items()}
        dev.prof_kernels(False)
    print(json.dumps(out))
    dev.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--w4", default="0,8")
    ap.add_argument("--shape", default="7b", choices=["7b", "8b"])
    ap.add_argument("--prof", action="store_true")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--order", default="lis", help="lis | seq | comma-separated layer list")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--bits", type=int, default=4, help="level of the swapped layers (8, 4, 3)")
    ap.add_argument("configs", nargs="*", default=["base:"])
    a = ap.parse_args()
    w4s = [int(x) for x in a.w4.split(",")]
    if a.child:
        child(a.steps, w4s, a.shape, a.prof, a.order, a.reps, a.bits)
        return
    for cfg in a.configs:
        name, _, kv = cfg.partition(":")
        env = dict(os.environ)
        for item in filter(None, kv.split(",")):
            k, _, v = item.partition("=")
            env[k] = v
        cmd = [sys.executable, __file__, "--child", "--steps", str(a.steps), "--w4", a.w4, "--shape", a.shape,
               "--order", a.order, "--reps", str(a.reps), "--bits", str(a.bits)]
        if a.prof:
            cmd.append("--prof")
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        print(name, line[-1] if line else r.stderr[-600:], flush=True)


if __name__ == "__main__":
    main()
