"""Where does a 7B decode step go?  (experiment tool, B200 only)

    python tools/step_breakdown.py [--steps 10] [--w4 0|8|32]

Times the BASELINE configs[1] decode step (B=64, ctx 2048) with parts of the
step switched off through MS_SKIP (runtime.cu skip_mask: bit0 qkv_post, bit1
residual_norm, bit2 silu_mul, bit3 attention, bit4 layer GEMMs) -- one child
process per mask because the mask is read once per process.  Differences
between masks are the in-step cost of each part (PDL overlap included).
Results become numerically meaningless when anything is skipped.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MASKS = {"full": 0, "no_rows": 7, "no_qkvpost": 1, "no_norm": 2, "no_silu": 4, "no_attn": 8, "no_gemm": 16, "no_attn_rows": 15, "gemm_only": 15,
         "rows_only": 24, "nothing": 31}


def child(steps, w4, shape):
    import numpy as np

    import bench
    if shape == "8b":  # Llama-3-8B (GQA 32/8), BASELINE configs[2] decode shape
        from paper_2506_02006_b200.device import LLAMA3_8B
        bench.SHAPE = dict(LLAMA3_8B)
    dev, table = bench.build_model(0, 4 * steps + 16)
    layers = list(range(32)) if w4 == 32 else bench.W4_LAYERS[:w4]
    for l in layers:
        t = dev.swap_begin(l, 4)
        dev.swap_wait(t)
        dev.swap_commit(t)
    slots = np.arange(bench.BATCH, dtype=np.int32)
    pos = np.full(bench.BATCH, bench.CTX - 1, dtype=np.int32)
    for _ in range(3):
        dev.decode(slots, pos, table, want_next=False)
        pos = pos + 1
    dev.sync()
    dev.timer_start()
    for _ in range(steps):
        dev.decode(slots, pos, table, want_next=False)
        pos = pos + 1
    ms = dev.timer_stop() / steps
    prof = {}
    if os.environ.get("PROF"):
        dev.prof_kernels(True)
        for _ in range(steps):
            dev.decode(slots, pos, table, want_next=False)
            pos = pos + 1
        prof = {k: (round(v[0] / steps * 1e3, 1), v[1] // steps) for k, v in dev.prof_kernels_read().items()}
    print(json.dumps({"ms_per_step": ms, "us_per_step_by_kernel": prof}))
    dev.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--w4", type=int, default=8)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--shape", default="7b", choices=["7b", "8b"])
    ap.add_argument("--masks", default="full,no_rows,no_attn,no_gemm,gemm_only,nothing")
    a = ap.parse_args()
    if a.child:
        child(a.steps, a.w4, a.shape)
        return
    res = {}
    for name in a.masks.split(","):
        env = dict(os.environ, MS_SKIP=str(MASKS[name]))
        out = subprocess.run([sys.executable, __file__, "--child", "--steps", str(a.steps), "--w4", str(a.w4),
                              "--shape", a.shape],
                             env=env, capture_output=True, text=True)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        res[name] = json.loads(line[-1]) if line else out.stderr[-400:]
        print(name, res[name], flush=True)
    print(json.dumps({"w4_layers": a.w4, "ms_per_step": res}))


if __name__ == "__main__":
    main()
