"""Regenerates the frozen golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref, built from /root/reference by oracle/Makefile) and the
C oracle.  Run in the build container (the reference sources are not on the
GPU box):  python tests/golden/make_golden.py

Fixtures:
  quantizer.json   reference quantize_weights (toy_model.cpp:40-60) on g128 groups,
                   expressed as integer codes + fp64 scales (bit-exact targets)
  kvpool.json      reference KvBlockPool op sequences and their results
  generator.json   first values of the counter RNG weight generator (C oracle)
  engine_*.log     reference event logs for small engine scenarios (sha256 + text)
  decoder_tiny.npz the C oracle's Llama-style decoder on BASELINE config 1 (tiny
                   model, seed 7): prefill logits of 4 prompts, then 12 greedy
                   decode steps with layer 1 switched to W4 g128 after step 4
                   (logits + tokens).  Freezes the decoder contract (DESIGN.md
                   section 4) so that a matched change to the oracle and a
                   kernel cannot pass silently: tests/test_oracle_decoder.py
                   recomputes it bit for bit.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def quantizer(ref):
    out = []
    rng = np.random.default_rng(1234)
    cases = [
        ("kat_endpoints", [[1.0, -1.0] + [0.0] * 126]),
        ("kat_zero_group", [[0.0] * 128]),
        ("kat_half_away", [[2.5 / 7 * 7, -2.5, 7.0] + [0.0] * 125]),
        ("random_small", (rng.uniform(-1, 1, (4, 128)) * 0.05).tolist()),
        ("random_wide", (rng.uniform(-3, 3, (2, 128))).tolist()),
    ]
    for name, rows in cases:
        rows = [[float(O.bf16_to_f32(O.f32_to_bf16(np.array(r, np.float32)))[i]) for i in range(len(r))]
                for r in rows]
        q = ref.quantize_weights(rows, 4)
        scales = []
        codes = []
        for r, qr in zip(rows, q):
            m = max(abs(v) for v in r)
            s = 1.0 if m == 0 else m / 7.0
            scales.append(s)
            codes.append([int(round(qv / s)) for qv in qr])
        out.append({"name": name, "weights": rows, "codes": codes, "scales": scales, "dequant_ref": q})
    return out


def kvpool(ref):
    seqs = []
    # the survey golden (cap 8, bt 16) and a deferred-detach scenario
    p = ref.KvBlockPool(ref.KvConfig(16, 2 << 20, 8))
    log = []
    p.admit(1); log.append(["alloc", 1, 32, p.alloc_for_tokens(1, 32)])
    p.admit(2); log.append(["alloc", 2, 17, p.alloc_for_tokens(2, 17)])
    log.append(["attach", 3, p.attach_blocks(3)])
    p.admit(3); log.append(["alloc", 3, 20, p.alloc_for_tokens(3, 20)])
    log.append(["release", 1, p.release(1)])
    p.admit(4); log.append(["alloc", 4, 48, p.alloc_for_tokens(4, 48)])
    log.append(["detach", 3, list(p.detach_blocks(3))])
    seqs.append({"name": "survey_a9", "capacity": 8, "ops": log})
    return seqs


def generator():
    return {"seed": 7, "tensor": 17, "scale": 0.0625, "offset": 0.0,
            "first": O.gen_weight(7, 17, 64, 0.0625).tolist()}


TINY = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024, max_pos=128)


def decoder_tiny():
    """(prompts, prefill logits, decode tokens, decode logits) of the oracle."""
    rng = np.random.default_rng(3)
    B, P, steps = 4, 24, 12
    prompts = rng.integers(0, TINY["V"], size=(B, P)).astype(np.int32)
    m = O.RefModel(TINY, 7)
    try:
        seqs = [m.new_seq(P + steps + 1) for _ in range(B)]
        pre, toks = [], []
        for b in range(B):
            t, lg = m.prefill(seqs[b], prompts[b])
            pre.append(lg)
            toks.append(t)
        toks = np.array(toks, np.int32)
        dtok, dlog = [], []
        for step in range(steps):
            if step == 4:
                m.set_precision(1, 4)
            nxt, lg = m.forward(seqs, toks)
            dtok.append(nxt.copy())
            dlog.append(lg.copy())
            toks = nxt
    finally:
        m.close()
    return dict(prompts=prompts, prefill_logits=np.array(pre, np.float32), decode_tokens=np.array(dtok, np.int32),
                decode_logits=np.array(dlog, np.float32), first_tokens=np.array([int(np.argmax(x)) for x in pre],
                                                                                np.int32))


def main():
    O.build(ref=False)
    np.savez_compressed(os.path.join(HERE, "decoder_tiny.npz"), **decoder_tiny())
    O.build(ref=True)
    ref = O.ref_core()
    with open(os.path.join(HERE, "quantizer.json"), "w") as f:
        json.dump(quantizer(ref), f)
    with open(os.path.join(HERE, "kvpool.json"), "w") as f:
        json.dump(kvpool(ref), f)
    with open(os.path.join(HERE, "generator.json"), "w") as f:
        json.dump(generator(), f)
    # reference engine logs for the tests' small scenarios
    sys.path.insert(0, os.path.dirname(HERE))
    from scenarios import SCENARIOS  # noqa: PLC0415
    index = {}
    for name, (cfg, arm) in SCENARIOS.items():
        import tempfile
        d = tempfile.mkdtemp()
        cfg = dict(cfg)
        if arm.startswith("morph"):
            seq = os.path.join(d, "seq.json")
            ref.save_sequence(ref.baseline_sequence("front_to_back", cfg["model"]["num_layers"], 0, 4), seq)
            cfg["sequence_file"] = seq
        rep = json.loads(ref.run_arm(json.dumps(cfg), arm, d))
        text = open(os.path.join(d, f"events_{arm}.log")).read()
        with open(os.path.join(HERE, f"engine_{name}.log"), "w") as f:
            f.write(text)
        rep.pop("fingerprint")
        index[name] = {"sha256": hashlib.sha256(text.encode()).hexdigest(), "report": rep}
    with open(os.path.join(HERE, "engine_index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
