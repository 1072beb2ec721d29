"""The C oracle's decoder is pinned (CPU only, no GPU):

* against the frozen fixture tests/golden/decoder_tiny.npz (BASELINE config 1
  tiny model, prefill + greedy decode with a W4 g128 layer switched in at a
  token boundary): bit-exact, so a change to the oracle's math shows up here
  even if a kernel were changed to match it;
* its fast paths against its plain definitions: the blocked GEMM against the
  sequential fp64 chain (bit-identical), and the batched prefill
  (ref_prefill_rows, used by the full-size GPU parity tests) against the
  token-by-token prefill (bit-identical logits and residual-stream trace).
"""
import os
import sys

import numpy as np

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

TINY = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024, max_pos=128)


def test_decoder_matches_frozen_golden():
    import make_golden as G
    gold = np.load(os.path.join(HERE, "golden", "decoder_tiny.npz"))
    now = G.decoder_tiny()
    for k in gold.files:
        assert np.array_equal(gold[k], now[k]), k


def test_blocked_gemm_is_the_sequential_chain():
    rng = np.random.default_rng(0)
    for B, N, K in [(21, 37, 300), (1, 5, 17), (64, 8, 128), (300, 3, 64)]:
        W = O.f32_to_bf16(rng.uniform(-1, 1, (N, K)).astype(np.float32))
        X = O.f32_to_bf16(rng.uniform(-1, 1, (B, K)).astype(np.float32))
        Y = O.gemm_bf16(W, X)
        Wf = O.bf16_to_f32(W).astype(np.float64)
        Xf = O.bf16_to_f32(X).astype(np.float64)
        ref = np.zeros((B, N))
        for k in range(K):
            ref = ref + Xf[:, k:k + 1] * Wf[None, :, k]
        assert np.array_equal(Y, ref.astype(np.float32)), (B, N, K)


def test_batched_prefill_is_token_by_token():
    rng = np.random.default_rng(9)
    n = 40
    prompt = rng.integers(0, TINY["V"], size=n).astype(np.int32)
    m = O.RefModel(TINY, 7)
    try:
        m.set_precision(2, 4)
        s0 = m.new_seq(64)
        tr0 = m.prefill_trace(s0, prompt)
        s1 = m.new_seq(64)
        nxt0, lg0 = m.prefill(s1, prompt)
        s2 = m.new_seq(64)
        nxt, lg, tr = m.prefill_rows(s2, prompt, want_trace=True)
        assert nxt == nxt0 and np.array_equal(lg, lg0)
        assert np.array_equal(tr, tr0)
        for l in range(TINY["L"]):
            k0, v0 = m.seq_kv(s1, l, n)
            k2, v2 = m.seq_kv(s2, l, n)
            assert np.array_equal(k0, k2) and np.array_equal(v0, v2)
        rows = [0, 5, 17, 38, 39]
        s3 = m.new_seq(64)
        nxt3, lg3, tr3 = m.prefill_rows(s3, prompt, rows=rows, want_trace=True)
        assert nxt3 == nxt0 and np.array_equal(lg3, lg0)
        assert np.array_equal(tr3[:TINY["L"]], tr0[:TINY["L"]])
        assert np.array_equal(tr3[TINY["L"], rows], tr0[TINY["L"], rows])
    finally:
        m.close()
