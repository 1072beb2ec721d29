"""The opt-in kernel variants keep oracle parity: the tiny-model smoke decode
(prefill logits, greedy decode, a W4 swap at a token boundary and a KV attach,
each checked against the CPU oracle inside __graft_entry__.smoke) is re-run in a
child process with each switch set (the switches are read once per process).

    MS_GRAPH=0         decode steps launched eagerly (no CUDA-graph replay)
    MS_ATTN_SPLITS=3   forced split-KV (combine kernel) on the decode path
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"MS_GRAPH": "0"}, {"MS_ATTN_SPLITS": "3"}, {"MS_PDL": "0"}])
def test_variant_smoke_matches_oracle(env):
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT,
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "smoke ok" in r.stdout, (env, r.stdout[-2000:], r.stderr[-4000:])


# hd 128 shapes exercise the paths the tiny model (hd 64) does not: the MHA
# warp-per-block consumer (G = 1) and the GQA tensor-core / TMA consumer (G = 4),
# both with the QKV post-processing fused into attention.
@pytest.mark.parametrize("shape", [dict(L=2, d=512, H=4, KVH=4, hd=128, ffn=1024, V=1024),
                                   # V > 8192: the vocab-chunked argmax
                                   dict(L=2, d=512, H=4, KVH=1, hd=128, ffn=1024, V=16384)])
def test_hd128_decode_matches_oracle(shape):
    import numpy as np

    import oracle as O
    from paper_2506_02006_b200.device import DeviceModel, layer_pages

    ctx_max = 160
    pages = 2 * shape["L"] * layer_pages(shape, 16) + layer_pages(shape, 4) + 64
    dev = DeviceModel(shape, max_batch=4, max_prefill_tokens=128, max_pos=ctx_max, arena_pages=pages)
    ref = O.RefModel(dict(shape, max_pos=ctx_max), 7)
    try:
        dev.weights_synthetic(7)
        dev.hist_reserve(2, ctx_max)
        dev.kv_attach(0, 20)
        table = np.arange(20, dtype=np.int64).reshape(2, 10)
        n0 = [100, 37]  # prompt lengths: 7 and 3 blocks, partial last blocks
        seqs = [ref.new_seq(ctx_max) for _ in range(2)]
        toks = []
        for b in range(2):
            prompt = ((np.arange(n0[b], dtype=np.int32) * 131 + 17 * b) % shape["V"]).astype(np.int32)
            dev.hist_write(b, 0, prompt)
            t, lg = dev.prefill(b, n0[b], table[b], want_logits=True)
            _, rl = ref.prefill(seqs[b], prompt)
            assert np.max(np.abs(lg - rl)) <= 2e-2 * np.max(np.abs(rl))
            toks.append(t)
        pos = np.array(n0, np.int32)
        toks = np.array(toks, np.int32)
        for step in range(6):
            if step == 3:  # W4 swap of layer 1 at a token boundary, freed pages carved into KV ids
                t = dev.swap_begin(1, 4)
                dev.swap_wait(t)
                freed = dev.swap_commit(t)
                dev.kv_attach(100, freed - layer_pages(shape, 4))
                ref.set_precision(1, 4)
            got, lg = dev.decode(np.arange(2), pos, table, want_logits=True)
            _, rl = ref.forward(seqs, toks)
            for b in range(2):
                assert np.max(np.abs(lg[b] - rl[b])) <= 2e-2 * np.max(np.abs(rl[b])), (step, b)
                assert got[b] == int(np.argmax(lg[b])), (step, b)  # greedy token of the device logits, lowest id on ties
            toks = got
            pos += 1
    finally:
        ref.close()
        dev.close()
