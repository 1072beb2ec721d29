"""The CPU oracle pinned against the reference: g128 quantizer codes against the
reference quantize_weights (golden + live), the generator golden vector, and the
packed-image layouts against independent unpacking."""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_quantizer_matches_reference_golden():
    for case in json.load(open(os.path.join(GOLD, "quantizer.json"))):
        w = O.f32_to_bf16(np.array(case["weights"], np.float32))
        codes, s64, s16 = O.quantize_groups(w)
        assert codes.tolist() == case["codes"], case["name"]
        assert s64[:, 0].tolist() == case["scales"], case["name"]
        # code * scale is exactly the reference's quantize_weights output
        deq = codes.astype(np.float64) * s64
        assert np.allclose(deq, np.array(case["dequant_ref"]), rtol=0, atol=1e-15)


def test_quantizer_kats_and_bounds():
    # toy_model.cpp KATs: endpoints exact, zero group -> scale 1 / codes 0, half away from zero
    w = O.f32_to_bf16(np.array([[1.0, -1.0] + [0.0] * 126, [0.0] * 128], np.float32))
    codes, s64, _ = O.quantize_groups(w)
    assert codes[0, 0] == 7 and codes[0, 1] == -7 and s64[1, 0] == 1.0 and not codes[1].any()
    rng = np.random.default_rng(7)
    x = O.f32_to_bf16(rng.uniform(-10, 10, (64, 256)).astype(np.float32))
    codes, s64, _ = O.quantize_groups(x)
    xf = O.bf16_to_f32(x).astype(np.float64).reshape(64, 2, 128)
    err = np.abs(xf - codes.reshape(64, 2, 128) * s64[:, :, None])
    assert np.all(err <= s64[:, :, None] / 2 + 1e-12)
    assert codes.min() >= -7 and codes.max() <= 7


@pytest.mark.skipif(not O.have_ref_core(), reason="oracle/_ref not built")
@pytest.mark.parametrize("bits", [8, 4, 3])
def test_quantizer_matches_live_reference(bits):
    """Every precision level of the reference (toy_model.hpp:26 kQ8/kQ4/kQ3):
    the g128 restatement reproduces quantize_weights(rows, bits) exactly
    (codes recovered from the reference's dequantised rows, and the products)."""
    ref = O.ref_core()
    rng = np.random.default_rng(99 + bits)
    w = O.f32_to_bf16((rng.standard_normal((16, 256)) * 0.02).astype(np.float32))
    w[3, :128] = 0  # zero group: scale 1, codes 0
    codes, s64, _ = O.quantize_groups(w, bits=bits)
    rows = O.bf16_to_f32(w).astype(np.float64).reshape(32, 128)
    q = np.array(ref.quantize_weights(rows.tolist(), bits))
    assert np.array_equal(np.round(q / s64.reshape(32, 1)).astype(np.int8).reshape(16, 256), codes)
    assert np.array_equal(q, codes.reshape(32, 128).astype(np.float64) * s64.reshape(32, 1))
    qmax = (1 << (bits - 1)) - 1
    assert codes.min() >= -qmax and codes.max() <= qmax


def test_generator_golden():
    g = json.load(open(os.path.join(GOLD, "generator.json")))
    assert O.gen_weight(g["seed"], g["tensor"], 64, g["scale"], g["offset"]).tolist() == g["first"]


def test_pack_layouts_roundtrip():
    rng = np.random.default_rng(0)
    N, K = 256, 384
    w = O.f32_to_bf16(rng.uniform(-1, 1, (N, K)).astype(np.float32))
    p = O.pack_bf16(w).reshape(N // 128, K // 64, 16, 8, 8, 8)  # [nt][kb][g][c][r][e]
    back = p.transpose(0, 2, 4, 1, 3, 5).reshape(N, K)
    assert np.array_equal(back, w)
    codes, _, s16 = O.quantize_groups(O.f32_to_bf16(rng.uniform(-1, 1, (N, K)).astype(np.float32)))
    img = O.pack_w4(codes, s16).reshape(N // 128, K // 128, 8448)
    for nt in range(N // 128):
        for g in range(K // 128):
            chunk = img[nt, g]
            words = chunk[:8192].view(np.uint32).reshape(4, 128, 4)  # [j][row][w]
            shifts = np.array([(e & 1) * 16 + (e >> 1) * 4 for e in range(8)], np.uint32)
            nib = ((words[..., None] >> shifts) & 0xF).astype(np.int16) - 8
            dec = nib.transpose(1, 0, 2, 3).reshape(128, 128)  # [row][j*32 + w*8 + e]
            assert np.array_equal(dec, codes[nt * 128:(nt + 1) * 128, g * 128:(g + 1) * 128])
            assert np.array_equal(chunk[8192:].view(np.uint16), s16[nt * 128:(nt + 1) * 128, g])


def test_pack_w8_layout():
    rng = np.random.default_rng(1)
    N, K = 256, 384
    codes, _, s16 = O.quantize_groups(O.f32_to_bf16(rng.uniform(-1, 1, (N, K)).astype(np.float32)), bits=8)
    img = O.pack_w8(codes, s16).reshape(N // 128, K // 128, 16640)
    for nt in range(N // 128):
        for g in range(K // 128):
            chunk = img[nt, g]
            b = chunk[:16384].reshape(8, 128, 16).astype(np.int16) - 128  # [j][row][e]
            dec = b.transpose(1, 0, 2).reshape(128, 128)
            assert np.array_equal(dec, codes[nt * 128:(nt + 1) * 128, g * 128:(g + 1) * 128])
            assert np.array_equal(chunk[16384:].view(np.uint16), s16[nt * 128:(nt + 1) * 128, g])
    # Q3 codes use the 4-bit container layout
    c3, _, s3 = O.quantize_groups(O.f32_to_bf16(rng.uniform(-1, 1, (N, K)).astype(np.float32)), bits=3)
    assert np.array_equal(O.pack_quant(c3, s3, 3), O.pack_w4(c3, s3))


def test_oracle_forward_deterministic_and_prefill_equals_decode():
    cfg = dict(L=2, d=256, H=4, KVH=2, hd=64, ffn=256, V=512, max_pos=64)
    m = O.RefModel(cfg, 3)
    s1, s2 = m.new_seq(64), m.new_seq(64)
    toks = np.arange(10, dtype=np.int32) * 37 % 512
    a, la = m.prefill(s1, toks)
    for t in toks[:-1]:
        m.forward([s2], [t], want_logits=False)
    b, lb = m.forward([s2], [toks[-1]])
    assert a == b[0] and np.array_equal(la, lb[0])
    m.close()
