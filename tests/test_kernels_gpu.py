"""Kernel-level parity: every CUDA kernel on the hot path against the CPU oracle
(oracle/ref_llama.c) on the same seeded inputs.  Integer / byte work is
bit-exact; floating point within the tolerance stated in each test.
Runs only on a B200 (-m gpu), through the C ABI (include/morphserve.h).
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _native():
    from paper_2506_02006_b200 import _native as N
    return N


def dev_u16(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def to_np_u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def test_generator_bit_exact():
    N = _native()
    for tensor, n, scale, off in [(0, 1 << 16, 1.0, 0.0), (17, 4096, 0.1, 1.0), (99, 123457, 1 / 64.0, 0.0)]:
        out = torch.empty(n, dtype=torch.int16, device="cuda")
        N.check(N.lib().ms_k_gen_weight(7, tensor, n, scale, off, C.c_void_p(out.data_ptr()), stream()))
        torch.cuda.synchronize()
        assert np.array_equal(to_np_u16(out), O.gen_weight(7, tensor, n, scale, off))


@pytest.mark.parametrize("N_,K", [(128, 64), (256, 256), (512, 768), (1536, 256)])
def test_pack_bf16_bit_exact(N_, K):
    N = _native()
    w = O.gen_weight(3, 5, N_ * K, 0.05).reshape(N_, K)
    dw = dev_u16(w)
    out = torch.empty(N_ * K, dtype=torch.int16, device="cuda")
    N.check(N.lib().ms_k_pack_bf16(C.c_void_p(dw.data_ptr()), N_, K, C.c_void_p(out.data_ptr()), stream()))
    torch.cuda.synchronize()
    assert np.array_equal(to_np_u16(out), O.pack_bf16(w))


@pytest.mark.parametrize("bits", [4, 8, 3])
@pytest.mark.parametrize("N_,K", [(128, 128), (256, 768), (512, 256)])
def test_quant_codes_and_image_bit_exact(N_, K, bits):
    """g128 quantiser + packer at every precision level (Q4 / Q8 / Q3) against
    the oracle restatement of quantize_weights (toy_model.cpp:47-60)."""
    N = _native()
    w = O.gen_weight(11, 6, N_ * K, 0.02).reshape(N_, K).copy()
    w[3, :128] = 0          # all-zero group -> scale 1, codes 0 (toy_model.cpp:43,53)
    w[5, 128 - 1] = w[5, 0]  # ties are fine, exercise equal maxima
    dw = dev_u16(w)
    chunk = 16640 if bits == 8 else 8448
    img = torch.empty((N_ // 128) * (K // 128) * chunk, dtype=torch.uint8, device="cuda")
    codes = torch.empty(N_ * K, dtype=torch.int8, device="cuda")
    N.check(N.lib().ms_k_quant(bits, C.c_void_p(dw.data_ptr()), N_, K, C.c_void_p(img.data_ptr()),
                               C.c_void_p(codes.data_ptr()), stream()))
    torch.cuda.synchronize()
    rc, _, rs = O.quantize_groups(w, bits=bits)
    assert np.array_equal(codes.cpu().numpy().reshape(N_, K), rc)
    assert np.array_equal(img.cpu().numpy(), O.pack_quant(rc, rs, bits))


def _run_gemm(bits, W, X, TM, splits=0):
    """W [N,K] bf16 (np u16), X [M,K] bf16 -> fp32 [M,N] (sum of split partials)."""
    N = _native()
    Nn, K = W.shape
    M = X.shape[0]
    dw = dev_u16(W)
    if bits == 16:
        wp = torch.empty(Nn * K, dtype=torch.int16, device="cuda")
        N.check(N.lib().ms_k_pack_bf16(C.c_void_p(dw.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), stream()))
    else:
        chunk = 16640 if bits == 8 else 8448
        wp = torch.empty((Nn // 128) * (K // 128) * chunk, dtype=torch.uint8, device="cuda")
        N.check(N.lib().ms_k_quant(bits, C.c_void_p(dw.data_ptr()), Nn, K, C.c_void_p(wp.data_ptr()), None,
                                   stream()))
    m_tiles = (M + TM - 1) // TM
    xp = torch.zeros(m_tiles * TM * K, dtype=torch.int16, device="cuda")
    dx = dev_u16(X)
    N.check(N.lib().ms_k_pack_act(C.c_void_p(dx.data_ptr()), M, K, TM, C.c_void_p(xp.data_ptr()), stream()))
    out = torch.zeros(16 * M * Nn, dtype=torch.float32, device="cuda")
    used = C.c_int()
    N.check(N.lib().ms_k_gemm(bits, C.c_void_p(wp.data_ptr()), Nn, K, C.c_void_p(xp.data_ptr()), M, TM, splits,
                              C.c_void_p(out.data_ptr()), C.byref(used), stream()))
    torch.cuda.synchronize()
    s = used.value
    return out[: s * M * Nn].view(s, M, Nn).sum(0).cpu().numpy(), s


@pytest.mark.parametrize("Nn,K,M,TM,splits", [
    (128, 128, 1, 16, 1), (256, 256, 4, 16, 0), (512, 768, 33, 48, 3), (1024, 4096, 64, 64, 0),
    (384, 1024, 300, 256, 1), (128, 128, 16, 16, 2),
    # >= 4 waves of tiles: whole tiles per CTA, round-robin through the grouped
    # raster (gemm.cu SegIter), including a partial last group of token tiles
    (512, 256, 2500, 256, 3), (5120, 128, 4096, 256, 0)])
def test_gemm_bf16(Nn, K, M, TM, splits):
    W = O.gen_weight(21, 1, Nn * K, 1 / np.sqrt(K)).reshape(Nn, K)
    X = O.gen_weight(21, 2, M * K, 1.0).reshape(M, K)
    got, _ = _run_gemm(16, W, X, TM, splits)
    ref = O.gemm_bf16(W, X)
    # fp32 tensor-core accumulation vs fp64: |err| <= 1e-5 * sum|w x| (K <= 4096)
    bound = 1e-5 * (np.abs(O.bf16_to_f32(X)) @ np.abs(O.bf16_to_f32(W)).T) + 1e-6
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)


@pytest.mark.parametrize("Nn,K,M,TM,splits", [
    (128, 128, 1, 16, 1), (256, 768, 4, 16, 0), (512, 1024, 64, 64, 0), (256, 256, 200, 208, 1),
    (512, 256, 2500, 256, 3), (768, 512, 100, 112, 5), (1024, 1024, 600, 256, 0),
    # Llama-2-7B decode shapes (o / down): two 128-row tiles per activation chunk
    (4096, 4096, 64, 64, 0), (4096, 11008, 64, 64, 0),
    # odd K-group counts with stream-K ranges crossing tiles, TM 128
    (1280, 1152, 48, 48, 7), (512, 512, 128, 128, 3), (1280, 640, 33, 48, 0), (640, 512, 64, 64, 3)])
def test_gemm_w4(Nn, K, M, TM, splits):
    _check_quant_gemm(4, Nn, K, M, TM, splits)


def _check_quant_gemm(bits, Nn, K, M, TM, splits):
    W = O.gen_weight(22, 1, Nn * K, 1 / np.sqrt(K)).reshape(Nn, K)
    X = O.gen_weight(22, 2, M * K, 1.0).reshape(M, K)
    got, _ = _run_gemm(bits, W, X, TM, splits)
    codes, _, s16 = O.quantize_groups(W, bits=bits)
    Wq = O.dequant_w4(codes, s16)  # bf16(code * scale), every level
    ref = O.gemm_bf16(Wq, X)
    bound = 1e-5 * (np.abs(O.bf16_to_f32(X)) @ np.abs(O.bf16_to_f32(Wq)).T) + 1e-6
    assert np.all(np.abs(got - ref) <= bound), np.max(np.abs(got - ref) / bound)


@pytest.mark.parametrize("bits", [8, 3])
@pytest.mark.parametrize("Nn,K,M,TM,splits", [
    (128, 128, 1, 16, 1), (512, 1024, 64, 64, 0), (768, 512, 100, 112, 5), (1280, 1152, 48, 48, 7),
    (512, 256, 2500, 256, 3), (1024, 1024, 600, 256, 0),
    # Llama-2-7B decode shapes (o / down)
    (4096, 4096, 64, 64, 0), (4096, 11008, 64, 64, 0)])
def test_gemm_q8_q3(bits, Nn, K, M, TM, splits):
    """Q8 (byte codes, fp32 magic conversion) and Q3 (4-bit containers) through
    the same tcgen05 kernel family, same bf16(code * scale) contract."""
    _check_quant_gemm(bits, Nn, K, M, TM, splits)


@pytest.mark.parametrize("H,KVH,hd,ctxs,splits", [
    (4, 2, 64, [1, 5, 16, 17, 100], 1),
    (8, 8, 128, [1, 33, 250], 1),
    (32, 8, 128, [2048, 7, 300], 4),
    (8, 1, 128, [64, 129], 2),
    # up to 16 split-KV slices (runtime.cu kAttnMaxSplits) over long and 1-token rows
    (4, 2, 64, [1, 5, 16, 17, 100], 2),
    (32, 8, 128, [2048, 7, 300, 1, 4100], 16),
    (32, 32, 128, [2048] * 9, 8),
    (32, 32, 128, [4100], 16),
    # MHA hd 128: warp-per-block consumer, long rows (many ring wraps)
    (32, 32, 128, [2048, 1, 1500, 17, 4096], 1),
    (8, 1, 128, [64, 129, 16, 17], 3),
    # persistent GQA: > 32 rows (prefix scan over several rows per lane), items
    # cut across CTAs next to 1-block items, and the 16-piece cap
    (32, 8, 128, [2048] * 3 + [1] * 40 + [513, 31, 16, 17], 1),
    (16, 4, 128, [int(x) for x in np.random.default_rng(5).integers(1, 1200, 70)], 1),
    (32, 8, 128, [3000], 1)])
def test_paged_attention(H, KVH, hd, ctxs, splits):
    N = _native()
    L, layer = 3, 1
    rows = len(ctxs)
    page_bytes = 16 * L * KVH * 2 * hd * 2
    max_blocks = max((c + 15) // 16 for c in ctxs)
    n_pages = rows * max_blocks + 5
    rng = np.random.default_rng(0)
    arena = O.f32_to_bf16(rng.uniform(-1, 1, n_pages * page_bytes // 2).astype(np.float32))
    perm = rng.permutation(n_pages).astype(np.int32)  # scattered pages
    pages = perm[: rows * max_blocks].reshape(rows, max_blocks)
    q = rng.uniform(-1, 1, (rows, H, hd)).astype(np.float32)
    d_arena = dev_u16(arena)
    d_q = torch.from_numpy(q).cuda()
    d_pages = torch.from_numpy(pages.copy()).cuda()
    d_ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    out = torch.empty(rows * H * hd, dtype=torch.int16, device="cuda")
    ws = torch.empty(splits * rows * H * (hd + 2) + 16, dtype=torch.float32, device="cuda")
    N.check(N.lib().ms_k_attn_decode(C.c_void_p(d_q.data_ptr()), C.c_void_p(d_arena.data_ptr()), page_bytes, L,
                                     layer, H, KVH, hd, C.c_void_p(d_pages.data_ptr()), max_blocks,
                                     C.c_void_p(d_ctx.data_ptr()), rows, splits, C.c_void_p(ws.data_ptr()),
                                     C.c_void_p(out.data_ptr()), stream()))
    torch.cuda.synchronize()
    got = O.bf16_to_f32(to_np_u16(out)).reshape(rows, H * hd)
    head_elems = 16 * hd
    for r, ctx in enumerate(ctxs):
        k = np.empty((ctx, KVH, hd), np.uint16)
        v = np.empty((ctx, KVH, hd), np.uint16)
        for t in range(ctx):
            base = pages[r, t // 16] * (page_bytes // 2) + layer * KVH * 2 * head_elems
            for kh in range(KVH):
                off = base + kh * 2 * head_elems + (t % 16) * hd
                k[t, kh] = arena[off: off + hd]
                v[t, kh] = arena[off + head_elems: off + head_elems + hd]
        _, ref32 = O.attention(q[r].reshape(-1), k, v, H, KVH, hd)
        # bf16 output rounding (2^-8 relative) + fp32 softmax/accumulation
        np.testing.assert_allclose(got[r], ref32, rtol=1e-2, atol=2e-3)


@pytest.mark.parametrize("H,KVH,hd,n,qscale", [(4, 2, 64, 1, 1.0), (4, 2, 64, 77, 1.0), (8, 8, 128, 130, 1.0),
                                               (32, 8, 128, 300, 1.0), (8, 1, 128, 64, 1.0),
                                               (4, 4, 128, 700, 1.0), (4, 2, 128, 640, 1.0),
                                               (4, 4, 128, 555, 40.0), (2, 2, 128, 1030, 12.0)])
def test_prefill_attention(H, KVH, hd, n, qscale):
    """Causal prefill attention over paged KV vs the oracle, query by query.
    qscale > 1 spreads the scores over many powers of two, so the running
    max moves mid-sequence (the tcgen05 kernel's lazy O rescale)."""
    N = _native()
    L, layer = 2, 1
    page_bytes = 16 * L * KVH * 2 * hd * 2
    nb = (n + 15) // 16
    n_pages = nb + 3
    rng = np.random.default_rng(5)
    arena = O.f32_to_bf16(rng.uniform(-1, 1, n_pages * page_bytes // 2).astype(np.float32))
    pages = rng.permutation(n_pages).astype(np.int32)[:nb]
    q = (rng.uniform(-1, 1, (n, H, hd)) * qscale).astype(np.float32)
    if qscale > 1:  # rising score scale along the sequence: later keys/queries dominate
        q *= np.linspace(0.2, 1.0, n, dtype=np.float32)[:, None, None]
    d_arena = dev_u16(arena)
    d_q = torch.from_numpy(q).cuda()
    d_pages = torch.from_numpy(pages.copy()).cuda()
    out = torch.empty(n * H * hd, dtype=torch.int16, device="cuda")
    N.check(N.lib().ms_k_attn_prefill(C.c_void_p(d_q.data_ptr()), C.c_void_p(d_arena.data_ptr()), page_bytes, L,
                                      layer, H, KVH, hd, C.c_void_p(d_pages.data_ptr()), n,
                                      C.c_void_p(out.data_ptr()), stream()))
    torch.cuda.synchronize()
    got = O.bf16_to_f32(to_np_u16(out)).reshape(n, H * hd)
    head_elems = 16 * hd
    k = np.empty((n, KVH, hd), np.uint16)
    v = np.empty((n, KVH, hd), np.uint16)
    for t in range(n):
        base = pages[t // 16] * (page_bytes // 2) + layer * KVH * 2 * head_elems
        for kh in range(KVH):
            off = base + kh * 2 * head_elems + (t % 16) * hd
            k[t, kh] = arena[off: off + hd]
            v[t, kh] = arena[off + head_elems: off + head_elems + hd]
    for qi in sorted({0, n // 3, n // 2, n - 1, min(n - 1, 127), min(n - 1, 128), min(n - 1, 255), n - 2 if n > 1 else 0}):
        _, ref32 = O.attention(q[qi].reshape(-1), k[: qi + 1], v[: qi + 1], H, KVH, hd)
        # P is rounded to bf16 for the PV MMA (scores keep fp32 accuracy via the q hi/lo split)
        np.testing.assert_allclose(got[qi], ref32, rtol=2e-2, atol=4e-3)
