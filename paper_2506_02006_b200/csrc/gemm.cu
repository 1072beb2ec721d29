// gemm.cu -- the decoder linear layers on 5th-gen tensor cores (tcgen05).
//
// P[slot][m][n] = sum_{k in segment} W[n][k] * X[m][k] for one weight matrix W
// [N x K] (BF16, or g128-quantised Q8 / Q4 / Q3 codes dequantised in the
// staging path) and a token
// block X [M x K] (BF16), fp32 partials.  "Swap-AB": the weight rows are the
// UMMA M=128 side and the tokens the UMMA N side (16..256, runtime), so a
// decode batch of 64 is one N=64 instruction and a prefill is N=256 tiles --
// one kernel for decode (HBM-bound) and prefill (tensor-bound).
//
// Replaces the priced stand-ins `decode_ms_per_layer[tag]` (reference
// proj/src/sim_config.cpp:23-27) and `tokens * prefill_ms_per_token`
// (proj/src/engine.cpp:477-478); the per-layer precision comes from the layer
// table snapshot taken at step launch (engine.cpp:523-525).
//
// Persistent, stream-K balanced: one CTA per SM walks a contiguous range of
// the global (tile, k-step) sequence, so every SM streams the same number of
// weight bytes whatever the matrix shape.  A tile split between CTAs leaves
// one fp32 partial slot per CTA segment; the consuming row kernels sum the
// slots in slot order (deterministic, see PartSpec in kernels.h).  The
// partials of a decode step stay in L2.
//
// Data movement: every operand chunk is ONE contiguous 1-D bulk async copy
// (cp.async.bulk -> SASS UBLKCP), because both operands are pre-packed into
// the UMMA canonical K-major no-swizzle image:
//   weight chunk (n_tile, kb64)  = 16 KB  [row_group 16][k_chunk 8][row 8][8 bf16]
//   W4 chunk (n_tile, g128)      = 8448 B [j 4][row 128][16 B codes] + 128 bf16 scales
//                                  (Q4 and Q3 codes, 4-bit containers)
//   W8 chunk (n_tile, g128)      = 16640 B [j 8][row 128][16 B codes] + 128 bf16 scales
//   activation chunk (m_tile,kb) = TM*128 B, same core-matrix order.
// Weight chunks are found through the variant image's page table, so a layer
// image may live in any free pages of the KV/weight arena.
//
// Warp roles (mbarrier pipelines, no __syncthreads in the main loop):
//   warp 0 lane 0    producer: bulk copies into a `stages`-deep smem ring (W4: raw
//                    int4 chunks into their own deeper ring; B is fetched by the
//                    first dequantiser thread once the MMA released the stage)
//   warp 1 lane 0    UMMA issuer: tcgen05.mma kind::f16 M=128 N=TM K=16 into one
//                    of two TMEM accumulators (double buffered across segments)
//   warps 2..5       epilogue: tcgen05.ld -> fp32 partials, overlapping the next
//                    segment's loads and MMAs
//   warps 6..13 (W4) dequantisers: int4 -> bf16(code*scale) via the 0x4300 magic
//                    (exact), st.shared in the canonical layout, proxy fence.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm_common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ms {

// (chunk sizes, ChunkCursor, SegIter, nib_magic: gemm_common.cuh)

// Epilogue of one accumulator (128 weight rows x TM tokens, this warp's 32
// lanes at TMEM address d): fp32 partials out[m][n], or -- fused SiLU
// (GemmEpi) -- bf16(silu(gate) * up) into the packed activation image: lanes
// 2i / 2i+1 hold gate / up of FFN column j = 64 n_tile + (row >> 1)
// (interleaved storage, gate_col); per token pair the even lane computes token
// 2t and the odd lane token 2t + 1.
__device__ __forceinline__ void epilogue_tile(uint32_t d, int quad, int lane, int n_tile, int m_tile, int M, int N,
                                              int TM, float* __restrict__ o, const GemmEpi& epi) {
  if (epi.silu_out) {
    const int j = n_tile * 64 + ((quad * 32 + lane) >> 1);
    const bool odd = lane & 1;
    const size_t col = act_col_off(j, epi.TMo);
    for (int c0 = 0; c0 < TM; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(d + (uint32_t)c0, v);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float ve = __uint_as_float(v[2 * t]), vo = __uint_as_float(v[2 * t + 1]);
        const float mine = odd ? vo : ve, send = odd ? ve : vo;
        const float other = __shfl_xor_sync(0xffffffffu, send, 1);
        const float g = odd ? other : mine, up = odd ? mine : other;
        const int m = m_tile * TM + c0 + 2 * t + (odd ? 1 : 0);
        if (m < M) epi.silu_out[act_row_off(m, epi.ffn, epi.TMo) + col] = f2bf(silu_f(g) * up);
      }
    }
    return;
  }
  const int n = n_tile * 128 + quad * 32 + lane;
  for (int c0 = 0; c0 < TM; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(d + (uint32_t)c0, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int m = m_tile * TM + c0 + j;
      if (m < M) o[(size_t)m * N + n] = __uint_as_float(v[j]);
    }
  }
}
__global__ void __launch_bounds__(192, 1)
    gemm_kernel(GemmWeights W, const uint16_t* __restrict__ X, int M, int TM, GemmPlanDev plan,
                float* __restrict__ out, int stages, GemmEpi epi) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = W.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int nk = plan.nk;

  const uint32_t b_bytes = (uint32_t)TM * 128u;  // one 64-wide activation chunk
  const uint32_t a_bytes = 16384u;
  const uint32_t stage_bytes = a_bytes + b_bytes;  // A + B ring stage
  const uint32_t tm_cols = TM <= 32 ? 32u : TM <= 64 ? 64u : TM <= 128 ? 128u : 256u;

  uint8_t* sbase = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(sbase + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = full + 2 * stages;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  auto sA = [&](int s) { return sbase + (size_t)s * stage_bytes; };
  auto sB = [&](int s) { return sbase + (size_t)s * stage_bytes + a_bytes; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  // Producer (thread 0, which initialised the barriers): weights do not
  // depend on the previous kernel, so the first ring of weight chunks is
  // issued before the TMEM allocation / CTA barrier and the grid dependency.
  uint32_t npre = 0;
  ChunkCursor cur(W, kBf16ChunkBytes);
  if (threadIdx.x == 0) {
    SegIter pre(plan, cta);
    int t, k0, k1;
    while (npre < (uint32_t)stages && pre.next(t, k0, k1)) {
      const int n_tile = t % plan.n_tiles;
      cur.seek(W.first_chunk + (int64_t)n_tile * nk + k0);
      for (int k = k0; k < k1 && npre < (uint32_t)stages; ++k, ++npre, cur.advance()) {
        mbar_expect_tx(&full[npre], a_bytes + b_bytes);
        bulk_g2s(sA(npre), cur.get(), a_bytes, &full[npre]);
      }
    }
  }
  if (warp == 1) tmem_alloc_dyn(tmem_slot, 2 * tm_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t kb_per_mtile = W.K / 64;
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // the whole warp walks the ring and waits on it; lane 0 issues the copies
    // (a lone spinning lane was measured slower in the attention producers)
    npre = __shfl_sync(0xffffffffu, npre, 0);
    pdl_wait();
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t it = 0;
    while (seg.next(t, k0, k1)) {
      const int n_tile = t % plan.n_tiles, m_tile = t / plan.n_tiles;
      const uint8_t* xb = reinterpret_cast<const uint8_t*>(X) + (size_t)m_tile * kb_per_mtile * b_bytes;
      cur.seek(W.first_chunk + (int64_t)n_tile * nk + k0);
      for (int k = k0; k < k1; ++k, ++it, cur.advance()) {
        if (it < npre) {  // weight chunk already in flight: only the activations remain
          if (lane == 0) bulk_g2s(sB(it), xb + (size_t)k * b_bytes, b_bytes, &full[it]);
          continue;
        }
        const int s = it % stages;
        if (it >= (uint32_t)stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&full[s], a_bytes + b_bytes);
          bulk_g2s(sA(s), cur.get(), a_bytes, &full[s]);
          bulk_g2s(sB(s), xb + (size_t)k * b_bytes, b_bytes, &full[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    // whole warp, warp-uniform control; one elected lane issues
    const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)TM);
    const uint64_t dA0 = umma_desc(smem_u32(sA(0)), 128u, 1024u);
    const uint64_t dB0 = umma_desc(smem_u32(sB(0)), 128u, 1024u);
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t u = 0, s = 0, ph = 0;
    while (seg.next(t, k0, k1)) {
      const uint32_t acc = u & 1, use = u >> 1;
      if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * tm_cols;
      for (int k = k0; k < k1; ++k) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t da = desc_add(dA0, s * stage_bytes), db = desc_add(dB0, s * stage_bytes);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, desc_add(da, kk * 256u), desc_add(db, kk * 256u), idesc, (k != k0 || kk != 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == (uint32_t)stages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      ++u;
    }
  } else {
    // ------------------------------------------------------------- epilogue
    pdl_wait();
    const int quad = warp & 3;
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t u = 0;
    while (seg.next(t, k0, k1)) {
      const uint32_t acc = u & 1, use = u >> 1;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const int n_tile = t % plan.n_tiles, m_tile = t / plan.n_tiles;
      const int slot = plan.aligned ? 0 : cta - plan_cta_of(plan, (int64_t)t * nk);
      float* o = out + (size_t)slot * M * N;
      const uint32_t d = tmem_base + acc * tm_cols + ((uint32_t)(quad * 32) << 16);
      epilogue_tile(d, quad, lane, n_tile, m_tile, M, N, TM, o, epi);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      ++u;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, 2 * tm_cols);
}

// MS_GEMM_DEBUG (experiments only): bit0 skip activation loads, bit1 skip MMAs,
// bit3 CTA-0 timeline, bit4 producer stamps, bit5 one raw-chunk producer, bit6 per-CTA start/end,
// bit2 (W4 TMEM) skip the dequant ALU work and TMEM stores, bits 16..19 (W4) pre-issued raw units.
static int gemm_debug() {
  static const int v = [] {
    const char* e = std::getenv("MS_GEMM_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// --------------------------------------------------------------------------
// W4A16 g128: dequantise straight into TENSOR MEMORY and issue the A-from-TMEM
// form of tcgen05.mma, so the dequantised operand never touches shared memory
// (shared memory only carries the raw int4 chunks and the activations).
//   warp 0 lane 0   producer: raw int4 chunk ring (weights: no grid dependency)
//   warp 1 lane 0   UMMA issuer: tcgen05.mma [d], [a_tmem], b_desc  (M=128, N=TM)
//   warps 2..5      epilogue (TMEM accumulators -> fp32 partials)
//   warp 6 lane 0   activation (B) ring, after the grid dependency (own warp:
//                   two spin-waiting roles in one warp serialise each other)
//   warp 7 lane 0   second raw-chunk producer: warps 0 and 7 issue alternate
//                   units (one thread's issue rate -- cursor arithmetic and
//                   the bulk-copy instruction under the dequantisers' issue
//                   pressure, ~0.5 us per unit -- capped the weight stream)
//   warps 8..       kG dequantiser groups of 4 warps: warp w writes TMEM lanes
//                   32*(w%4).. (its rows); bf16(code*scale) via the 0x4300
//                   magic, tcgen05.st.32x32b.x32, wait::st, arrive.
// TMEM: [acc_bufs x TM columns of fp32 accumulators][astages x 64 columns of
// packed bf16 A (row = lane, 2 K-elements per 32-bit column)] -- 512 columns.
// kG dequantiser groups of 4 warps each keep kG chunks in flight, so the
// dequant ALU work (~4 instructions per bf16x2) is latency-hidden.
constexpr int kMaxAStages = 8;
constexpr int kDqWarp0 = 8;  // first dequantiser warp
constexpr int kProducers = 2;  // raw-chunk producer threads (warps 0 and 7)


// kGPS = 128-wide K groups per pipeline unit (1 or 2): two groups per unit
// halve the per-unit handshakes (mbarrier round trips, MMA commits, B copies)
// per weight byte.  kBits = code width of the chunk format: 4 (the 4- and
// 3-bit levels, nibble containers) or 8 (Q8, one byte per code; kGPS = 1).
//
// Q8 conversion, per pair of codes: byte_perm puts code + 128 into the
// mantissa of 2^23 (fp32 0x4B0000xx), one FADD removes 2^23 + 128 (exact),
// one FMUL by the fp32 scale (exact: 7 x 8 significant bits), and one
// cvt.rn.bf16x2.f32 rounds both products once: bf16(code * scale), the same
// contract as the 4-bit levels.
__device__ __forceinline__ uint32_t w8_pair(uint32_t word, int e, float s) {
  const float a = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7440u | (uint32_t)e)) - 8388736.0f;
  const float b = __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7440u | (uint32_t)(e + 1))) - 8388736.0f;
  __nv_bfloat162 v = __floats2bfloat162_rn(a * s, b * s);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int kG, int kGPS, int kBits>
__global__ void __launch_bounds__((kDqWarp0 + 4 * kG) * 32, 1)
    gemm_w4_tmem_kernel(GemmWeights W, const uint16_t* __restrict__ X, int M, int TM, GemmPlanDev plan,
                        float* __restrict__ out, int bstages, int rstages, int astages, int dbg, GemmEpi epi) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = W.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // (debug, dbg bits 8..15) rotate the CTA -> work map, to tell per-SM from per-range effects apart
  const int rot = (dbg >> 8) & 255;
  const int cta = rot ? (int)((blockIdx.x + (unsigned)rot) % gridDim.x) : (int)blockIdx.x;
  const int nk = plan.nk;
  const uint32_t b_bytes = (uint32_t)TM * 128u;  // one 64-wide activation chunk; a B stage holds 2 * kGPS
  static_assert(kBits == 4 || (kBits == 8 && kGPS == 1), "Q8 units hold one K group");
  constexpr uint32_t chunkB = kBits == 8 ? (uint32_t)kW8ChunkBytes : (uint32_t)kW4ChunkBytes;
  constexpr uint32_t code_bytes = kBits == 8 ? 16384u : 8192u;
  constexpr uint32_t raw_stage = kBits == 8 ? 16640u : (kGPS == 1 ? 8576u : 16896u);
  constexpr uint32_t raw_bytes = kGPS * chunkB;
  constexpr uint32_t a_cols = 64u * kGPS;  // packed bf16x2 TMEM columns of one A stage
  const int64_t gpr = W.K / 128;           // W4 chunks (K groups) per weight row tile
  const uint32_t tm_cols = TM <= 32 ? 32u : TM <= 64 ? 64u : TM <= 128 ? 128u : 256u;
  const uint32_t acc_bufs = TM <= 128 ? 2u : 1u;
  const uint32_t a_col0 = acc_bufs * tm_cols;
  // (debug, dbg bit3, kernel microbench only) CTA 0 timeline: [event][it] globaltimer
  uint64_t* tl = (dbg & 8) && blockIdx.x == 0 ? reinterpret_cast<uint64_t*>(out + (size_t)150 * M * N) : nullptr;
  auto stamp = [&](int ev, uint32_t i) {
    if (tl && i < 64) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      tl[ev * 64 + i] = t;
    }
  };

  uint64_t t0_dbg = 0;
  if (dbg & 64) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0_dbg));
  uint8_t* bbase = smem;
  uint8_t* rbase = smem + (size_t)bstages * 2 * kGPS * b_bytes;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(rbase + (size_t)rstages * raw_stage);
  uint64_t* bempty = bfull + bstages;
  uint64_t* rfull = bempty + bstages;
  uint64_t* rempty = rfull + rstages;
  uint64_t* afull = rempty + rstages;
  uint64_t* aempty = afull + kMaxAStages;
  uint64_t* tfull = aempty + kMaxAStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  auto sB = [&](int s) { return bbase + (size_t)s * 2 * kGPS * b_bytes; };
  auto sRaw = [&](int r) { return rbase + (size_t)r * raw_stage; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < bstages; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int r = 0; r < rstages; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], 4);  // the 4 warps of the dequantiser group that took the chunk
    }
    for (int a = 0; a < astages; ++a) {
      mbar_init(&afull[a], 4);
      mbar_init(&aempty[a], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  stamp(6, threadIdx.x == 0 ? 0 : 64);
  // Producer (thread 0, which initialised the barriers): the first ring of raw
  // int4 chunks is issued before the TMEM allocation and the CTA barrier.
  uint32_t npre = 0;
  ChunkCursor cur(W, (int)chunkB);
  // one unit's kGPS consecutive chunks into raw stage r (one copy when they
  // are contiguous in the same page); leaves the cursor at the next unit
  auto issue_unit = [&](int r, uint32_t dit) {
    const uint8_t* c0 = cur.get();
    cur.advance();
    const uint8_t* c1 = kGPS == 1 ? c0 : cur.get();
    if (kGPS != 1) cur.advance();
    if (dbg & 16) stamp(1, dit);
    mbar_expect_tx(&rfull[r], raw_bytes);
    if (dbg & 16) stamp(2, dit);
    if (kGPS == 1) {
      bulk_g2s(sRaw(r), c0, chunkB, &rfull[r]);
      return;
    }
    if (c1 == c0 + chunkB) {
      bulk_g2s(sRaw(r), c0, 2 * chunkB, &rfull[r]);
    } else {
      bulk_g2s(sRaw(r), c0, chunkB, &rfull[r]);
      bulk_g2s(sRaw(r) + chunkB, c1, chunkB, &rfull[r]);
    }
  };
  // decode tiles: only two units ahead of the pipeline start -- the first
  // chunks then arrive ~1 us sooner (every SM's initial burst queues in HBM
  // together) and the dequantisers start earlier; measured 2-5% per W4 decode
  // GEMM isolated, neutral in the step.  Long prefills (compute bound) fill
  // the whole ring.  Both producer threads need the count.
  // (debug, dbg bits 16..19: pre-issued unit count override, A/B only)
  const uint32_t pre_cap = ((dbg >> 16) & 15) ? (uint32_t)min(rstages, (dbg >> 16) & 15)
                         : TM <= 128 ? (uint32_t)min(rstages, 2) : (uint32_t)rstages;
  if (threadIdx.x == (kDqWarp0 - 1) * 32) {
    SegIter pre(plan, cta);
    int t, k0, k1;
    while (npre < pre_cap && pre.next(t, k0, k1)) npre += min((uint32_t)(k1 - k0), pre_cap - npre);
  }
  if (threadIdx.x == 0) {
    SegIter pre(plan, cta);
    int t, k0, k1;
    while (npre < pre_cap && pre.next(t, k0, k1)) {
      cur.seek(W.first_chunk + (int64_t)(t % plan.n_tiles) * gpr + (int64_t)k0 * kGPS);
      for (int k = k0; k < k1 && npre < pre_cap; ++k, ++npre) {
        issue_unit((int)npre, 64);
        stamp(0, npre);
      }
    }
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t kb_per_mtile = W.K / 64;
  pdl_trigger();

  // (debug, dbg bit5) a single producer thread, for A/B timing
  const uint32_t nprod = (dbg & 32) ? 1u : (uint32_t)kProducers;
  if (warp == 0 || warp == kDqWarp0 - 1) {
    // the whole warp waits on the ring, lane 0 issues and moves the cursor
    npre = __shfl_sync(0xffffffffu, npre, 0);
    if (warp == 0 || nprod > 1) {
      // ----------------------------------------------------------- producers
      // raw int4 chunks (independent of the activation ring, so the weight
      // stream runs `rstages` ahead; weights need no grid dependency).
      // Producer p issues the units it = p, p + kProducers, ... (after the
      // pre-issued ones); ring slot / phase kept incrementally.
      const uint32_t p = warp == 0 ? 0u : 1u;
      SegIter seg(plan, cta);
      int t, k0, k1;
      uint32_t it = 0;
      while (seg.next(t, k0, k1)) {
        const uint32_t end = it + (uint32_t)(k1 - k0);
        uint32_t u = it > npre ? it : npre;
        u += (p + nprod - u % nprod) % nprod;  // first unit of this producer
        if (u >= end) {
          it = end;
          continue;
        }
        const int n_tile = t % plan.n_tiles;
        cur.seek(W.first_chunk + (int64_t)n_tile * gpr + (int64_t)(k0 + (int)(u - it)) * kGPS);
        uint32_t r = u % (uint32_t)rstages, ph = ((u / (uint32_t)rstages) & 1) ^ 1;
        for (; u < end; u += nprod) {
          if ((dbg & 16) && lane == 0) stamp(5, u);
          mbar_wait(&rempty[r], ph);
          if (lane == 0) {
            if (dbg & 16) stamp(3, u);
            issue_unit((int)r, u);
            stamp(0, u);
            for (uint32_t i = 0; i < (nprod - 1) * kGPS; ++i) cur.advance();  // the other producer's units
          }
          __syncwarp();
          r += nprod;
          while (r >= (uint32_t)rstages) {
            r -= (uint32_t)rstages;
            ph ^= 1;
          }
        }
        it = end;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    // whole warp, warp-uniform control; one elected lane issues
    const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)TM);
    const uint64_t dB0 = umma_desc(smem_u32(sB(0)), 128u, 1024u);
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t it = 0, u = 0, s = 0, sph = 0, a = 0, aph = 0;
    while (seg.next(t, k0, k1)) {
      const uint32_t acc = acc_bufs == 2 ? (u & 1) : 0u;
      const uint32_t use = acc_bufs == 2 ? (u >> 1) : u;
      if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * tm_cols;
      for (int k = k0; k < k1; ++k, ++it) {
        mbar_wait(&bfull[s], sph);
        mbar_wait(&afull[a], aph);
        tc_fence_after();
        stamp(4, it);
        const uint64_t db = desc_add(dB0, s * 2u * kGPS * b_bytes);
        const uint32_t ta = tmem_base + a_col0 + a * a_cols;
        if (elect_one()) {
#pragma unroll
          for (int sub = 0; sub < 2 * kGPS; ++sub) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (!(dbg & 2))
                umma_bf16_ts(d, ta + sub * 32u + kk * 8u, desc_add(db, sub * b_bytes + kk * 256u), idesc,
                             (k != k0 || sub != 0 || kk != 0) ? 1u : 0u);
            }
          }
          umma_commit(&bempty[s]);
          umma_commit(&aempty[a]);
        }
        __syncwarp();
        stamp(7, it);
        if (++s == (uint32_t)bstages) {
          s = 0;
          sph ^= 1;
        }
        if (++a == (uint32_t)astages) {
          a = 0;
          aph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      ++u;
    }
  } else if (warp == 6) {
    // activation (B) chunks: own warp (a spin-wait here must not hold up the
    // weight producer), after the grid dependency; the whole warp waits on
    // the ring, lane 0 issues
    pdl_wait();
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t it = 0;
    uint32_t s = 0, ph = 1;
    while (seg.next(t, k0, k1)) {
      const int m_tile = t / plan.n_tiles;
      const uint8_t* xb = reinterpret_cast<const uint8_t*>(X) + (size_t)m_tile * kb_per_mtile * b_bytes;
      for (int k = k0; k < k1; ++k, ++it) {
        if (it >= (uint32_t)bstages) mbar_wait(&bempty[s], ph);
        if (lane == 0) {
          if (dbg & 1) {  // (debug) no activation traffic: complete the stage empty
            mbar_expect_tx(&bfull[s], 0);
          } else {
            mbar_expect_tx(&bfull[s], 2 * kGPS * b_bytes);
            bulk_g2s(sB(s), xb + (size_t)(2 * kGPS * k) * b_bytes, 2 * kGPS * b_bytes, &bfull[s]);
          }
          if (!(dbg & 16)) stamp(5, it);
        }
        __syncwarp();
        if (++s == (uint32_t)bstages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------- epilogue
    pdl_wait();
    const int quad = warp & 3;
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t u = 0;
    while (seg.next(t, k0, k1)) {
      const uint32_t acc = acc_bufs == 2 ? (u & 1) : 0u;
      const uint32_t use = acc_bufs == 2 ? (u >> 1) : u;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const int n_tile = t % plan.n_tiles, m_tile = t / plan.n_tiles;
      const int slot = plan.aligned ? 0 : cta - plan_cta_of(plan, (int64_t)t * nk);
      float* o = out + (size_t)slot * M * N;
      const uint32_t d = tmem_base + acc * tm_cols + ((uint32_t)(quad * 32) << 16);
      epilogue_tile(d, quad, lane, n_tile, m_tile, M, N, TM, o, epi);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      ++u;
    }
  } else {
    // ---------------------------------------------------------- dequantisers
    // kG groups of 4 warps; group g takes k-steps it = g, g + kG, ... (so kG
    // chunks are in flight); warp quadrant q owns TMEM lanes / weight rows
    // 32q..32q+31 and dequantises the whole 128-wide group of its row: 64
    // packed bf16x2 columns, two tcgen05.st.32x32b.x32.
    const int quad = warp & 3, grp = (warp - kDqWarp0) >> 2;
    const int row = quad * 32 + lane;
    const __nv_bfloat162 bias = __floats2bfloat162_rn(136.0f, 136.0f);
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16) + a_col0;
    SegIter seg(plan, cta);
    int t, k0, k1;
    uint32_t it = 0;
    // this group's units are it = grp, grp + kG, ...: ring slots and phases
    // advance by kG (< rstages, astages) per unit, no division in the loop
    uint32_t rs = (uint32_t)grp, rph = 0, a = (uint32_t)grp, aph = 0;
    auto adv = [&] {
      rs += kG;
      while (rs >= (uint32_t)rstages) {
        rs -= (uint32_t)rstages;
        rph ^= 1;
      }
      a += kG;
      if (a >= (uint32_t)astages) {  // kG <= astages (launch_q_groups)
        a -= (uint32_t)astages;
        aph ^= 1;
      }
    };
    while (seg.next(t, k0, k1)) {
      // first k-step of this segment owned by this group
      int k = k0 + (int)((grp - (int)(it % kG) + kG) % kG);
      it += (uint32_t)(k - k0);
      for (; k < k1; k += kG, it += kG) {
        mbar_wait(&rfull[rs], rph);
        if (lane == 0 && quad == 0 && !(dbg & 16)) stamp(1, it);
        const uint8_t* raw = sRaw(rs);
        constexpr int kQ = kBits == 8 ? 8 : 4;  // uint4 of codes per row per K group
        __nv_bfloat162 sc[kGPS];
        uint4 q[kGPS][kQ];
#pragma unroll
        for (int h = 0; h < kGPS; ++h) {
          const uint8_t* rh = raw + h * chunkB;
          sc[h].x = __ushort_as_bfloat16(*reinterpret_cast<const uint16_t*>(rh + code_bytes + 2 * row));
          sc[h].y = sc[h].x;
#pragma unroll
          for (int j = 0; j < kQ; ++j) q[h][j] = *reinterpret_cast<const uint4*>(rh + (j * 128 + row) * 16);
        }
        // raw chunk consumed (values are in registers): order these generic-proxy
        // reads before the producer's next async-proxy (bulk copy) write
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[rs]);
        if (it >= (uint32_t)astages) mbar_wait(&aempty[a], aph ^ 1);
        if (lane == 0 && quad == 0 && !(dbg & 16)) stamp(2, it);
        tc_fence_after();
        if (dbg & 4) {  // (debug) no dequant ALU / TMEM stores: hand the stage straight on
          __syncwarp();
          if (lane == 0) mbar_arrive(&afull[a]);
          adv();
          continue;
        }
#pragma unroll
        for (int h = 0; h < kGPS; ++h)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t o[32];
            if (kBits == 8) {
              const float s32 = __bfloat162float(sc[h].x);
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const uint4 qq = q[h][hh * 4 + jj];
                const uint32_t words[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                  o[jj * 8 + w * 2 + 0] = w8_pair(words[w], 0, s32);
                  o[jj * 8 + w * 2 + 1] = w8_pair(words[w], 2, s32);
                }
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < 2; ++jj) {
                const uint4 qq = q[h][hh * 2 + jj];
                const uint32_t words[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
                for (int w = 0; w < 4; ++w)
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const uint32_t x = nib_magic(words[w] >> (4 * i));
                    __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&x);
                    v = __hmul2(__hsub2(v, bias), sc[h]);  // exact code, then one rounding of code*scale
                    o[jj * 16 + w * 4 + i] = *reinterpret_cast<uint32_t*>(&v);
                  }
              }
            }
            tmem_st32(lane_base + (uint32_t)a * a_cols + (uint32_t)h * 64u + (uint32_t)hh * 32u, o);
          }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[a]);
        if (lane == 0 && quad == 0 && !(dbg & 16)) stamp(3, it);
        adv();
      }
      it -= (uint32_t)(k - k1);  // back to the segment end
    }
  }

  tc_fence_before();
  __syncthreads();
  stamp(6, threadIdx.x == 0 ? 1 : 64);
  if ((dbg & 64) && threadIdx.x == 0) {  // (debug) per-CTA start / end globaltimer after the CTA-0 timeline
    uint64_t* ce = reinterpret_cast<uint64_t*>(out + (size_t)150 * M * N) + 1024 + 2 * blockIdx.x;
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    ce[0] = (t0_dbg & 0xFFFFFFFFFFFFull) | ((uint64_t)smid << 48);  // start (low 48 bits) | SM id
    ce[1] = t;
  }
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

// Ring sizes of the quantised kernel: activation (B) stages, raw chunk
// stages (the rest of the shared-memory budget), TMEM A stages, dequantiser
// groups (*groups).  Parity waits are only sound while a barrier is at most
// one phase behind its waiter, which the sizes guarantee by construction:
//  - raw stages are even, so with the two producers issuing alternate units
//    each raw stage is always filled by the same producer (which issued the
//    stage's previous round itself before waiting on its release);
//  - raw stages >= groups + A stages: a group starts waiting for unit u
//    only after finishing u - groups, which needed the MMA of
//    u - groups - astages, so every unit <= u - rstages has landed.
static int pick_q_stages(int TM, int gps, int bits, int* rstages, int* astages, int* groups, size_t* smem_out) {
  const size_t budget = 215 * 1024;
  const size_t bst = (size_t)TM * 128 * 2 * gps;
  const size_t raw_stage = bits == 8 ? 16640 : (gps == 1 ? 8576 : 16896);
  const int bs = gps == 1 ? (TM <= 64 ? (bits == 8 ? 4 : 6) : (TM <= 128 ? 4 : 2)) : (TM <= 64 ? 3 : (TM <= 128 ? 2 : 1));
  int rs = (int)((budget - bs * bst) / raw_stage);
  if (rs > 16) rs = 16;
  rs &= ~1;
  const int tm_cols = TM <= 32 ? 32 : TM <= 64 ? 64 : TM <= 128 ? 128 : 256;
  const int acc = (TM <= 128 ? 2 : 1) * tm_cols;
  const int as_max = std::min(kMaxAStages, (512 - acc) / (64 * gps));
  // three groups when three A stages and six raw stages fit, else two
  const int g = as_max >= 3 && rs >= 6 ? 3 : 2;
  *groups = g;
  *rstages = rs;
  *astages = std::min(as_max, rs - g);
  *smem_out = bs * bst + (size_t)rs * raw_stage + (2 * bs + 2 * rs + 2 * kMaxAStages + 4) * 8 + 64;
  return *astages >= g && rs >= 2 * g ? bs : -1;
}

void gemm_inline_pages(GemmWeights& w, int wkind, const uint64_t* host_pages) {
  const int64_t chunks = (int64_t)(w.N / 128) * (w.K / chunk_k(wkind));
  const int64_t p0 = w.first_chunk / w.chunks_per_page;
  const int64_t p1 = (w.first_chunk + chunks - 1) / w.chunks_per_page;
  w.n_inl = 0;
  if (p1 - p0 + 1 > kGemmInlinePages) return;
  w.inl_p0 = (int)p0;
  for (int64_t p = p0; p <= p1; ++p) w.inl[p - p0] = host_pages[p];
  w.n_inl = (int)(p1 - p0 + 1);
}

GemmPlanDev gemm_plan(int N, int K, int M, int TM, int wkind, int num_sms, size_t part_elems) {
  GemmPlanDev p{};
  p.n_tiles = N / 128;
  p.TM = TM;
  // int4: two 128-wide K groups per pipeline unit when K allows
  // (one group per unit for token tiles > 128: the activation stage of a
  // two-group unit would leave a single B stage, serialising loads and MMAs);
  // int8: one K group per unit (a group's raw chunk is already 16.6 KB)
  p.nk = wkind == 16 ? K / 64 : wkind == 8 ? K / 128 : K / (K % 256 == 0 && TM <= 128 ? 256 : 128);
  p.tiles = p.n_tiles * ((M + TM - 1) / TM);
  p.T = (int64_t)p.tiles * p.nk;
  p.C = (int)std::min<int64_t>(num_sms, p.T);
  p.aligned = 0;
  // slots needed by the stream-K partition
  int max_slots = 1;
  const bool fits32 = (p.T + 1) * (int64_t)p.C < ((int64_t)1 << 31);
  if (fits32)
    for (int t = 0; t < p.tiles; ++t) max_slots = std::max(max_slots, plan_count(p, t));
  // whole tiles per CTA when stream-K cannot hold its partial slots, or when
  // there are >= 4 waves of tiles: the partial last wave then costs little,
  // and the round-robin raster (SegIter) keeps the tiles in flight in L2,
  // where contiguous stream-K ranges spread them over the whole matrix
  if (!fits32 || (size_t)max_slots * M * N > part_elems || p.tiles >= 4 * num_sms) {
    static const int raster = [] {
      const char* e = std::getenv("MS_GEMM_RASTER");
      const int v = e ? std::atoi(e) : 8;
      return v < 1 ? 1 : v;
    }();
    p.aligned = raster;
    p.C = std::min(num_sms, p.tiles);
    max_slots = 1;
  }
  p.slots = max_slots;
  return p;
}

template <int kG, int kGPS, int kBits>
static cudaError_t launch_q_tmem(const GemmWeights& w, const uint16_t* x, int M, int TM, const GemmPlanDev& plan,
                                 float* out, cudaStream_t stream, const GemmEpi& epi) {
  int rs = 0, as = 0, g = 0;
  size_t sm = 0;
  const int bs = pick_q_stages(TM, kGPS, kBits, &rs, &as, &g, &sm);
  if (bs < 0 || g != kG) return cudaErrorInvalidConfiguration;
  static std::atomic<uint64_t> attr{0};
  max_smem_once(gemm_w4_tmem_kernel<kG, kGPS, kBits>, 227 * 1024, attr);
  return launch_pdl(gemm_w4_tmem_kernel<kG, kGPS, kBits>, dim3(plan.C), dim3((kDqWarp0 + 4 * kG) * 32), sm, stream, w, x, M,
                    TM, plan, out, bs, rs, as, gemm_debug(), epi);
}

// Three dequantiser groups (fastest in the 7B step), two when TMEM or the raw
// ring holds fewer stages (pick_q_stages).
template <int kGPS, int kBits>
static cudaError_t launch_q_groups(const GemmWeights& w, const uint16_t* x, int M, int TM, const GemmPlanDev& plan,
                                   float* out, cudaStream_t stream, const GemmEpi& epi) {
  int rs = 0, as = 0, g = 0;
  size_t sm = 0;
  pick_q_stages(TM, kGPS, kBits, &rs, &as, &g, &sm);
  if (g == 3) return launch_q_tmem<3, kGPS, kBits>(w, x, M, TM, plan, out, stream, epi);
  return launch_q_tmem<2, kGPS, kBits>(w, x, M, TM, plan, out, stream, epi);
}

cudaError_t gemm_launch(const GemmWeights& w, int wkind, const uint16_t* x, int M, int TM, const GemmPlanDev& plan,
                        float* out, cudaStream_t stream, const GemmEpi& epi) {
  // the fused SiLU epilogue needs whole tiles (one slot)
  if (epi.silu_out && !plan.aligned) return cudaErrorInvalidValue;
  if (wkind == 8) return launch_q_groups<1, 8>(w, x, M, TM, plan, out, stream, epi);
  if (wkind == 4) {
    // the plan fixed the unit: K / nk = 256 -> two K groups per pipeline unit
    if (w.K / plan.nk == 256) return launch_q_groups<2, 4>(w, x, M, TM, plan, out, stream, epi);
    return launch_q_groups<1, 4>(w, x, M, TM, plan, out, stream, epi);
  }
  if (wkind != 16) return cudaErrorInvalidValue;
  static const int max_st = [] {  // (experiments) ring depth cap
    const char* e = std::getenv("MS_GEMM_STAGES");
    return e ? std::atoi(e) : 8;
  }();
  const size_t stage = (size_t)16384 + (size_t)TM * 128;
  int st = (int)((size_t)(215 * 1024) / stage);
  st = std::max(2, std::min(st, max_st));
  const size_t smem = st * stage + (2 * st + 4) * 8 + 64;
  static std::atomic<uint64_t> attr{0};
  max_smem_once(gemm_kernel, 227 * 1024, attr);
  return launch_pdl(gemm_kernel, dim3(plan.C), dim3(192), smem, stream, w, x, M, TM, plan, out, st, epi);
}

}  // namespace ms
