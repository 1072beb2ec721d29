// layer.cu -- the fused decode layer: everything of one decoder layer after
// its attention, as ONE persistent kernel (one CTA per SM):
//
//   O GEMM -> [grid barrier] -> residual + RMSNorm(norm2) -> [barrier] ->
//   gate_up GEMM -> [barrier] -> SiLU(g)*u -> [barrier] -> down GEMM ->
//   [barrier] -> residual + RMSNorm(next layer's norm1 | final norm)
//
// Replaces, for a decode step, the six launches of the unfused path (three
// stream-K GEMMs + residual_norm / silu_mul / residual_norm row kernels) of the
// priced stand-in `decode_ms_per_layer[tag]` (reference
// proj/src/sim_config.cpp:23-27).  Same arithmetic as those kernels (fp32
// partial slots summed in slot order, bf16 rounding points of DESIGN.md 4).
//
// Why: at decode sizes a layer's three matrices are 4-30 us of HBM time each
// (7B: 34 / 180 / 90 MB BF16, 8 / 45 / 23 MB W4A16) and every separate launch
// paid a ramp (first weight bytes ~2-3 us after launch, uneven DRAM service
// across SMs) and a drain.  Here the weight producer of every CTA streams the
// weight chunks of the three GEMMs back to back -- it never waits for a grid
// barrier, only for ring slots -- so the next GEMM's weights are already in
// shared memory while the grid barrier and the row pass of the previous one
// run.  Only the activation (B) loads and the partial-slot writes wait for the
// barriers.
//
// Warp roles (BF16 | W4A16 g128):
//   warp 0 lane 0   weight producer: BF16 16 KB chunks into the A half of the
//                   (A, B) ring | raw int4 chunks into the raw ring
//   warp 1          UMMA issuer (one elected lane, warp-uniform control)
//   warps 2..5      epilogue (TMEM accumulators -> fp32 partial slots), then
//                   the row phases, grid-barrier arrivals
//   warp 6          activation (B) producer: waits for the phase's grid barrier,
//                   then bulk-copies the packed activations
//   warps 7..       (W4) kG groups of 4 dequantiser warps: bf16(code * scale)
//                   straight into tensor memory (the MMA reads A from TMEM)
//
// Grid barrier: one arrival counter per CTA (`bar[cta]`, only CTA `cta` writes
// it), monotonically increasing across launches; every launch makes the same
// number of arrivals per CTA, so at kernel start all counters are equal (the
// previous fused layer completed, ordered by the programmatic-dependent-launch
// chain), and barrier k of this launch is "every counter >= base + k".
// Nothing launch-specific is baked into the parameters: CUDA-graph replays
// behave like the captured launch.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm_common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kPhases = 3;          // O, gate_up, down
constexpr int kEpiThreads = 128;    // warps 2..5
constexpr int kLayerMaxAStages = 8;
constexpr int kLayerBarStride = 32;  // words between two CTAs' barrier counters (128 B)

// counters one 128-B line apart (kLayerBarStride words): the arrivals and the
// pollers' reads spread over many L2 slices instead of hammering one line
__device__ __forceinline__ void gbar_arrive(uint32_t* bar, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + (size_t)blockIdx.x * kLayerBarStride), "r"(v)
               : "memory");
}
// whole warp: until every CTA's counter reached v
__device__ __forceinline__ void gbar_wait(const uint32_t* bar, uint32_t v) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    bool ok = true;
    for (int i = lane; i < (int)gridDim.x; i += 32) {
      uint32_t x;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(bar + (size_t)i * kLayerBarStride) : "memory");
      ok = ok && (int)(x - v) >= 0;
    }
    if (__all_sync(0xffffffffu, ok)) break;
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  __syncwarp();
}
__device__ __forceinline__ uint32_t gbar_base(const uint32_t* bar) {
  uint32_t x;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(bar + (size_t)blockIdx.x * kLayerBarStride)
               : "memory");
  return x;
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// (debug) timeline stamp: event e of phase p of this CTA
__device__ __forceinline__ void tl_stamp(unsigned long long* tl, int e, int p) {
  if (!tl) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  tl[((size_t)blockIdx.x * 8 + e) * 3 + p] = t;
}

// the GEMM output at (m, col) of a phase: sum of its partial slots in slot order
__device__ __forceinline__ float4 slots4(const GemmPlanDev& plan, const float* part, int M, int N, int m, int col) {
  const float4* p = reinterpret_cast<const float4*>(part + (size_t)m * N + col);
  const size_t stride4 = (size_t)M * N / 4;
  const int n = part_slots(plan, m, col);
  float4 v[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) v[s] = s < n ? __ldcg(p + s * stride4) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < 6; ++s)
    if (s < n) {
      acc.x += v[s].x;
      acc.y += v[s].y;
      acc.z += v[s].z;
      acc.w += v[s].w;
    }
  for (int s = 6; s < n; ++s) {
    const float4 a = __ldcg(p + s * stride4);
    acc.x += a.x;
    acc.y += a.y;
    acc.z += a.z;
    acc.w += a.w;
  }
  return acc;
}

// residual add (h += GEMM output) + RMSNorm + pack, rows cta, cta+G, ... (epilogue
// warps).  Two passes over the row (the second re-reads the just-written h from
// L2) keep the register footprint small next to the dequantiser warps.
__device__ void rows_residual_norm(const DecodeLayerArgs& a, const GemmPlanDev& plan, const uint16_t* __restrict__ w,
                                   int tm_out, int row_begin, float* red) {
  const int t = threadIdx.x - 64;
  const int d = a.d, d4 = d >> 2;
  for (int m = blockIdx.x; m < a.M; m += gridDim.x) {
    float4* hr = reinterpret_cast<float4*>(a.h + (size_t)m * d);
    float ss = 0.f;
#pragma unroll 4
    for (int i4 = t; i4 < d4; i4 += kEpiThreads) {
      float4 v = __ldcg(hr + i4);
      const float4 s = slots4(plan, a.part, a.M, d, m, i4 * 4);
      v.x += s.x;
      v.y += s.y;
      v.z += s.z;
      v.w += s.w;
      __stcg(hr + i4, v);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    if (m < row_begin) continue;  // (uniform across the epilogue warps)
    ss = warp_sum(ss);
    if ((t & 31) == 0) red[t >> 5] = ss;
    epi_sync();
    const float tot = red[0] + red[1] + red[2] + red[3];
    epi_sync();  // red reused by the next row
    const float r = 1.0f / sqrtf(tot / (float)d + a.eps);
    const uint2* w4 = reinterpret_cast<const uint2*>(w);
    uint16_t* xrow = a.x + act_row_off(m - row_begin, d, tm_out);
#pragma unroll 4
    for (int i4 = t; i4 < d4; i4 += kEpiThreads) {
      const float4 v = __ldcg(hr + i4);
      const uint2 wv = w4[i4];
      uint2 o;
      o.x = pack_bf2((v.x * r) * __uint_as_float(wv.x << 16), (v.y * r) * __uint_as_float(wv.x & 0xFFFF0000u));
      o.y = pack_bf2((v.z * r) * __uint_as_float(wv.y << 16), (v.w * r) * __uint_as_float(wv.y & 0xFFFF0000u));
      *reinterpret_cast<uint2*>(xrow + act_col_off(i4 * 4, tm_out)) = o;
    }
  }
}

// SiLU(gate) * up over all (row, column quad) pairs, spread over the grid;
// two pairs per thread in flight (all their partial-slot loads issued first)
__device__ void rows_silu(const DecodeLayerArgs& a, const GemmPlanDev& plan) {
  const int t = threadIdx.x - 64;
  const int ffn = a.ffn, f4 = ffn >> 2, N = 2 * ffn;
  const int total = a.M * f4;
  const int stride = gridDim.x * kEpiThreads;
  auto silu = [](float g) { return __fdividef(g, 1.0f + __expf(-g)); };  // as silu_mul_kernel
  for (int idx = blockIdx.x * kEpiThreads + t; idx < total; idx += 2 * stride) {
    float4 g[2], u[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = idx + q * stride;
      if (i < total) {
        const int m = i / f4, j4 = i - m * f4;
        g[q] = slots4(plan, a.part, a.M, N, m, j4 * 4);
        u[q] = slots4(plan, a.part, a.M, N, m, ffn + j4 * 4);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = idx + q * stride;
      if (i < total) {
        const int m = i / f4, j4 = i - m * f4;
        uint2 o;
        o.x = pack_bf2(silu(g[q].x) * u[q].x, silu(g[q].y) * u[q].y);
        o.y = pack_bf2(silu(g[q].z) * u[q].z, silu(g[q].w) * u[q].w);
        *reinterpret_cast<uint2*>(a.x + act_row_off(m, ffn, a.TM) + act_col_off(j4 * 4, a.TM)) = o;
      }
    }
  }
}

}  // namespace

template <bool kW4, int kG>
__global__ void __launch_bounds__(kW4 ? (7 + 4 * kG) * 32 : 224, 1)
    decode_layer_kernel(const __grid_constant__ DecodeLayerArgs a, int stages, int rstages, int astages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int TM = a.TM;
  if (threadIdx.x == 0) tl_stamp(a.tl, 6, 0);
  const uint32_t b_bytes = (uint32_t)TM * 128u;  // one 64-wide activation chunk
  const uint32_t tm_cols = TM <= 32 ? 32u : TM <= 64 ? 64u : TM <= 128 ? 128u : 256u;
  // BF16: stage = A 16 KB + B (one 64-wide k-step); W4: B stage = 4 chunks (K = 256 per unit)
  constexpr uint32_t a_bytes = 16384u;
  constexpr uint32_t raw_stage = 16896u;                 // two 8448-B W4 chunks (one unit)
  constexpr uint32_t raw_bytes = 2u * (uint32_t)kW4ChunkBytes;
  constexpr uint32_t a_cols = 128u;                      // W4: TMEM columns of one dequantised A unit
  const uint32_t stage_bytes = kW4 ? 4u * b_bytes : a_bytes + b_bytes;
  const uint32_t acc_bufs = (kW4 && TM > 128) ? 1u : 2u;
  const uint32_t a_col0 = acc_bufs * tm_cols;

  uint8_t* sbase = smem;
  uint8_t* rbase = smem + (size_t)stages * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(rbase + (size_t)(kW4 ? rstages : 0) * raw_stage);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* rfull = tempty + 2;      // [rstages] (W4)
  uint64_t* rempty = rfull + rstages;
  uint64_t* afull = rempty + rstages;  // [kLayerMaxAStages] (W4)
  uint64_t* aempty = afull + kLayerMaxAStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + kLayerMaxAStages);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [4] row-reduction scratch
  uint32_t* s_base = tmem_slot + 8;                       // grid-barrier counter at launch
  uint64_t* bgo = reinterpret_cast<uint64_t*>(tmem_slot + 10);  // barrier 2p+2 passed -> activation producer
  auto sA = [&](uint32_t s) { return sbase + (size_t)s * stage_bytes; };
  auto sB = [&](uint32_t s) { return sbase + (size_t)s * stage_bytes + (kW4 ? 0u : a_bytes); };
  auto sRaw = [&](uint32_t r) { return rbase + (size_t)r * raw_stage; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    mbar_init(bgo, 1);
    if (kW4) {
      for (int r = 0; r < rstages; ++r) {
        mbar_init(&rfull[r], 1);
        mbar_init(&rempty[r], 4);
      }
      for (int i = 0; i < astages; ++i) {
        mbar_init(&afull[i], 4);
        mbar_init(&aempty[i], 1);
      }
    }
    fence_mbar_init();
  }

  // ---- weight producer, first ring issued before the TMEM allocation / CTA
  // barrier (weights never depend on the previous kernel)
  const uint32_t wring = kW4 ? (uint32_t)rstages : (uint32_t)stages;
  uint32_t npre = 0;
  auto issue_weight = [&](ChunkCursor& cur, uint32_t it) {
    if (kW4) {
      const uint32_t r = it % (uint32_t)rstages;
      mbar_expect_tx(&rfull[r], raw_bytes);
      const uint8_t* c0 = cur.get();
      cur.advance();
      const uint8_t* c1 = cur.get();
      cur.advance();
      if (c1 == c0 + kW4ChunkBytes) {
        bulk_g2s(sRaw(r), c0, 2 * kW4ChunkBytes, &rfull[r]);
      } else {
        bulk_g2s(sRaw(r), c0, kW4ChunkBytes, &rfull[r]);
        bulk_g2s(sRaw(r) + kW4ChunkBytes, c1, kW4ChunkBytes, &rfull[r]);
      }
    } else {
      const uint32_t s = it % (uint32_t)stages;
      mbar_expect_tx(&full[s], a_bytes + b_bytes);
      bulk_g2s(sA(s), cur.get(), a_bytes, &full[s]);
      cur.advance();
    }
  };
  // chunks per k-step unit along K: BF16 one 64-wide chunk, W4 two 128-wide groups
  auto unit_chunk = [&](const GemmWeights& w, int n_tile, int k) -> int64_t {
    return kW4 ? w.first_chunk + (int64_t)n_tile * (w.K / 128) + (int64_t)k * 2
               : w.first_chunk + (int64_t)n_tile * (w.K / 64) + k;
  };
  if (threadIdx.x == 0) {
    ChunkCursor cur(a.w[0], kW4 ? kW4ChunkBytes : kBf16ChunkBytes);
    SegIter pre(a.plan[0], cta);
    int t, k0, k1;
    while (npre < wring && cta < a.plan[0].C && pre.next(t, k0, k1)) {
      cur.seek(unit_chunk(a.w[0], t % a.plan[0].n_tiles, k0));
      for (int k = k0; k < k1 && npre < wring; ++k, ++npre) issue_weight(cur, npre);
    }
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------ weight producer
      uint32_t it = 0;
      for (int p = 0; p < kPhases; ++p) {
        const GemmWeights& w = a.w[p];
        const GemmPlanDev& plan = a.plan[p];
        if (cta >= plan.C) continue;
        ChunkCursor cur(w, kW4 ? kW4ChunkBytes : kBf16ChunkBytes);
        SegIter seg(plan, cta);
        int t, k0, k1;
        while (seg.next(t, k0, k1)) {
          const uint32_t n = (uint32_t)(k1 - k0);
          if (it + n <= npre) {  // whole segment pre-issued
            it += n;
            continue;
          }
          const int skip = it < npre ? (int)(npre - it) : 0;
          it += (uint32_t)skip;
          cur.seek(unit_chunk(w, t % plan.n_tiles, k0 + skip));
          if (skip == 0 && k0 < k1) tl_stamp(a.tl, 5, p);
          for (int k = k0 + skip; k < k1; ++k, ++it) {
            if (it >= wring) {
              const uint32_t s = it % wring;
              mbar_wait(kW4 ? &rempty[s] : &empty[s], ((it / wring) & 1) ^ 1);
            }
            issue_weight(cur, it);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- UMMA issuer
    const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)TM);
    const uint64_t dA0 = umma_desc(smem_u32(sA(0)), 128u, 1024u);
    const uint64_t dB0 = umma_desc(smem_u32(sB(0)), 128u, 1024u);
    uint32_t u = 0, s = 0, ph = 0, ai = 0, aph = 0;
    for (int p = 0; p < kPhases; ++p) {
      const GemmPlanDev& plan = a.plan[p];
      if (cta >= plan.C) continue;
      SegIter seg(plan, cta);
      int t, k0, k1;
      while (seg.next(t, k0, k1)) {
        const uint32_t acc = acc_bufs == 2 ? (u & 1) : 0u;
        const uint32_t use = acc_bufs == 2 ? (u >> 1) : u;
        if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * tm_cols;
        bool first = true;
        for (int k = k0; k < k1; ++k) {
          mbar_wait(&full[s], ph);
          if (kW4) mbar_wait(&afull[ai], aph);
          tc_fence_after();
          if (first && lane == 0) tl_stamp(a.tl, 4, p);
          first = false;
          const uint64_t db = desc_add(dB0, s * stage_bytes);
          if (elect_one()) {
            if (kW4) {
              const uint32_t ta = tmem_base + a_col0 + ai * a_cols;
#pragma unroll
              for (int sub = 0; sub < 4; ++sub)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  umma_bf16_ts(d, ta + sub * 32u + kk * 8u, desc_add(db, sub * b_bytes + kk * 256u), idesc,
                               (k != k0 || sub != 0 || kk != 0) ? 1u : 0u);
              umma_commit(&aempty[ai]);
            } else {
              const uint64_t da = desc_add(dA0, s * stage_bytes);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(d, desc_add(da, kk * 256u), desc_add(db, kk * 256u), idesc, (k != k0 || kk != 0) ? 1u : 0u);
            }
            umma_commit(&empty[s]);
          }
          __syncwarp();
          if (++s == (uint32_t)stages) {
            s = 0;
            ph ^= 1;
          }
          if (kW4 && ++ai == (uint32_t)astages) {
            ai = 0;
            aph ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
        ++u;
      }
    }
  } else if (warp < 6) {
    // ------------------------------- epilogue, row phases, grid-barrier arrivals
    pdl_wait();  // partial slots are still read by the attention kernel before it
    // this CTA's barrier counter before its first arrival of the launch
    if (threadIdx.x == 64) *s_base = gbar_base(a.bar);
    epi_sync();
    const uint32_t base = *s_base;
    const int quad = warp & 3;
    uint32_t u = 0;
    for (int p = 0; p < kPhases; ++p) {
      const GemmPlanDev& plan = a.plan[p];
      const int N = a.w[p].N, nk = plan.nk;
      SegIter seg(plan, cta);
      int t, k0, k1;
      while (cta < plan.C && seg.next(t, k0, k1)) {
        const uint32_t acc = acc_bufs == 2 ? (u & 1) : 0u;
        const uint32_t use = acc_bufs == 2 ? (u >> 1) : u;
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        const int n_tile = t % plan.n_tiles;
        const int slot = plan.aligned ? 0 : cta - plan_cta_of(plan, (int64_t)t * nk);
        const int n = n_tile * 128 + quad * 32 + lane;
        float* o = a.part + (size_t)slot * a.M * N;
        const uint32_t d = tmem_base + acc * tm_cols + ((uint32_t)(quad * 32) << 16);
        for (int c0 = 0; c0 < TM; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(d + (uint32_t)c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = c0 + j;
            if (m < a.M) o[(size_t)m * N + n] = __uint_as_float(v[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        ++u;
      }
      // phase p's partials complete (this CTA) -> barrier 2p+1
      epi_sync();
      if (threadIdx.x == 64) {
        tl_stamp(a.tl, 0, p);
        gbar_arrive(a.bar, base + 2 * p + 1);
      }
      if (warp == 2) gbar_wait(a.bar, base + 2 * p + 1);
      epi_sync();
      if (threadIdx.x == 64) tl_stamp(a.tl, 1, p);
      if (p == 0) rows_residual_norm(a, plan, a.norm2, TM, 0, red);
      else if (p == 1) rows_silu(a, plan);
      else rows_residual_norm(a, plan, a.norm_next, a.tm_out, a.row_begin, red);
      if (p < kPhases - 1) {
        // generic-proxy stores of x -> bulk-copy (async proxy) reads on other SMs
        asm volatile("fence.proxy.async.global;" ::: "memory");
        epi_sync();
        if (threadIdx.x == 64) {
          tl_stamp(a.tl, 2, p);
          gbar_arrive(a.bar, base + 2 * p + 2);
        }
        if (warp == 2) {  // one poller per CTA; the activation producer waits on `bgo`
          gbar_wait(a.bar, base + 2 * p + 2);
          if (lane == 0) mbar_arrive(bgo);
        }
      } else if (threadIdx.x == 64) {
        tl_stamp(a.tl, 2, p);
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------ activation (B) producer
    pdl_wait();  // phase 0's activations are the attention kernel's output
    uint32_t it = 0;
    for (int p = 0; p < kPhases; ++p) {
      const GemmPlanDev& plan = a.plan[p];
      if (p > 0) {
        mbar_wait(bgo, (uint32_t)(p - 1) & 1);  // barrier 2p: the row phase wrote this phase's activations
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (lane == 0) tl_stamp(a.tl, 3, p);
      if (cta >= plan.C) continue;
      SegIter seg(plan, cta);
      int t, k0, k1;
      const uint32_t unit = kW4 ? 4u * b_bytes : b_bytes;
      while (seg.next(t, k0, k1)) {
        const uint8_t* xb = reinterpret_cast<const uint8_t*>(a.x);  // one m-tile (M <= TM)
        for (int k = k0; k < k1; ++k, ++it) {
          const uint32_t s = it % (uint32_t)stages;
          if (it >= (uint32_t)stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
          if (lane == 0) {
            if (kW4) mbar_expect_tx(&full[s], unit);
            bulk_g2s(sB(s), xb + (size_t)k * unit, unit, &full[s]);
          }
          __syncwarp();
        }
      }
    }
  } else if constexpr (kW4) {
    // ------------------------------------------------------------ dequantisers
    // group g takes the units it = g, g + kG, ... of the global unit sequence;
    // warp quadrant q owns TMEM lanes / weight rows 32q..32q+31
    const int quad = warp & 3, grp = (warp - 7) >> 2;
    const int row = quad * 32 + lane;
    const __nv_bfloat162 bias = __floats2bfloat162_rn(136.0f, 136.0f);
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16) + a_col0;
    uint32_t it = 0;
    for (int p = 0; p < kPhases; ++p) {
      const GemmPlanDev& plan = a.plan[p];
      if (cta >= plan.C) continue;
      SegIter seg(plan, cta);
      int t, k0, k1;
      while (seg.next(t, k0, k1)) {
        int k = k0 + (int)((grp - (int)(it % kG) + kG) % kG);
        it += (uint32_t)(k - k0);
        for (; k < k1; k += kG, it += kG) {
          const uint32_t rs = it % (uint32_t)rstages, ai = it % (uint32_t)astages;
          mbar_wait(&rfull[rs], (it / rstages) & 1);
          const uint8_t* raw = sRaw(rs);
          __nv_bfloat162 sc[2];
          uint4 q[2][4];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint8_t* rh = raw + hh * kW4ChunkBytes;
            sc[hh].x = __ushort_as_bfloat16(*reinterpret_cast<const uint16_t*>(rh + 8192 + 2 * row));
            sc[hh].y = sc[hh].x;
#pragma unroll
            for (int j = 0; j < 4; ++j) q[hh][j] = *reinterpret_cast<const uint4*>(rh + (j * 128 + row) * 16);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[rs]);
          if (it >= (uint32_t)astages) mbar_wait(&aempty[ai], ((it / astages) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t o[32];
#pragma unroll
              for (int jj = 0; jj < 2; ++jj) {
                const uint4 qq = q[hh][half * 2 + jj];
                const uint32_t words[4] = {qq.x, qq.y, qq.z, qq.w};
#pragma unroll
                for (int wd = 0; wd < 4; ++wd)
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const uint32_t x = nib_magic(words[wd] >> (4 * i));
                    __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&x);
                    v = __hmul2(__hsub2(v, bias), sc[hh]);  // exact code, then one rounding of code*scale
                    o[jj * 16 + wd * 4 + i] = *reinterpret_cast<uint32_t*>(&v);
                  }
              }
              tmem_st32(lane_base + ai * a_cols + (uint32_t)hh * 64u + (uint32_t)half * 32u, o);
            }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&afull[ai]);
        }
        it -= (uint32_t)(k - k1);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) tl_stamp(a.tl, 7, 0);
  if (warp == 1) tmem_dealloc(tmem_base, 512);
}

namespace {
int layer_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <bool kW4, int kG>
cudaError_t launch_layer(const DecodeLayerArgs& a, int grid, cudaStream_t s) {
  const int TM = a.TM;
  const size_t budget = 215 * 1024;
  int stages, rstages = 0, astages = 0;
  size_t ring;
  if (kW4) {
    const size_t bst = (size_t)TM * 128 * 4;
    stages = TM <= 64 ? 3 : (TM <= 128 ? 2 : 1);
    rstages = std::min(16, (int)((budget - stages * bst) / 16896));
    if (rstages < 2) return cudaErrorInvalidValue;
    const int tm_cols = TM <= 32 ? 32 : TM <= 64 ? 64 : TM <= 128 ? 128 : 256;
    const int acc = (TM <= 128 ? 2 : 1) * tm_cols;
    astages = std::min(kLayerMaxAStages, (512 - acc) / 128);
    if (astages < kG) return cudaErrorInvalidValue;
    ring = stages * bst + (size_t)rstages * 16896;
  } else {
    static const int max_st = layer_env("MS_GEMM_STAGES", 8);
    const size_t st = 16384 + (size_t)TM * 128;
    stages = std::max(2, std::min(max_st, (int)(budget / st)));
    ring = stages * st;
  }
  const size_t smem = ring + (size_t)(2 * stages + 4 + 2 * rstages + 2 * kLayerMaxAStages) * 8 + 128 + 64;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_layer_kernel<kW4, kG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  return launch_pdl(decode_layer_kernel<kW4, kG>, dim3(grid), dim3(kW4 ? (7 + 4 * kG) * 32 : 224), smem, s, a, stages,
                    rstages, astages);
}
}  // namespace

bool decode_layer_ok(const DecodeLayerArgs& a, bool w4) {
  if (a.M < 1 || a.M > a.TM || a.TM > 256 || a.TM % 16) return false;
  if (w4 && a.TM > 128) return false;  // (TMEM: two accumulators + >= 2 dequantised A stages)
  if (a.d % 128) return false;
  for (int p = 0; p < kPhases; ++p) {
    if (w4 && a.w[p].K % 256) return false;
    if (a.plan[p].aligned) return false;  // stream-K decode plans only
  }
  return true;
}

cudaError_t decode_layer_launch(const DecodeLayerArgs& a, bool w4, int grid, cudaStream_t s) {
  if (!w4) return launch_layer<false, 1>(a, grid, s);
  // dequantiser groups: MS_W4_GROUPS (default 3), at most the TMEM A stages
  // left beside the double-buffered accumulators (one stage per group)
  static const int groups = layer_env("MS_W4_GROUPS", 3);
  const int tm_cols = a.TM <= 32 ? 32 : a.TM <= 64 ? 64 : a.TM <= 128 ? 128 : 256;
  const int astages = std::min(kLayerMaxAStages, (512 - (a.TM <= 128 ? 2 : 1) * tm_cols) / 128);
  switch (std::min(groups, astages)) {
    case 2: return launch_layer<true, 2>(a, grid, s);
    case 4: return launch_layer<true, 4>(a, grid, s);
    default: return launch_layer<true, 3>(a, grid, s);
  }
}

}  // namespace ms
