// attention.cu -- paged GQA decode attention over the resizable KV arena.
//
// Replaces the priced stand-in `attn_ms_per_kv_block * batch_blocks`
// (reference proj/src/sim_config.cpp:23-27): this kernel walks each sequence's
// device block table (page indices mirrored from the host KvBlockPool, whose
// logical ids stay bit-exact with the reference) and streams the K/V tiles of
// every block through a shared-memory ring filled by 1-D bulk async copies
// (one cp.async.bulk of block_tokens*head_dim*4 bytes per block per KV head:
// the K tile and the V tile of a (page, layer, kv_head) are adjacent).
//
// One CTA = one (kv_head, query row, KV split).  Warp 4 lane 0 produces; warps
// 0..3 each own block_tokens/4 tokens of every block and all G = H/KVH query
// heads of the group (GQA reuse: each K/V byte feeds G heads), keep an online
// softmax in the log2 domain, and merge at the end.  Split-KV slices are
// merged by attn_combine_kernel.
//
// The same kernel runs prefill attention: every prefill token is a query row
// with ctx_len = position + 1 that shares one page-table row (page_row[r]=0).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

// q enters every attention path rounded to bf16
__device__ __forceinline__ float bf16r(float x) { return bf2f(f2bf(x)); }

// K/V ring depth and CTAs per SM (MS_ATTN_STAGES / MS_ATTN_CTAS override,
// experiments): bytes in flight per SM = CTAs x stages x 8 KB.
constexpr int kAttnMaxStages = 12;
static int attn_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// CTA -> (kv_head, row, split, splits) under the whole/tail item map (AttnArgs).
__device__ __forceinline__ void attn_item(const AttnArgs& a, int& kvh, int& row, int& split, int& ns) {
  const int bid = blockIdx.x;
  int item;
  if (bid < a.whole_items) {
    item = bid;
    split = 0;
    ns = 1;
  } else {
    const int j = bid - a.whole_items;
    item = a.whole_items + j / a.tail_splits;
    split = j % a.tail_splits;
    ns = a.tail_splits;
  }
  row = item / a.KVH;
  kvh = item - row * a.KVH;
}

// Sum of the first n split-K partial slots of one element (slot order fixed,
// as elementwise.cu sum_slots: bit-identical to the unfused qkv_post path).
__device__ __forceinline__ float attn_sum_slots(const float* p, size_t stride, int n) {
  float v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = s < n ? __ldcg(p + s * stride) : 0.f;
  float acc = 0.f;
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s < n) acc += v[s];
  for (int s = 8; s < n; ++s) acc += __ldcg(p + s * stride);
  return acc;
}

// Fused QKV post-processing for one (kv_head, row) CTA: q of the G heads of the
// group (RoPE'd, fp32) into `qs`, and -- by the CTA that streams the row's last
// block -- the rotated K and the V of the new token into the paged cache.  The
// arithmetic is qkv_post_kernel's (elementwise.cu), element for element.
template <int HD, int G>
__device__ __forceinline__ void attn_qkv_fused(const AttnArgs& a, int kvh, int row, bool append, float* qs, int tid,
                                               int nthr) {
  constexpr int half = HD / 2;
  const int H = a.H, KVH = a.KVH;
  const int N = (H + 2 * KVH) * HD;
  const int p = a.pos[row];
  const size_t stride = (size_t)a.rows * N;
  const int nheads = G + (append ? 2 : 0);
  for (int idx = tid; idx < nheads * half; idx += nthr) {
    const int hh = idx / half, i = idx - hh * half;
    const int hs = hh < G ? kvh * G + hh : (hh == G ? H + kvh : H + KVH + kvh);  // q, k, v head slot
    const int c0 = hs * HD + i;
    const float* src = a.qkv_part + (size_t)row * N + c0;
    float x0 = attn_sum_slots(src, stride, part_slots(a.qkv_plan, row, c0));
    float x1 = attn_sum_slots(src + half, stride, part_slots(a.qkv_plan, row, c0 + half));
    if (hs < H + KVH) {
      const float c = a.rope_cos[(size_t)p * half + i], sn = a.rope_sin[(size_t)p * half + i];
      const float y0 = x0 * c - x1 * sn;
      const float y1 = x1 * c + x0 * sn;
      x0 = y0;
      x1 = y1;
    }
    if (hh < G) {
      qs[hh * HD + i] = x0;
      qs[hh * HD + i + half] = x1;
    } else {
      const int prow = a.page_row ? a.page_row[row] : row;
      const int32_t page = a.pages[(size_t)prow * a.page_stride + p / a.kv.block_tokens];
      const bool is_v = hh == G + 1;
      uint16_t* dst = reinterpret_cast<uint16_t*>(a.kv.arena + (int64_t)page * a.kv.page_bytes + a.kv.layer_off(a.layer) +
                                                  (int64_t)kvh * 2 * a.kv.head_bytes() +
                                                  (is_v ? a.kv.head_bytes() : 0)) +
                      (p % a.kv.block_tokens) * HD;
      dst[i] = f2bf(x0);
      dst[i + half] = f2bf(x1);
    }
  }
  // the new K/V token is read back through the async (bulk copy) proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int HD, int G, int BT>
__global__ void __launch_bounds__(160) attn_decode_kernel(AttnArgs a) {
  constexpr int VEC = HD / 32;
  constexpr int TPW = BT / 4;  // tokens per consumer warp per block
  constexpr uint32_t kStageBytes = (uint32_t)BT * HD * 2 * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  // MHA (one head per KV head) at hd 128: warp-per-block consumer
  constexpr bool kWarpPerBlock = G == 1 && HD == 128 && BT == 16;
  __shared__ __align__(16) float pbuf[4 * 16];
  const int kAttnStages = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAttnStages * kStageBytes);
  uint64_t* empty = full + kAttnStages;
  uint64_t* kv_ready = empty + kAttnStages;  // the new token's K/V is in the cache (fused QKV); 16 B slot
  float* scratch = reinterpret_cast<float*>(kv_ready + 2);  // [4][G][HD] acc + [4][G][2] m,l

  // No grid-dependency wait before the producer starts: the K/V of earlier
  // tokens, the block table and ctx_len were written by kernels that completed
  // before this grid launched (the previous kernel -- the QKV GEMM -- writes
  // only its fp32 partials, and every row kernel waits before it triggers),
  // so the ring fills while the QKV GEMM drains and the consumers wait for it.
  // Only the block receiving the new token waits, for the consumers' append.
  int kvh, row, split, nsplit;
  attn_item(a, kvh, row, split, nsplit);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctx = a.ctx_len[row];
  const int nb = (ctx + BT - 1) / BT;
  const int b0 = (int)((int64_t)nb * split / nsplit), b1 = (int)((int64_t)nb * (split + 1) / nsplit);
  const int prow = a.page_row ? a.page_row[row] : row;
  const int32_t* ptab = a.pages + (size_t)prow * a.page_stride;
  const int64_t kv_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarpPerBlock ? 1 : 4);
    }
    mbar_init(kv_ready, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // q source: fused QKV post-processing into shared memory, or the q buffer
  float* qsm = scratch + (size_t)4 * G * HD + 8 * G;  // [G][HD] fp32
  const bool fused = a.qkv_part != nullptr;
  const bool append = fused && b1 == nb;  // this CTA writes (then streams) the new token's block
  if (warp != 4) {  // consumers (named barrier 1): after the QKV GEMM, q into smem, new K/V into the cache
    pdl_wait();
    pdl_trigger();
    if (fused) {
      attn_qkv_fused<HD, G>(a, kvh, row, append, qsm, threadIdx.x, 128);  // ends with a generic->async proxy fence
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0 && append) mbar_arrive(kv_ready);
    }
  }
  const float* qsrc = fused ? qsm : a.q + ((size_t)row * a.H + kvh * G) * HD;

  float m[G], l[G], acc[G][VEC];
  if (warp == 4) {
    pdl_trigger();  // every thread of the CTA signals (the consumers after their wait)
    // page ids of the next 32 blocks in one warp-wide load, handed to lane 0
    // by shuffle (no dependent global load in front of each copy)
    int pid = 0;
    for (int it = 0; it < b1 - b0; ++it) {
      if ((it & 31) == 0) pid = it + lane < b1 - b0 ? __ldg(ptab + b0 + it + lane) : 0;
      const int page = __shfl_sync(0xffffffffu, pid, it & 31);
      const int s = it % kAttnStages;
      // the whole warp waits on the ring (measured on the GQA producer: lane-0-only
      // waits were 1.5% slower per 8B step)
      if (it >= kAttnStages) mbar_wait(&empty[s], ((it / kAttnStages) & 1) ^ 1);
      if (append && b0 + it == nb - 1) mbar_wait(kv_ready, 0);
      if (lane == 0) {
        const char* src = a.kv.arena + (int64_t)page * a.kv.page_bytes + kv_off;
        mbar_expect_tx(&full[s], kStageBytes);
        bulk_g2s(smem + (size_t)s * kStageBytes, src, kStageBytes, &full[s]);
      }
      __syncwarp();
    }
  } else if constexpr (kWarpPerBlock) {
    // ---- MHA consumer: one warp per 16-token block (blocks it = warp, warp+4, ...).
    // Lane (t = lane/2, half h = lane%2) computes token t's score over 64 of the
    // 128 dims from register-resident q (no cross-lane reduction but one
    // shuffle), the block softmax is 4 shuffle rounds, and P.V runs with each
    // lane owning 4 output dims.  The 16-byte K chunks are rotated per lane
    // (chunk (2i + 2t + h) mod 16) so the LDS.128s are bank-conflict free.
    const int t = lane >> 1, h = lane & 1;
    const int rot = (2 * t + h) & 15;
    float qr[8][8];
    {
      const float* qp = qsrc;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = (2 * i + rot) & 15;
        const float4 x0 = *reinterpret_cast<const float4*>(qp + c * 8);
        const float4 x1 = *reinterpret_cast<const float4*>(qp + c * 8 + 4);
        qr[i][0] = bf16r(x0.x) * a.scale_log2;
        qr[i][1] = bf16r(x0.y) * a.scale_log2;
        qr[i][2] = bf16r(x0.z) * a.scale_log2;
        qr[i][3] = bf16r(x0.w) * a.scale_log2;
        qr[i][4] = bf16r(x1.x) * a.scale_log2;
        qr[i][5] = bf16r(x1.y) * a.scale_log2;
        qr[i][6] = bf16r(x1.z) * a.scale_log2;
        qr[i][7] = bf16r(x1.w) * a.scale_log2;
      }
    }
    float* pb = pbuf + warp * 16;
    m[0] = -INFINITY;
    l[0] = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[0][e] = 0.f;
    for (int it = warp; it < b1 - b0; it += 4) {
      const int s = it % kAttnStages;
      mbar_wait(&full[s], (it / kAttnStages) & 1);
      const uint8_t* Kt = smem + (size_t)s * kStageBytes;
      const uint8_t* Vt = Kt + BT * HD * 2;
      float sp = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = (2 * i + rot) & 15;
        const uint4 kr = *reinterpret_cast<const uint4*>(Kt + t * (HD * 2) + c * 16);
        sp = fmaf(qr[i][0], __uint_as_float(kr.x << 16), sp);
        sp = fmaf(qr[i][1], __uint_as_float(kr.x & 0xFFFF0000u), sp);
        sp = fmaf(qr[i][2], __uint_as_float(kr.y << 16), sp);
        sp = fmaf(qr[i][3], __uint_as_float(kr.y & 0xFFFF0000u), sp);
        sp = fmaf(qr[i][4], __uint_as_float(kr.z << 16), sp);
        sp = fmaf(qr[i][5], __uint_as_float(kr.z & 0xFFFF0000u), sp);
        sp = fmaf(qr[i][6], __uint_as_float(kr.w << 16), sp);
        sp = fmaf(qr[i][7], __uint_as_float(kr.w & 0xFFFF0000u), sp);
      }
      float sc = sp + __shfl_xor_sync(0xffffffffu, sp, 1);
      const int tok0 = (b0 + it) * BT;
      if (tok0 + t >= ctx) sc = -INFINITY;
      float mx = sc;
#pragma unroll
      for (int o = 2; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mn = fmaxf(m[0], mx);  // finite: every block holds >= 1 valid token
      const float corr = exp2f(m[0] - mn);
      const float p = exp2f(sc - mn);
      float ps = p;
#pragma unroll
      for (int o = 2; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l[0] = l[0] * corr + ps;
      m[0] = mn;
      if (h == 0) pb[t] = p;
      __syncwarp();
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[0][e] *= corr;
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 pv = *reinterpret_cast<const float4*>(pb + j4 * 4);
        const float pj[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const uint2 vr = *reinterpret_cast<const uint2*>(Vt + (j4 * 4 + jj) * (HD * 2) + lane * 8);
          acc[0][0] = fmaf(pj[jj], __uint_as_float(vr.x << 16), acc[0][0]);
          acc[0][1] = fmaf(pj[jj], __uint_as_float(vr.x & 0xFFFF0000u), acc[0][1]);
          acc[0][2] = fmaf(pj[jj], __uint_as_float(vr.y << 16), acc[0][2]);
          acc[0][3] = fmaf(pj[jj], __uint_as_float(vr.y & 0xFFFF0000u), acc[0][3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // stash per-warp state (same layout as the generic consumer)
    float* sacc = scratch + (size_t)warp * G * HD;
    float* sml = scratch + (size_t)4 * G * HD + (size_t)warp * G * 2;
#pragma unroll
    for (int e = 0; e < VEC; ++e) sacc[lane * VEC + e] = acc[0][e];
    if (lane == 0) {
      sml[0] = m[0];
      sml[1] = l[0];
    }
  } else {
    float qv[G][VEC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* qp = qsrc + (size_t)g * HD + lane * VEC;
#pragma unroll
      for (int i = 0; i < VEC; ++i) qv[g][i] = bf16r(qp[i]) * a.scale_log2;
      m[g] = -INFINITY;
      l[g] = 0.f;
#pragma unroll
      for (int i = 0; i < VEC; ++i) acc[g][i] = 0.f;
    }
    for (int it = 0; it < b1 - b0; ++it) {
      const int s = it % kAttnStages;
      mbar_wait(&full[s], (it / kAttnStages) & 1);
      const uint16_t* Kt = reinterpret_cast<const uint16_t*>(smem + (size_t)s * kStageBytes);
      const uint16_t* Vt = Kt + BT * HD;
      const int tok0 = (b0 + it) * BT;
      float sc[TPW][G];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + 4 * i;
        float kf[VEC];
        if constexpr (VEC == 4) {
          const uint2 kr = *reinterpret_cast<const uint2*>(Kt + t * HD + lane * 4);
          kf[0] = __uint_as_float(kr.x << 16);
          kf[1] = __uint_as_float(kr.x & 0xFFFF0000u);
          kf[2] = __uint_as_float(kr.y << 16);
          kf[3] = __uint_as_float(kr.y & 0xFFFF0000u);
        } else {
          const uint32_t kr = *reinterpret_cast<const uint32_t*>(Kt + t * HD + lane * 2);
          kf[0] = __uint_as_float(kr << 16);
          kf[1] = __uint_as_float(kr & 0xFFFF0000u);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float p = 0.f;
#pragma unroll
          for (int e = 0; e < VEC; ++e) p = fmaf(qv[g][e], kf[e], p);
          sc[i][g] = p;
        }
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int g = 0; g < G; ++g) sc[i][g] = warp_sum(sc[i][g]);

      float vf[TPW][VEC];
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int t = warp + 4 * i;
        if constexpr (VEC == 4) {
          const uint2 vr = *reinterpret_cast<const uint2*>(Vt + t * HD + lane * 4);
          vf[i][0] = __uint_as_float(vr.x << 16);
          vf[i][1] = __uint_as_float(vr.x & 0xFFFF0000u);
          vf[i][2] = __uint_as_float(vr.y << 16);
          vf[i][3] = __uint_as_float(vr.y & 0xFFFF0000u);
        } else {
          const uint32_t vr = *reinterpret_cast<const uint32_t*>(Vt + t * HD + lane * 2);
          vf[i][0] = __uint_as_float(vr << 16);
          vf[i][1] = __uint_as_float(vr & 0xFFFF0000u);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);

#pragma unroll
      for (int g = 0; g < G; ++g) {
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < TPW; ++i)
          if (tok0 + warp + 4 * i < ctx) mx = fmaxf(mx, sc[i][g]);
        const float mn = fmaxf(m[g], mx);
        if (mn == -INFINITY) continue;
        const float corr = exp2f(m[g] - mn);
        float lsum = l[g] * corr;
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[g][e] *= corr;
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const float p = (tok0 + warp + 4 * i < ctx) ? exp2f(sc[i][g] - mn) : 0.f;
          lsum += p;
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[g][e] = fmaf(p, vf[i][e], acc[g][e]);
        }
        l[g] = lsum;
        m[g] = mn;
      }
    }
    // stash per-warp state
    float* sacc = scratch + (size_t)warp * G * HD;
    float* sml = scratch + (size_t)4 * G * HD + (size_t)warp * G * 2;
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) sacc[g * HD + lane * VEC + e] = acc[g][e];
      if (lane == 0) {
        sml[g * 2 + 0] = m[g];
        sml[g * 2 + 1] = l[g];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 128) {
    const float* sml = scratch + (size_t)4 * G * HD;
    for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
      const int g = idx / HD, dim = idx - g * HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, sml[(w * G + g) * 2]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float f = exp2f(sml[(w * G + g) * 2] - M);
          L += sml[(w * G + g) * 2 + 1] * f;
          O += scratch[(size_t)(w * G + g) * HD + dim] * f;
        }
      }
      const int h = kvh * G + g;
      const float o = L > 0.f ? O / L : 0.f;
      if (nsplit == 1) {
        const int K = a.H * HD;
        const size_t off = a.out_packed ? act_off(row, h * HD + dim, K, a.TM) : (size_t)row * K + h * HD + dim;
        a.out[off] = f2bf(o);
      } else {
        const size_t base = ((size_t)split * a.rows + row) * a.H + h;
        a.part_o[base * HD + dim] = o;
        if (dim == 0) {
          a.part_ml[base * 2 + 0] = M;
          a.part_ml[base * 2 + 1] = L;
        }
      }
    }
  }
}

template <int HD>
__global__ void attn_combine_kernel(AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x, h = blockIdx.y, dim = threadIdx.x;
  if (row * a.KVH + h / (a.H / a.KVH) < a.whole_items) return;  // written directly by its CTA
  const int ns = a.tail_splits;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, a.part_ml[(((size_t)s * a.rows + row) * a.H + h) * 2]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < ns; ++s) {
      const size_t base = ((size_t)s * a.rows + row) * a.H + h;
      const float ms_ = a.part_ml[base * 2], ls = a.part_ml[base * 2 + 1];
      if (ms_ == -INFINITY) continue;
      const float f = ls * exp2f(ms_ - M);
      L += f;
      O += f * a.part_o[base * HD + dim];
    }
  }
  const float o = L > 0.f ? O / L : 0.f;
  const int K = a.H * HD;
  const size_t off = a.out_packed ? act_off(row, h * HD + dim, K, a.TM) : (size_t)row * K + h * HD + dim;
  a.out[off] = f2bf(o);
}

// ---------------------------------------------------------------------------
// GQA decode attention (G = H / KVH >= 2 query heads per KV head, hd 128) on the
// tensor cores: per 16-token block one consumer warp computes S = Q K^T with
// mma.sync m16n8k16 (the G query heads are the M rows, bf16(q) as on every
// attention path; rows G..15 are padding), the online
// softmax on the accumulator fragments, and O += P V (P bf16).  The producer
// warp stages each block's K and V rows with 16-byte cp.async into an
// XOR-swizzled layout (chunk c of row r at c ^ (r & 7)) so the ldmatrix
// fragment loads are bank-conflict free; completion is tracked per stage by an
// mbarrier.  (TMA tensor copies now: one 3-D box per block, 128B-swizzled.)  About 140 instructions per block
// per warp, versus ~1000 for the CUDA-core consumer with G shuffle reductions.
__device__ __forceinline__ void gqa_ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void gqa_ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void gqa_mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset (from the K rows' base) of 16-B chunk c (0..7) of half h of row r in
// the TMA tile [half][32 rows][128 B] with the 128B swizzle (chunk ^ row % 8)
__device__ __forceinline__ uint32_t gqa_tsw(int r, int h, int c) {
  return (uint32_t)(h * 4096 + r * 128 + ((c ^ (r & 7)) * 16));
}

template <int G>
__global__ void __launch_bounds__(160) attn_gqa_mma_kernel(AttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  constexpr int HD = 128, BT = 16;
  constexpr uint32_t kStageBytes = (uint32_t)BT * HD * 2 * 2;  // [half][K rows 0-15 | V rows 16-31][128 B], swizzled
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128B-swizzled TMA destinations need 1024-B alignment
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int S = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* kv_ready = empty + S;  // the new token's K/V is in the cache (fused QKV)
  float* scratch = reinterpret_cast<float*>(kv_ready + 1);  // [4][G][HD] acc + [4][G][2] m,l, then q [G][HD]

  // producer streams before the grid-dependency wait (see attn_decode_kernel)
  int kvh, row, split, nsplit;
  attn_item(a, kvh, row, split, nsplit);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctx = a.ctx_len[row];
  const int nb = (ctx + BT - 1) / BT;
  const int b0 = (int)((int64_t)nb * split / nsplit), b1 = (int)((int64_t)nb * (split + 1) / nsplit);
  const int prow = a.page_row ? a.page_row[row] : row;
  const int32_t* ptab = a.pages + (size_t)prow * a.page_stride;
  const int64_t kv_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);  // producer lane 0: expect_tx of the block's tensor copy
      mbar_init(&empty[s], 1);  // the one warp that consumed the block
    }
    mbar_init(kv_ready, 1);
    fence_mbar_init();
  }
  __syncthreads();
  float* qsm = scratch + (size_t)4 * G * HD + 8 * G;  // [G][HD] fp32
  const bool fused = a.qkv_part != nullptr;
  const bool append = fused && b1 == nb;  // this CTA writes (then streams) the new token's block

  if (warp == 4) {
    // ------------------------------------------------------------ producer
    // streams from the start; only the block holding the new token waits for
    // the consumers' fused QKV append
    pdl_trigger();
    int pid = 0;  // page ids of the next 32 blocks, one warp-wide load
    for (int it = 0; it < b1 - b0; ++it) {
      if ((it & 31) == 0) pid = it + lane < b1 - b0 ? __ldg(ptab + b0 + it + lane) : 0;
      const int page = __shfl_sync(0xffffffffu, pid, it & 31);
      const int s = it % S;
      if (it >= S) mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      if (append && b0 + it == nb - 1) mbar_wait(kv_ready, 0);
      // one TMA tensor copy per block: the 32 K|V rows of 256 B, as two 128-B
      // halves, 128B-swizzled by the copy engine (conflict-free ldmatrix)
      if (lane == 0) {
        const int64_t row = ((int64_t)page * a.kv.page_bytes + kv_off) >> 8;  // 256-B row of the arena
        mbar_expect_tx(&full[s], kStageBytes);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(smem_u32(smem + (size_t)s * kStageBytes)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"((int)row), "r"(0), "r"(smem_u32(&full[s]))
            : "memory");
      }
      __syncwarp();
    }
    return;
  }
  // ------------------------------------------------------------- consumers
  pdl_wait();
  pdl_trigger();
  if (fused) {  // consumers only (named barrier 1): q into smem, new K/V into the cache
    attn_qkv_fused<HD, G>(a, kvh, row, append, qsm, threadIdx.x, 128);  // ends with a generic->async proxy fence
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (threadIdx.x == 0 && append) mbar_arrive(kv_ready);
  }
  const float* qsrc = fused ? qsm : a.q + ((size_t)row * a.H + kvh * G) * HD;
  const int g = lane >> 2, t4 = lane & 3;  // fragment row (query head) / column pair
  // Q A-fragments: rows g < G hold bf16(q) of query head g (unscaled, the
  // attention contract of every path); rows >= G (and g + 8) are zero
  uint32_t qh[8][2];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      float x0 = 0.f, x1 = 0.f;
      if (g < G) {
        const float* qp = qsrc + (size_t)g * HD + ks * 16 + hf * 8 + 2 * t4;
        x0 = qp[0];
        x1 = qp[1];
      }
      qh[ks][hf] = pack_bf2(x0, x1);
    }
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m = -INFINITY, l = 0.f;  // for query head g (rows g + 8 are padding)
  // ldmatrix row / chunk of this lane: matrices 0..3 = (rows 0-7 | 8-15) x (chunk c | c+1)
  const int lr = (lane & 7) + ((lane >> 4) << 3), lc = (lane >> 3) & 1;
  for (int it = warp; it < b1 - b0; it += 4) {
    const int s = it % S;
    mbar_wait(&full[s], (it / S) & 1);
    const uint32_t kt = smem_u32(smem + (size_t)s * kStageBytes), vt = kt + 16 * 128;  // V rows = lines 16..31
    // ---- S = Q K^T: n-tile 0 = tokens 0-7, n-tile 1 = tokens 8-15 (A rows
    // g + 8 are zero padding of the m16 shape)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t k0, k1, k2, k3;  // (tok 0-7, dims 16ks..+7), (tok 0-7, +8..), (tok 8-15, ..), (tok 8-15, +8..)
      gqa_ldsm_x4(kt + gqa_tsw(lr, ks >> 2, 2 * (ks & 3) + lc), k0, k1, k2, k3);
      gqa_mma(sc[0], qh[ks][0], 0u, qh[ks][1], 0u, k0, k1);
      gqa_mma(sc[1], qh[ks][0], 0u, qh[ks][1], 0u, k2, k3);
    }
    // ---- online softmax for head g over this block's 16 tokens
    const int tok0 = (b0 + it) * BT;
    // tokens 2t4, 2t4+1, 8+2t4, 9+2t4 of head g, scaled to the log2 domain
    const float sl = a.scale_log2;
    float v4[4] = {sc[0][0] * sl, sc[0][1] * sl, sc[1][0] * sl, sc[1][1] * sl};
    const int tk[4] = {2 * t4, 2 * t4 + 1, 8 + 2 * t4, 9 + 2 * t4};
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (tok0 + tk[e] >= ctx) v4[e] = -INFINITY;
      mx = fmaxf(mx, v4[e]);
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m, mx);  // finite: every block holds >= 1 valid token
    const float corr = exp2f(m - mn);
    float p[4], ps = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      p[e] = exp2f(v4[e] - mn);
      ps += p[e];
    }
    ps += __shfl_xor_sync(0xffffffffu, ps, 1);
    ps += __shfl_xor_sync(0xffffffffu, ps, 2);
    l = l * corr + ps;
    m = mn;
    const uint32_t pa0 = pack_bf2(p[0], p[1]), pa2 = pack_bf2(p[2], p[3]);
    // ---- O = O * corr + P V
#pragma unroll
    for (int jp = 0; jp < 8; ++jp) {
      o[2 * jp][0] *= corr;
      o[2 * jp][1] *= corr;
      o[2 * jp + 1][0] *= corr;
      o[2 * jp + 1][1] *= corr;
      uint32_t v0, v1, v2, v3;  // trans: (tok 0-7, dims 16jp..), (tok 8-15, ..), (tok 0-7, +8), (tok 8-15, +8)
      const int vr = (lane & 7) + (((lane >> 3) & 1) << 3), vc = 2 * jp + (lane >> 4);
      gqa_ldsm_x4_t(vt + gqa_tsw(vr, vc >> 3, vc & 7), v0, v1, v2, v3);
      gqa_mma(o[2 * jp], pa0, 0u, pa2, 0u, v0, v1);  // rows g + 8 of O stay 0
      gqa_mma(o[2 * jp + 1], pa0, 0u, pa2, 0u, v2, v3);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // stash per-warp state: head g < G, dims 8j + 2t4, +1
  if (g < G) {
    float* sacc = scratch + ((size_t)warp * G + g) * HD;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      sacc[8 * j + 2 * t4] = o[j][0];
      sacc[8 * j + 2 * t4 + 1] = o[j][1];
    }
    if (t4 == 0) {
      float* sml = scratch + (size_t)4 * G * HD + ((size_t)warp * G + g) * 2;
      sml[0] = m;
      sml[1] = l;
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const float* smlv = scratch + (size_t)4 * G * HD;
  for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
    const int gg = idx / HD, dim = idx - gg * HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, smlv[(w * G + gg) * 2]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(smlv[(w * G + gg) * 2] - M);
        L += smlv[(w * G + gg) * 2 + 1] * f;
        O += scratch[(size_t)(w * G + gg) * HD + dim] * f;
      }
    }
    const int h = kvh * G + gg;
    const float ov = L > 0.f ? O / L : 0.f;
    if (nsplit == 1) {
      const int K = a.H * HD;
      const size_t off = a.out_packed ? act_off(row, h * HD + dim, K, a.TM) : (size_t)row * K + h * HD + dim;
      a.out[off] = f2bf(ov);
    } else {
      const size_t base = ((size_t)split * a.rows + row) * a.H + h;
      a.part_o[base * HD + dim] = ov;
      if (dim == 0) {
        a.part_ml[base * 2 + 0] = M;
        a.part_ml[base * 2 + 1] = L;
      }
    }
  }
}

// 3-D tensor map over the KV arena viewed as [half 2][row R][64 bf16]: row = one
// 256-B (K or V token) row, strides 256 B (rows) and 128 B (halves); box
// {64, 32, 2} = one block's 16 K + 16 V rows.  Encoded once per arena.
static bool gqa_tensor_map(const KvGeom& kv, int64_t arena_bytes, CUtensorMap* out) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[3] = {64, (cuuint64_t)(arena_bytes / 256), 2};
  const cuuint64_t strides[2] = {256, 128};  // bytes, dims 1 and 2
  const cuuint32_t box[3] = {64, 32, 2};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, kv.arena, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Item map: one CTA per (row, kv_head) item, or `splits` CTAs per item under
// uniform split-KV (merged by attn_combine_kernel).
static void attn_item_map(AttnArgs& a) {
  a.whole_items = a.splits > 1 ? 0 : a.rows * a.KVH;
  a.tail_splits = a.splits > 1 ? a.splits : 1;
}

template <int G>
static cudaError_t launch_gqa(const AttnArgs& a_in, cudaStream_t stream) {
  // 12 stages (96 KB, still 2 CTAs per SM): since the producer streams before
  // the grid-dependency wait, a deeper ring keeps streaming through the
  // consumers' fused-QKV prologue (8B step 6.53 -> 6.49 ms; 8 stages before)
  static const int stages = [] {
    int st = std::max(4, std::min(kAttnMaxStages, attn_env("MS_ATTN_STAGES", 12)));
    return st / 4 * 4;  // stage s is always consumed by warp s % 4
  }();
  AttnArgs a = a_in;
  a.stages = stages;
  static thread_local const char* map_arena = nullptr;
  static thread_local int64_t map_bytes = 0;
  static thread_local CUtensorMap tmap;
  if (a.arena_bytes <= 0) return cudaErrorInvalidValue;
  if (map_arena != a.kv.arena || map_bytes != a.arena_bytes) {
    if (!gqa_tensor_map(a.kv, a.arena_bytes, &tmap)) return cudaErrorInvalidValue;
    map_arena = a.kv.arena;
    map_bytes = a.arena_bytes;
  }
  const size_t smem = 1024 + (size_t)stages * 8192 + 2 * stages * 8 +
                      ((size_t)4 * G * 128 + 8 * G + (size_t)G * 128) * 4;
  static std::atomic<uint64_t> attr{0};
  max_smem_once(attn_gqa_mma_kernel<G>, 200 * 1024, attr);
  attn_item_map(a);
  const int ctas = a.whole_items + (a.rows * a.KVH - a.whole_items) * a.tail_splits;
  cudaError_t e = launch_pdl(attn_gqa_mma_kernel<G>, dim3(ctas), dim3(160), smem, stream, a, tmap);
  if (e != cudaSuccess || a.whole_items == a.rows * a.KVH) return e;
  return launch_pdl(attn_combine_kernel<128>, dim3(a.rows, a.H), dim3(128), 0, stream, a);
}


template <int HD, int G>
static cudaError_t launch_g(const AttnArgs& a_in, cudaStream_t stream) {
  constexpr int BT = 16;
  // warp-per-block consumers (G == 1, HD == 128) need stages % 4 == 0: stage s is
  // then always consumed by warp s % 4, so no warp can wait on a stage two
  // phases ahead of its fill (a parity wait would pass on the stale phase).
  constexpr bool kWpb = G == 1 && HD == 128;
  static const int stages = [] {
    int st = std::max(2, std::min(kAttnMaxStages, attn_env("MS_ATTN_STAGES", kWpb ? 8 : 6)));
    if (kWpb) st = std::max(4, st / 4 * 4);
    return st;
  }();
  static const int ctas_per_sm = attn_env("MS_ATTN_CTAS", 0);
  AttnArgs a = a_in;
  a.stages = stages;
  size_t smem = (size_t)stages * BT * HD * 4 + 2 * stages * 8 + 16 + (size_t)4 * G * (HD + 2) * 4 + (size_t)G * HD * 4;
  if (ctas_per_sm > 0) smem = std::max(smem, (size_t)(220 * 1024) / ctas_per_sm);  // cap residency
  static std::atomic<uint64_t> attr{0};
  max_smem_once(attn_decode_kernel<HD, G, BT>, 200 * 1024, attr);
  attn_item_map(a);
  const int ctas = a.whole_items + (a.rows * a.KVH - a.whole_items) * a.tail_splits;
  cudaError_t e = launch_pdl(attn_decode_kernel<HD, G, BT>, dim3(ctas), dim3(160), smem, stream, a);
  if (e != cudaSuccess || a.whole_items == a.rows * a.KVH) return e;
  return launch_pdl(attn_combine_kernel<HD>, dim3(a.rows, a.H), dim3(HD), 0, stream, a);
}

// MS_ATTN_GQA_MMA=0 (experiments): CUDA-core consumer for GQA as well.
static bool gqa_mma_enabled() {
  static const bool v = attn_env("MS_ATTN_GQA_MMA", 1) != 0;
  return v;
}

template <int HD>
static cudaError_t launch_hd(const AttnArgs& a, cudaStream_t stream) {
  if constexpr (HD == 128) {
    if (gqa_mma_enabled() && a.arena_bytes > 0) {
      switch (a.H / a.KVH) {
        case 2: return launch_gqa<2>(a, stream);
        case 4: return launch_gqa<4>(a, stream);
        case 8: return launch_gqa<8>(a, stream);
        default: break;
      }
    }
  }
  switch (a.H / a.KVH) {
    case 1: return launch_g<HD, 1>(a, stream);
    case 2: return launch_g<HD, 2>(a, stream);
    case 4: return launch_g<HD, 4>(a, stream);
    case 8: return launch_g<HD, 8>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t attn_decode_launch(const AttnArgs& a, cudaStream_t stream) {
  if (a.kv.block_tokens != 16) return cudaErrorInvalidValue;
  if (a.kv.head_dim == 128) return launch_hd<128>(a, stream);
  if (a.kv.head_dim == 64) return launch_hd<64>(a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace ms
