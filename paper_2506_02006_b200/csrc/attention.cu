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
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

constexpr int kAttnStages = 6;

template <int HD, int G, int BT>
__global__ void __launch_bounds__(160) attn_decode_kernel(AttnArgs a) {
  constexpr int VEC = HD / 32;
  constexpr int TPW = BT / 4;  // tokens per consumer warp per block
  constexpr uint32_t kStageBytes = (uint32_t)BT * HD * 2 * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAttnStages * kStageBytes);
  uint64_t* empty = full + kAttnStages;
  float* scratch = reinterpret_cast<float*>(empty + kAttnStages);  // [4][G][HD] acc + [4][G][2] m,l

  pdl_wait();
  pdl_trigger();
  const int kvh = blockIdx.x, row = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctx = a.ctx_len[row];
  const int nb = (ctx + BT - 1) / BT;
  const int b0 = (int)((int64_t)nb * split / a.splits), b1 = (int)((int64_t)nb * (split + 1) / a.splits);
  const int prow = a.page_row ? a.page_row[row] : row;
  const int32_t* ptab = a.pages + (size_t)prow * a.page_stride;
  const int64_t kv_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  float m[G], l[G], acc[G][VEC];
  if (warp == 4) {
    if (lane == 0) {
      for (int it = 0; it < b1 - b0; ++it) {
        const int s = it % kAttnStages;
        if (it >= kAttnStages) mbar_wait(&empty[s], ((it / kAttnStages) & 1) ^ 1);
        const char* src = a.kv.arena + (int64_t)ptab[b0 + it] * a.kv.page_bytes + kv_off;
        mbar_expect_tx(&full[s], kStageBytes);
        bulk_g2s(smem + (size_t)s * kStageBytes, src, kStageBytes, &full[s]);
      }
    }
  } else {
    float qv[G][VEC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* qp = a.q + ((size_t)row * a.H + kvh * G + g) * HD + lane * VEC;
#pragma unroll
      for (int i = 0; i < VEC; ++i) qv[g][i] = qp[i] * a.scale_log2;
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
      if (a.splits == 1) {
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
  float M = -INFINITY;
  for (int s = 0; s < a.splits; ++s) M = fmaxf(M, a.part_ml[(((size_t)s * a.rows + row) * a.H + h) * 2]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int s = 0; s < a.splits; ++s) {
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

template <int HD, int G>
static cudaError_t launch_g(const AttnArgs& a, cudaStream_t stream) {
  constexpr int BT = 16;
  const size_t smem = (size_t)kAttnStages * BT * HD * 4 + 2 * kAttnStages * 8 + (size_t)4 * G * (HD + 2) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel<HD, G, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(a.KVH, a.rows, a.splits);
  cudaError_t e = launch_pdl(attn_decode_kernel<HD, G, BT>, grid, dim3(160), smem, stream, a);
  if (e != cudaSuccess || a.splits == 1) return e;
  return launch_pdl(attn_combine_kernel<HD>, dim3(a.rows, a.H), dim3(HD), 0, stream, a);
}

template <int HD>
static cudaError_t launch_hd(const AttnArgs& a, cudaStream_t stream) {
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
