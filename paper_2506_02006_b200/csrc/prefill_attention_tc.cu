// prefill_attention_tc.cu -- causal prefill attention on the 5th-gen tensor
// cores (tcgen05 + TMEM), head_dim 128.
//
// Part of `start_prefill` (reference proj/src/engine.cpp:472-485, priced as
// tokens * prefill_ms_per_token at :477-478): the long-prompt prefill of
// BASELINE.json configs[3] (Llama-2-13B, 8k tokens) spends ~40% of its time in
// attention.  prefill_attention.cu does it with mma.sync (m16n8k16); this
// kernel issues tcgen05.mma with 128x128 tiles.
//
// CTA = (128-query tile, query head), 8 warps.  Per 128-key tile of the
// sequence's paged KV:
//   all threads   cp.async the K rows into the UMMA canonical K-major layout
//                 (double buffered) and the V rows as they are; transpose V
//                 into a canonical V^T (keys = K dimension) in shared memory
//   one lane      S = Q_hi K^T + Q_lo K^T into TMEM (16 MMAs M128 N128 K16;
//                 q = hi + lo bf16 keeps fp32-level score accuracy, as the
//                 mma.sync kernel and the decode paths do)
//   warps 0..3    thread = query row = TMEM lane: masked online softmax
//                 (log2 domain) over the 128 scores, P (bf16) written to TMEM
//   one lane      O_tile = P V into TMEM (A = P from tensor memory)
//   warps 0..7    O (registers, 64 columns per thread) = O * corr + O_tile
// The phases run in order inside a CTA; the next tile's loads overlap them.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kTcTile = 128;           // queries per CTA and keys per KV tile
constexpr uint32_t kOpBytes = 32768;   // one 128 x 128 bf16 operand
constexpr uint32_t kTmemS = 0, kTmemP = 128, kTmemO = 256;

__device__ __forceinline__ void tc_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void tc_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tc_cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// byte offset of the 16-B chunk (row r, k-chunk c) of a [128 rows][128 k] canonical K-major operand
__device__ __forceinline__ uint32_t canon(int r, int c) {
  return (uint32_t)((((r >> 3) * 16 + c) << 7) + ((r & 7) << 4));
}

}  // namespace

__global__ void __launch_bounds__(256, 1) prefill_attn_tc_kernel(PrefillAttnArgs a) {
  constexpr int HD = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQh = smem;
  uint8_t* sQl = sQh + kOpBytes;
  uint8_t* sK = sQl + kOpBytes;         // [2] canonical K tiles
  uint8_t* sV = sK + 2 * kOpBytes;      // raw V rows [key][dim]
  uint8_t* sVt = sV + kOpBytes;         // canonical V^T (dims as rows, keys as k)
  float* sCorr = reinterpret_cast<float*>(sVt + kOpBytes);  // [128]
  float* sL = sCorr + kTcTile;                               // [128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sL + kTcTile); // [2]: S done, O_tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  int32_t* sPage = reinterpret_cast<int32_t*>(tmem_slot + 4);

  pdl_wait();
  pdl_trigger();
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * kTcTile, n = a.n;
  const int q_last = min(q0 + kTcTile, n) - 1;
  const int n_ktiles = q_last / kTcTile + 1;
  for (int b = threadIdx.x; b <= q_last / 16; b += blockDim.x) sPage[b] = a.pages[b];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);

  // ---- Q tile: fp32 -> (hi, lo) bf16, canonical layout
  for (int idx = threadIdx.x; idx < kTcTile * 16; idx += blockDim.x) {
    const int r = idx >> 4, c = idx & 15;
    const int q = q0 + r;
    uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
    if (q < n) {
      const float4* src = reinterpret_cast<const float4*>(a.q + ((size_t)q * a.H + h) * HD + c * 8);
      const float4 x0 = src[0], x1 = src[1];
      const float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint16_t h0 = f2bf(v[2 * e]), h1 = f2bf(v[2 * e + 1]);
        hi[e] = (uint32_t)h0 | ((uint32_t)h1 << 16);
        lo[e] = pack_bf2(v[2 * e] - bf2f(h0), v[2 * e + 1] - bf2f(h1));
      }
    }
    *reinterpret_cast<uint4*>(sQh + canon(r, c)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(sQl + canon(r, c)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
  __syncthreads();  // sPage, barriers
  const int64_t head_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();
  auto load_tile = [&](int kt) {
    const uint32_t k_u = smem_u32(sK + (kt & 1) * kOpBytes), v_u = smem_u32(sV);
    for (int idx = threadIdx.x; idx < kTcTile * 16; idx += blockDim.x) {
      const int r = idx >> 4, c = idx & 15;
      int t = kt * kTcTile + r;
      if (t > q_last) t = q_last;  // masked anyway; keeps the address valid
      const char* base = a.kv.arena + (int64_t)sPage[t >> 4] * a.kv.page_bytes + head_off + (t & 15) * HD * 2 + c * 16;
      tc_cp16(k_u + canon(r, c), base);
      tc_cp16(v_u + (uint32_t)(r * 256 + c * 16), base + a.kv.head_bytes());
    }
    tc_cp_commit();
  };
  load_tile(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = umma_idesc_bf16(128, 128);
  const uint64_t dQh = umma_desc(smem_u32(sQh), 128u, 2048u), dQl = umma_desc(smem_u32(sQl), 128u, 2048u);
  const uint64_t dVt = umma_desc(smem_u32(sVt), 128u, 2048u);

  // softmax state (warps 0..3: thread = query row) and O (all warps: 64 columns of one row)
  const int row = (warp & 3) * 32 + lane;
  const int half = warp >> 2;
  const int qrow = q0 + row;
  float m_run = -INFINITY, l_run = 0.f;
  float o[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) o[j] = 0.f;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;

  for (int kt = 0; kt < n_ktiles; ++kt) {
    // (a) tile kt landed (K canonical + raw V)
    tc_cp_wait<0>();
    __syncthreads();
    // (b) V -> V^T canonical: item = (dim pair, key chunk): 8 keys x 2 dims
    for (int it = threadIdx.x; it < 64 * 16; it += blockDim.x) {
      const int dp = it & 63, c = it >> 6;
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = *reinterpret_cast<const uint32_t*>(sV + (c * 8 + j) * 256 + dp * 4);
      uint32_t lo4[4], hi4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo4[j] = __byte_perm(w[2 * j], w[2 * j + 1], 0x5410);  // dim 2dp: keys 2j, 2j+1
        hi4[j] = __byte_perm(w[2 * j], w[2 * j + 1], 0x7632);  // dim 2dp+1
      }
      *reinterpret_cast<uint4*>(sVt + canon(2 * dp, c)) = make_uint4(lo4[0], lo4[1], lo4[2], lo4[3]);
      *reinterpret_cast<uint4*>(sVt + canon(2 * dp + 1, c)) = make_uint4(hi4[0], hi4[1], hi4[2], hi4[3]);
    }
    fence_proxy_async_smem();
    __syncthreads();
    // (c) next tile's loads (raw V buffer and the other K buffer are free)
    if (kt + 1 < n_ktiles) load_tile(kt + 1);
    // (d) S = Q K^T (hi + lo)
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dK = umma_desc(smem_u32(sK + (kt & 1) * kOpBytes), 128u, 2048u);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          umma_bf16(tmem + kTmemS, desc_add(dQh, ks * 256u), desc_add(dK, ks * 256u), idesc, ks ? 1u : 0u);
          umma_bf16(tmem + kTmemS, desc_add(dQl, ks * 256u), desc_add(dK, ks * 256u), idesc, 1u);
        }
        umma_commit(&bar[0]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[0], kt & 1);
    tc_fence_after();
    // (e) softmax: warps 0..3, thread = row
    if (warp < 4) {
      const int key0 = kt * kTcTile;
      float mx = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < kTcTile; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + kTmemS + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int key = key0 + c0 + j;
          const float s = (key > qrow || key >= n) ? -INFINITY : __uint_as_float(v[j]) * a.scale_log2;
          mx = fmaxf(mx, s);
        }
      }
      const float m_new = fmaxf(m_run, mx);
      const float corr = m_new == -INFINITY ? 1.f : exp2f(m_run - m_new);
      float psum = 0.f;
#pragma unroll
      for (int c1 = 0; c1 < kTcTile; c1 += 64) {
        uint32_t pk[32];
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + lane_off + kTmemS + c1 + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            float p2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int key = key0 + c1 + c0 + j + e;
              const float s = __uint_as_float(v[j + e]) * a.scale_log2;
              p2[e] = (key > qrow || key >= n || m_new == -INFINITY) ? 0.f : exp2f(s - m_new);
              psum += p2[e];
            }
            pk[(c0 + j) >> 1] = pack_bf2(p2[0], p2[1]);
          }
        }
        tmem_st32(tmem + lane_off + kTmemP + (uint32_t)(c1 >> 1), pk);
      }
      tmem_st_wait();
      l_run = l_run * corr + psum;
      m_run = m_new;
      sCorr[row] = corr;
    }
    tc_fence_before();
    __syncthreads();
    // (f) O_tile = P V
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16_ts(tmem + kTmemO, tmem + kTmemP + ks * 8u, desc_add(dVt, ks * 256u), idesc, ks ? 1u : 0u);
        umma_commit(&bar[1]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[1], kt & 1);
    tc_fence_after();
    // (g) O = O * corr + O_tile (64 columns of this thread's row)
    {
      const float cr = sCorr[row];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + lane_off + kTmemO + (uint32_t)(half * 64 + c0), v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) o[c0 + j] = o[c0 + j] * cr + __uint_as_float(v[j]);
      }
    }
    tc_fence_before();
    __syncthreads();  // S / P / O_tile and sCorr are rewritten by the next tile
  }
  if (warp < 4) sL[row] = l_run;
  __syncthreads();
  if (qrow < n) {
    const float inv = sL[row] > 0.f ? 1.f / sL[row] : 0.f;
    const int K = a.H * HD;
#pragma unroll
    for (int j = 0; j < 64; j += 2) {
      const int dim = half * 64 + j;
      const uint32_t v = pack_bf2(o[j] * inv, o[j + 1] * inv);
      const size_t off = a.TM > 0 ? act_off(qrow, h * HD + dim, K, a.TM) : (size_t)qrow * K + h * HD + dim;
      *reinterpret_cast<uint32_t*>(a.out + off) = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

cudaError_t prefill_attn_tc_launch(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.kv.block_tokens != 16 || a.kv.head_dim != 128) return cudaErrorNotSupported;
  const int qtiles = (a.n + kTcTile - 1) / kTcTile;
  const size_t smem = 6 * (size_t)kOpBytes + 2 * kTcTile * 4 + 2 * 8 + 16 + (size_t)((a.n + 15) / 16) * 4 + 16;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  return launch_pdl(prefill_attn_tc_kernel, dim3(qtiles, a.H), dim3(256), smem, stream, a);
}

}  // namespace ms
