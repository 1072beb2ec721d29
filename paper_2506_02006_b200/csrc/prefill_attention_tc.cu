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
//   warps 0..7    thread = (query row = TMEM lane, half of the keys): masked
//                 online softmax (log2 domain), P (bf16) written to TMEM
//   one lane      O_tile = P V into TMEM (A = P from tensor memory)
//   warps 0..7    O (registers, 64 columns per thread) = O * corr + O_tile
// Software pipelined: S of tile k+1 runs on the tensor cores during tile k's
// softmax, P V of tile k during tile k+1's V transpose, and the loads of tile
// k+2 during both (S and V^T double buffered in TMEM / shared memory).
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kTcTile = 128;           // queries per CTA and keys per KV tile
constexpr uint32_t kOpBytes = 32768;   // one 128 x 128 bf16 operand
constexpr uint32_t kTmemS = 0, kTmemP = 256, kTmemO = 384;  // S double-buffered: [0,128) and [128,256)

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
  uint8_t* sV = sK + 2 * kOpBytes;      // raw V rows [key][dim] of the next tile
  uint8_t* sVt = sV + kOpBytes;         // [2] canonical V^T (dims as rows, keys as k)
  float* sRed = reinterpret_cast<float*>(sVt + 2 * kOpBytes);       // [2][128] row max / sum halves
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 2 * kTcTile);  // [0,1] S(kt) done per buffer, [2] O_tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 4);

  pdl_wait();
  pdl_trigger();
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * kTcTile, n = a.n;
  const int q_last = min(q0 + kTcTile, n) - 1;
  const int n_ktiles = q_last / kTcTile + 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
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
      const float sl = a.scale_log2;  // scores come out of the MMA already in the log2 domain
      const float v[8] = {x0.x * sl, x0.y * sl, x0.z * sl, x0.w * sl, x1.x * sl, x1.y * sl, x1.z * sl, x1.w * sl};
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
  const int64_t head_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();
  // loads: thread = (token row, half of its 16 chunks); one page-id load per thread
  auto load_tile = [&](int kt) {
    const int r = threadIdx.x >> 1, c0 = (threadIdx.x & 1) * 8;
    int t = kt * kTcTile + r;
    if (t > q_last) t = q_last;  // masked anyway; keeps the address valid
    const char* base = a.kv.arena + (int64_t)__ldg(a.pages + (t >> 4)) * a.kv.page_bytes + head_off +
                       (t & 15) * HD * 2 + c0 * 16;
    const uint32_t k_u = smem_u32(sK + (kt & 1) * kOpBytes) + canon(r, c0);
    const uint32_t v_u = smem_u32(sV) + (uint32_t)(r * 256 + c0 * 16);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      tc_cp16(k_u + c * 128, base + c * 16);
      tc_cp16(v_u + c * 16, base + a.kv.head_bytes() + c * 16);
    }
    tc_cp_commit();
  };
  // raw V (landed) -> canonical V^T buffer `buf`: item = (dim pair, key chunk)
  auto transpose_v = [&](int buf) {
    uint8_t* dst = sVt + buf * kOpBytes;
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
      *reinterpret_cast<uint4*>(dst + canon(2 * dp, c)) = make_uint4(lo4[0], lo4[1], lo4[2], lo4[3]);
      *reinterpret_cast<uint4*>(dst + canon(2 * dp + 1, c)) = make_uint4(hi4[0], hi4[1], hi4[2], hi4[3]);
    }
    fence_proxy_async_smem();
  };
  load_tile(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = umma_idesc_bf16(128, 128);
  const uint64_t dQh = umma_desc(smem_u32(sQh), 128u, 2048u), dQl = umma_desc(smem_u32(sQl), 128u, 2048u);
  auto issue_s = [&](int kt) {  // S[kt & 1] = Q_hi K^T + Q_lo K^T
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dK = umma_desc(smem_u32(sK + (kt & 1) * kOpBytes), 128u, 2048u);
        const uint32_t d = tmem + kTmemS + (uint32_t)(kt & 1) * 128u;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          umma_bf16(d, desc_add(dQh, ks * 256u), desc_add(dK, ks * 256u), idesc, ks ? 1u : 0u);
          umma_bf16(d, desc_add(dQl, ks * 256u), desc_add(dK, ks * 256u), idesc, 1u);
        }
        umma_commit(&bar[kt & 1]);
      }
      __syncwarp();
    }
  };
  auto issue_pv = [&](int kt) {  // O_tile = P V(kt)
    if (warp == 0) {
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dVt = umma_desc(smem_u32(sVt + (kt & 1) * kOpBytes), 128u, 2048u);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16_ts(tmem + kTmemO, tmem + kTmemP + ks * 8u, desc_add(dVt, ks * 256u), idesc, ks ? 1u : 0u);
        umma_commit(&bar[2]);
      }
      __syncwarp();
    }
  };

  // softmax state and O: thread = (query row = TMEM lane, half of the key / dim columns)
  const int row = (warp & 3) * 32 + lane;
  const int half = warp >> 2;
  const int qrow = q0 + row;
  float m_run = -INFINITY, l_run = 0.f, prev_corr = 1.f;
  float o[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) o[j] = 0.f;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  auto o_update = [&]() {  // O = O * corr + O_tile (PV done)
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + lane_off + kTmemO + (uint32_t)(half * 64 + c0), v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) o[c0 + j] = o[c0 + j] * prev_corr + __uint_as_float(v[j]);
    }
  };

  // prologue: tile 0 -> V^T[0], S(0) in flight, tile 1 loading
  tc_cp_wait<0>();
  __syncthreads();
  transpose_v(0);
  __syncthreads();
  issue_s(0);
  if (n_ktiles > 1) load_tile(1);

  for (int kt = 0; kt < n_ktiles; ++kt) {
    // 1. previous tile's P V done: fold it into O (frees O_tile, P and V^T[(kt+1) & 1])
    if (kt > 0) {
      mbar_wait(&bar[2], (kt - 1) & 1);
      tc_fence_after();
      o_update();
    }
    // 2. next tile: V^T, then its S on the tensor cores while this tile's softmax runs
    if (kt + 1 < n_ktiles) {
      tc_cp_wait<0>();
      tc_fence_before();
      __syncthreads();
      transpose_v((kt + 1) & 1);
      __syncthreads();
      issue_s(kt + 1);
    }
    // 3. this tile's S
    mbar_wait(&bar[kt & 1], (kt >> 1) & 1);
    tc_fence_after();
    // 4. the K buffer S(kt) read and the raw V buffer are free: load tile kt + 2
    if (kt + 2 < n_ktiles) load_tile(kt + 2);
    // 5. softmax: the two halves of a row (warps w and w + 4) meet through
    // shared memory under a pairwise named barrier; masking only on the
    // diagonal tile (earlier tiles hold keys < q0 <= every query row)
    {
      const int key0 = kt * kTcTile + half * 64;
      const bool diag = kt == n_ktiles - 1;
      const uint32_t scol = tmem + lane_off + kTmemS + (uint32_t)(kt & 1) * 128u + (uint32_t)(half * 64);
      const int pair_bar = 1 + (warp & 3);
      float mx = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(scol + c0, v);
        tmem_ld_wait();
        if (diag) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int key = key0 + c0 + j;
            mx = fmaxf(mx, (key > qrow || key >= n) ? -INFINITY : __uint_as_float(v[j]));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
        }
      }
      sRed[half * kTcTile + row] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
      const float m_new = fmaxf(m_run, fmaxf(sRed[row], sRed[kTcTile + row]));
      const float corr = m_new == -INFINITY ? 1.f : exp2f(m_run - m_new);
      const float msub = m_new == -INFINITY ? 0.f : m_new;
      float psum = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(scol + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float p2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = key0 + c0 + j + e;
            float p = exp2f(__uint_as_float(v[j + e]) - msub);
            if (diag && (key > qrow || key >= n)) p = 0.f;
            p2[e] = p;
            psum += p;
          }
          pk[(c0 + j) >> 1] = pack_bf2(p2[0], p2[1]);
        }
      }
      tmem_st32(tmem + lane_off + kTmemP + (uint32_t)(half * 32), pk);
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // both halves read the maxima
      sRed[half * kTcTile + row] = psum;
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
      l_run = l_run * corr + sRed[row] + sRed[kTcTile + row];
      m_run = m_new;
      prev_corr = corr;
      tmem_st_wait();
    }
    // 6. this tile's P V (P in TMEM)
    tc_fence_before();
    __syncthreads();
    issue_pv(kt);
  }
  mbar_wait(&bar[2], (n_ktiles - 1) & 1);
  tc_fence_after();
  o_update();
  if (qrow < n) {
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
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
  const size_t smem = 7 * (size_t)kOpBytes + 2 * kTcTile * 4 + 4 * 8 + 16;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  return launch_pdl(prefill_attn_tc_kernel, dim3(qtiles, a.H), dim3(256), smem, stream, a);
}

}  // namespace ms
