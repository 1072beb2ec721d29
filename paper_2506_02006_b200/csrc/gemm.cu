// gemm.cu -- the decoder linear layers on 5th-gen tensor cores (tcgen05).
//
// Computes P[s][m][n] = sum_{k in split s} W[n][k] * X[m][k] for one weight
// matrix W [N x K] (BF16, or W4A16 g128 dequantized in the staging path) and a
// token block X [M x K] (BF16), fp32 partials per split-K slice.  "Swap-AB":
// the weight rows are the UMMA M=128 side, the tokens the UMMA N side (16..256),
// so a decode batch of 64 is one N=64 instruction and a prefill of 8k tokens is
// 32 N=256 tiles -- the same kernel serves decode (HBM-bound, split-K over all
// 148 SMs) and prefill (tensor-bound).
//
// Replaces the priced stand-ins `decode_ms_per_layer[tag]` (reference
// proj/src/sim_config.cpp:23-27) and `tokens * prefill_ms_per_token`
// (proj/src/engine.cpp:477-478).  Per-layer precision dispatch (BF16 vs W4) is
// chosen by the caller from the layer table snapshot taken at step launch
// (proj/src/engine.cpp:523-525).
//
// Data movement: every operand chunk is ONE contiguous 1-D bulk async copy
// (cp.async.bulk -> SASS UBLKCP) into shared memory, because both operands are
// pre-packed into the UMMA canonical K-major no-swizzle image:
//   weight chunk (n_tile, kb64)  = 16 KB  [row_group 16][k_chunk 8][row 8][8 bf16]
//   W4 chunk (n_tile, g128)      = 8448 B [j 4][row 128][16 B codes] + 128 bf16 scales
//   activation chunk (m_tile,kb) = TM*128 B, same core-matrix order.
// Weight chunks are addressed through the variant image's page table so a layer
// image can live in any free pages of the KV/weight arena (KV resizing needs no
// contiguity).
//
// Roles (warp-specialised, mbarrier pipelines):
//   warp 0 lane 0 : producer (bulk copies, expect_tx)
//   warp 1 lane 0 : UMMA issuer (tcgen05.mma kind::f16, M=128, N=TM, K=16)
//   W4 only, warps 2..5 : dequantisers (int4 -> bf16(code*scale) -> smem, proxy fence)
//   epilogue (4 warps covering the 4 TMEM lane quadrants): tcgen05.ld -> fp32 partials.
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "kernels.h"

namespace ms {

constexpr int kBf16ChunkBytes = 16384;
constexpr int kW4ChunkBytes = 8448;

__device__ __forceinline__ const uint8_t* chunk_ptr(const GemmWeights& w, int64_t ci, int chunk_bytes) {
  const int64_t c = w.first_chunk + ci;
  const int64_t page = c / w.chunks_per_page;
  const int64_t off = (c - page * w.chunks_per_page) * chunk_bytes;
  return reinterpret_cast<const uint8_t*>(w.pages[page]) + off;
}

template <bool kW4>
__global__ void __launch_bounds__(kW4 ? 192 : 128, 1)
    gemm_kernel(GemmWeights W, const uint16_t* __restrict__ X, int M, int TM, int splits,
                float* __restrict__ out, int stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = W.N, K = W.K;
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // k-steps: BF16 steps are 64 wide, W4 steps are one 128-wide group.
  const int kstep = kW4 ? 128 : 64;
  const int nk_total = K / kstep;
  const int k_begin = (int)((int64_t)nk_total * split / splits);
  const int k_end = (int)((int64_t)nk_total * (split + 1) / splits);
  const int nk = k_end - k_begin;

  const uint32_t b_bytes = (uint32_t)TM * 128u;  // one 64-wide activation chunk
  const uint32_t a_bytes = kW4 ? 32768u : 16384u;
  const uint32_t raw_bytes = kW4 ? (uint32_t)kW4ChunkBytes : 0u;
  const uint32_t stage_bytes = a_bytes + (kW4 ? 2 : 1) * b_bytes + ((raw_bytes + 127u) & ~127u);

  uint8_t* sbase = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (size_t)stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + stages;
  uint64_t* afull = bars + 2 * stages;  // W4: dequantised A ready
  uint64_t* accum = bars + 3 * stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * stages + 1);

  auto sA = [&](int s) { return sbase + (size_t)s * stage_bytes; };
  auto sB = [&](int s) { return sbase + (size_t)s * stage_bytes + a_bytes; };
  auto sRaw = [&](int s) { return sbase + (size_t)s * stage_bytes + a_bytes + 2 * b_bytes; };

  const uint32_t tm_cols = TM <= 32 ? 32u : TM <= 64 ? 64u : TM <= 128 ? 128u : 256u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&afull[s], 128);
    }
    mbar_init(accum, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(tmem_slot, tm_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_slot;

  const int64_t kb_per_row = K / 64;  // activation chunks per m_tile
  const uint8_t* xbase = reinterpret_cast<const uint8_t*>(X) + (size_t)m_tile * kb_per_row * b_bytes;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer
      for (int it = 0; it < nk; ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
        const int ks = k_begin + it;
        if (kW4) {
          mbar_expect_tx(&full[s], raw_bytes + 2 * b_bytes);
          bulk_g2s(sRaw(s), chunk_ptr(W, (int64_t)n_tile * nk_total + ks, kW4ChunkBytes), raw_bytes, &full[s]);
          bulk_g2s(sB(s), xbase + (size_t)(2 * ks) * b_bytes, 2 * b_bytes, &full[s]);
        } else {
          mbar_expect_tx(&full[s], a_bytes + b_bytes);
          bulk_g2s(sA(s), chunk_ptr(W, (int64_t)n_tile * nk_total + ks, kBf16ChunkBytes), a_bytes, &full[s]);
          bulk_g2s(sB(s), xbase + (size_t)ks * b_bytes, b_bytes, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- UMMA issuer
      const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)TM);
      for (int it = 0; it < nk; ++it) {
        const int s = it % stages;
        const uint32_t ph = (it / stages) & 1;
        mbar_wait(&full[s], ph);
        if (kW4) mbar_wait(&afull[s], ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA(s)), b0 = smem_u32(sB(s));
#pragma unroll
        for (int sub = 0; sub < (kW4 ? 2 : 1); ++sub) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t da = umma_desc(a0 + sub * 16384u + k * 256u, 128u, 1024u);
            const uint64_t db = umma_desc(b0 + sub * b_bytes + k * 256u, 128u, 1024u);
            umma_bf16(tmem_d, da, db, idesc, (it | sub | k) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(accum);
    }
  } else if (kW4) {
    // ---------------- dequantisers: thread t owns weight row t of the tile
    const int t = threadIdx.x - 64;
    const int rg = t >> 3, r = t & 7;
    for (int it = 0; it < nk; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      const uint8_t* raw = sRaw(s);
      const float sc = bf2f(*reinterpret_cast<const uint16_t*>(raw + 8192 + 2 * t));
      uint8_t* a = sA(s);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 q = *reinterpret_cast<const uint4*>(raw + (j * 128 + t) * 16);
        const uint32_t words[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int kk = j * 32 + w * 8;  // element offset within the 128-group
          const int sub = kk >> 6, c = (kk & 63) >> 3;
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c0 = (int)((words[w] >> (8 * e)) & 0xFu) - 8;
            const int c1 = (int)((words[w] >> (8 * e + 4)) & 0xFu) - 8;
            o[e] = pack_bf2((float)c0 * sc, (float)c1 * sc);
          }
          *reinterpret_cast<uint4*>(a + sub * 16384 + ((rg * 8 + c) * 8 + r) * 16) =
              make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&afull[s]);
    }
  }

  // ---------------- epilogue: TMEM -> fp32 partials [split][m][n]
  __syncwarp();
  const bool epi = kW4 ? (warp >= 2) : true;
  if (epi) {
    mbar_wait(accum, 0);
    tc_fence_after();
    const int quad = warp & 3;
    const int n = n_tile * 128 + quad * 32 + lane;
    float* o = out + (size_t)split * M * N;
    for (int c0 = 0; c0 < TM; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem_d + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0, v);
      tmem_ld_wait();
      if (nk == 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = m_tile * TM + c0 + j;
        if (m < M) o[(size_t)m * N + n] = __uint_as_float(v[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_d, tm_cols);
}

static int pick_stages(bool w4, int TM, size_t* smem_out) {
  const size_t b = (size_t)TM * 128;
  const size_t stage = w4 ? (32768 + 2 * b + 8448 + 127) / 128 * 128 : 16384 + b;
  const size_t budget = w4 ? 220 * 1024 : (TM <= 64 ? 110 * 1024 : 200 * 1024);
  int st = (int)(budget / stage);
  if (st > 8) st = 8;
  if (st < 2) st = 2;
  *smem_out = st * stage + (3 * st + 2) * 8 + 64;
  return st;
}

int gemm_pick_splits(int n_tiles, int m_tiles, int nk, int num_sms, int ctas_per_sm) {
  const int slots = num_sms * ctas_per_sm;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 16 && s <= nk; ++s) {
    const int units = n_tiles * m_tiles * s;
    const int waves = (units + slots - 1) / slots;
    const int per = (nk + s - 1) / s;
    // per-unit fixed cost ~ 2 k-steps (pipeline fill + epilogue)
    const double cost = (double)waves * (per + 2) + 0.02 * s;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

cudaError_t gemm_launch(const GemmWeights& w, bool w4, const uint16_t* x, int M, int TM, int splits, float* out,
                        cudaStream_t stream) {
  size_t smem = 0;
  const int stages = pick_stages(w4, TM, &smem);
  dim3 grid(w.N / 128, (M + TM - 1) / TM, splits);
  if (w4) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr = true;
    }
    gemm_kernel<true><<<grid, 192, smem, stream>>>(w, x, M, TM, splits, out, stages);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr = true;
    }
    gemm_kernel<false><<<grid, 128, smem, stream>>>(w, x, M, TM, splits, out, stages);
  }
  return cudaGetLastError();
}

int gemm_ctas_per_sm(bool w4, int TM) {
  size_t smem = 0;
  pick_stages(w4, TM, &smem);
  int per = (int)((228 * 1024) / (smem + 1024));
  return per < 1 ? 1 : per;
}

}  // namespace ms
