// prefill_attention_tc.cu -- causal prefill attention on the 5th-gen tensor
// cores (tcgen05 + TMEM), head_dim 128.
//
// Part of `start_prefill` (reference proj/src/engine.cpp:472-485, priced as
// tokens * prefill_ms_per_token at :477-478): the long-prompt prefill of
// BASELINE.json configs[3] (Llama-2-13B, 8k tokens) spends a large share of its
// time in attention.  prefill_attention.cu does it with mma.sync (m16n8k16);
// this kernel issues tcgen05.mma with 128x128 tiles.
//
// CTA = (256-query tile pair, query head), 11 warps, warp specialised, two
// independent softmax streams ("ping-pong"): stream A = queries q0..q0+127,
// stream B = q0+128..q0+255, sharing every K / V tile the CTA loads.
//   warps 8, 10  TMA producers for K and for V: per 128-key tile, 8 paged KV
//            blocks x 2 column halves, SWIZZLE_128B boxes {64 dims, 16 keys}
//            from a 2-D tensor map over the arena (rows of 256 B).  That image
//            is directly a K-major SW128 operand for K (S = Q K^T) and an
//            MN-major SW128 operand for V (O += P V): no transpose, no
//            per-thread copies.  K has 3 buffers (freed when both streams'
//            S(kt) completed), V 2 (freed when both PV(kt) completed).
//   warp 9   MMA issuer (one elected lane of a converged warp), order
//            S_A(0) S_B(0) | PV_A(kt) S_A(kt+1) PV_B(kt) S_B(kt+1) | ...:
//            while the softmax of one stream runs, the tensor cores work on
//            the other stream's tile, so neither the MMAs nor the softmax's
//            exp2 rate wait on the other's latency.  S_X(kt) = bf16(q) K^T (8
//            MMAs M128 N128 K16); O_X += P_X(kt) V (8
//            MMAs, A = P read from TMEM, B = V MN-major).  tcgen05 MMAs of one
//            thread execute in issue order, so S_X(kt+1) (issued after
//            PV_X(kt)) overwrites P_X(kt) only after PV_X(kt) read it, and the
//            commit that signals S_X(kt+1) also covers PV_X(kt).
//   warps 0-3 / 4-7  softmax of stream A / B: thread = one query row (TMEM
//            lane), all 128 keys of a tile in registers (one TMEM read).
//            Online softmax in the log2 domain (the fp32 scores scaled by
//            log2(e)/sqrt(hd) inside the exp2 FMA) with lazy rescaling: the
//            running max moves only when a tile's max exceeds it by more than
//            2^8, so O (in TMEM; complete up to PV_X(kt-1) when S_X(kt) lands)
//            is rescaled a handful of times per row instead of every tile.  P
//            (bf16) is written over its own S columns.
// TMEM: S/P of A [0,128), S/P of B [128,256), O_A [256,384), O_B [384,512).
// CTAs run head-major, longest query tiles first, so the K/V of the heads in
// flight stay in L2.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

#ifdef MS_PATTN_TL
// (experiment builds, -DMS_PATTN_TL) %globaltimer stamps of CTA 0:
// [event][kt] events 0/1 S_A/S_B issued, 2/3 PV_A/PV_B issued, 4/5 softmax A/B
// got S, 6/7 softmax A/B wrote P
__device__ unsigned long long g_pattn_tl[8][128];
__device__ __forceinline__ void pattn_stamp(int ev, int kt) {
  if (blockIdx.x == 0 && kt < 128) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_pattn_tl[ev][kt] = t;
  }
}
#else
__device__ __forceinline__ void pattn_stamp(int, int) {}
#endif

namespace {

constexpr int kTcTile = 128;           // queries per softmax stream and keys per KV tile (2 streams per CTA)
constexpr uint32_t kOpBytes = 32768;   // one 128 x 128 bf16 operand
constexpr uint32_t kHalfBytes = 16384; // one 64-column half of it (SW128 image)
constexpr int kKStages = 3, kVStages = 2;              // K / V tile buffers
constexpr uint32_t kTmemS = 0, kTmemO = 256;           // S/P of stream X at X*128, O of stream X at 256 + X*128
constexpr int kBars = kKStages * 2 + kVStages * 2 + 2 * 3;  // + per stream: sfull, pfull, ofinal
constexpr uint32_t kCtrlBytes = kBars * 8 + 16;        // barriers, TMEM slot
constexpr int kThreads = 352;
constexpr float kRescaleLog2 = 8.f;    // lazy rescale threshold (log2 domain)

// byte offset of the 16-B chunk (row r, k-chunk c) of a [128 rows][128 k] canonical
// K-major no-swizzle operand (core matrices 8 rows x 16 B; LBO 128, SBO 2048)
__device__ __forceinline__ uint32_t canon(int r, int c) {
  return (uint32_t)((((r >> 3) * 16 + c) << 7) + ((r & 7) << 4));
}
// SWIZZLE_128B shared-memory descriptor (layout type 2 at bits [61,64))
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return umma_desc(addr, lbo, sbo) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32p(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_bf2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_tc_kernel(PrefillAttnArgs a, const __grid_constant__ CUtensorMap tmap) {
  constexpr int HD = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* kfull = bar;                 // [kKStages]
  uint64_t* kempty = kfull + kKStages;   // [kKStages] both streams' S(kt) done
  uint64_t* vfull = kempty + kKStages;   // [kVStages]
  uint64_t* vempty = vfull + kVStages;   // [kVStages] both streams' PV(kt) done
  uint64_t* sfull = vempty + kVStages;   // [2] S_X(kt) in TMEM (and PV_X(kt-1) done)
  uint64_t* pfull = sfull + 2;           // [2] P_X(kt) written over S_X(kt) (4 softmax warps)
  uint64_t* ofinal = pfull + 2;          // [2] every MMA of stream X done (single phase)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + kBars);
  // operands: 1024-B aligned (SW128 atoms)
  uint8_t* ops = smem_raw + (((smem_u32(smem_raw) + kCtrlBytes + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint8_t* sQ = ops;                          // [2 streams] canonical no-swizzle, written by the softmax warps
  uint8_t* sK = sQ + 2 * kOpBytes;            // [kKStages] SW128 images [dim half][key][128 B]
  uint8_t* sV = sK + kKStages * kOpBytes;     // [kVStages] same

  // head-major, longest query tile pairs of a head first
  const int qpairs = (a.n + 2 * kTcTile - 1) / (2 * kTcTile);
  const int h = (int)blockIdx.x / qpairs;
  const int qp = qpairs - 1 - ((int)blockIdx.x - h * qpairs);
  const int kvh = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qp * 2 * kTcTile, n = a.n;
  const int rowsA = min(kTcTile, n - q0), rowsB = max(0, min(kTcTile, n - q0 - kTcTile));
  const int nkA = (q0 + rowsA - 1) / kTcTile + 1;                  // key tiles of stream A
  const int nkB = rowsB > 0 ? (q0 + kTcTile + rowsB - 1) / kTcTile + 1 : 0;
  const int n_ktiles = max(nkA, nkB);
  const int q_last = q0 + rowsA + rowsB - 1;
  const int last_blk = q_last >> 4;
  const int64_t head_row = (a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes()) >> 8;
  const int64_t rows_per_page = a.kv.page_bytes >> 8;
  const int v_rows = (int)(a.kv.head_bytes() >> 8);

  pdl_wait();
  pdl_trigger();
  // K or V of tile kt (whole producer warp): lane j < 8 holds the arena row of
  // the tile's block j (clamped to the last block: keys past the row are
  // masked) and issues its two column-half boxes.  The page ids of a tile are
  // fetched one tile ahead, eight in parallel.
  auto tile_row = [&](int kt) {
    const int blk = min(kt * 8 + (lane & 7), last_blk);
    return (int)(__ldg(a.pages + blk) * rows_per_page + head_row);
  };
  auto load = [&](int kt, bool is_v, int row) {
    const int s = is_v ? kt % kVStages : kt % kKStages;
    uint64_t* fb = is_v ? &vfull[s] : &kfull[s];
    const uint32_t dst = smem_u32((is_v ? sV : sK) + s * kOpBytes) + (uint32_t)lane * 2048u;
    if (lane == 0) mbar_expect_tx(fb, kOpBytes);
    __syncwarp();
    if (lane < 8) {
      const int r = row + (is_v ? v_rows : 0);
      tma2d(dst, &tmap, 0, r, fb);
      tma2d(dst + kHalfBytes, &tmap, 64, r, fb);
    }
  };
  int row_k = 0, row_v = 0;  // producers: page rows of the next K / V tile to load
  if (warp == 8) {
    if (lane == 0) {
      for (int i = 0; i < kBars; ++i) mbar_init(&bar[i], (&bar[i] >= pfull && &bar[i] < pfull + 2) ? 4 : 1);
      fence_mbar_init();
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    __syncwarp();
    for (int kt = 0; kt < min(kKStages, n_ktiles); ++kt) {
      const int row = tile_row(kt);
      load(kt, false, row);
      if (kt < kVStages) load(kt, true, row);
    }
    if (n_ktiles > kKStages) row_k = tile_row(kKStages);
  }
  if (warp == 10 && n_ktiles > kVStages) row_v = tile_row(kVStages);
  if (warp == 9) tmem_alloc<512>(tmem_slot);

  // ---- Q tiles of both streams (softmax warps): fp32 -> bf16, canonical
  // layout; rows past the sequence are zero
  if (warp < 8) {
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      float4 x[8][2];
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int idx = threadIdx.x + (half * 8 + it) * 256, r = idx >> 4, c = idx & 15;
        const int q = min(q0 + r, n - 1);
        const float4* src = reinterpret_cast<const float4*>(a.q + ((size_t)q * a.H + h) * HD + c * 8);
        x[it][0] = __ldg(src);
        x[it][1] = __ldg(src + 1);
      }
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int idx = threadIdx.x + (half * 8 + it) * 256, r = idx >> 4, c = idx & 15;
        uint32_t w[4] = {0, 0, 0, 0};
        if (q0 + r < n) {
          const float4 x0 = x[it][0], x1 = x[it][1];
          w[0] = pack_bf2(x0.x, x0.y);
          w[1] = pack_bf2(x0.z, x0.w);
          w[2] = pack_bf2(x1.x, x1.y);
          w[3] = pack_bf2(x1.z, x1.w);
        }
        *reinterpret_cast<uint4*>(sQ + (r >> 7) * kOpBytes + canon(r & 127, c)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------ K producer
    // K(kt) as soon as both streams' S(kt - kKStages) released its buffer
    for (int kt = kKStages; kt < n_ktiles; ++kt) {
      const int rw = row_k;
      if (kt + 1 < n_ktiles) row_k = tile_row(kt + 1);
      mbar_wait(&kempty[kt % kKStages], ((kt / kKStages) - 1) & 1);
      load(kt, false, rw);
    }
    __syncwarp();
  } else if (warp == 10) {
    // ------------------------------------------------------ V producer
    // V(kt) as soon as both streams' PV(kt - kVStages) released its buffer
    for (int kt = kVStages; kt < n_ktiles; ++kt) {
      const int rw = row_v;
      if (kt + 1 < n_ktiles) row_v = tile_row(kt + 1);
      mbar_wait(&vempty[kt % kVStages], ((kt / kVStages) - 1) & 1);
      load(kt, true, rw);
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc = umma_idesc_bf16(128, 128);
    const uint32_t idesc_pv = idesc | (1u << 16);  // B (= V) MN-major
    auto issue_s = [&](int X, int kt) {  // S_X(kt) = Q_X K(kt)^T into stream X's S columns
      const int s = kt % kKStages;
      if (elect_one()) {
        const uint64_t dQ = umma_desc(smem_u32(sQ + X * kOpBytes), 128u, 2048u);
        const uint64_t dK = desc_sw128(smem_u32(sK + s * kOpBytes), 16u, 1024u);
        const uint32_t d = tmem + kTmemS + (uint32_t)X * 128u;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t dk = desc_add(dK, (uint32_t)(ks >> 2) * kHalfBytes + (uint32_t)(ks & 3) * 32u);
          umma_bf16(d, desc_add(dQ, ks * 256u), dk, idesc, ks ? 1u : 0u);
        }
        umma_commit(&sfull[X]);
        pattn_stamp(X, kt);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int X, int kt) {  // O_X += P_X(kt) V(kt)
      const int sv = kt % kVStages;
      if (elect_one()) {
        const uint64_t dV = desc_sw128(smem_u32(sV + sv * kOpBytes), kHalfBytes, 1024u);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16_ts(tmem + kTmemO + (uint32_t)X * 128u, tmem + kTmemS + (uint32_t)X * 128u + ks * 8u,
                       desc_add(dV, ks * 2048u), idesc_pv, (kt | ks) ? 1u : 0u);
        const int nk = X == 0 ? nkA : nkB;
        if (kt == nk - 1) umma_commit(&ofinal[X]);
        pattn_stamp(2 + X, kt);
      }
      __syncwarp();
    };
    mbar_wait(&kfull[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    if (nkB > 0) issue_s(1, 0);
    if (elect_one()) umma_commit(&kempty[0]);
    __syncwarp();
    for (int kt = 0; kt < n_ktiles; ++kt) {
      const int sv = kt % kVStages;
      const bool a_on = kt < nkA, b_on = kt < nkB;
      const bool a_next = kt + 1 < nkA, b_next = kt + 1 < nkB;
      mbar_wait(&vfull[sv], (kt / kVStages) & 1);
      if (kt == n_ktiles - 1) {
        // keys past the sequence in the last tile: zero their V rows -- P is
        // 0 there, but the arena bytes past the sequence are arbitrary and
        // 0 * NaN would not be 0
        const int r0 = q_last + 1 - kt * kTcTile;
        if (r0 < kTcTile) {
          uint8_t* vb = sV + sv * kOpBytes;
          for (int i = lane; i < (kTcTile - r0) * 16; i += 32) {
            const int r = r0 + (i >> 4), c = i & 15;
            *reinterpret_cast<uint4*>(vb + (c >> 3) * kHalfBytes + r * 128 + (c & 7) * 16) = make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async_smem();
          __syncwarp();
        }
      }
      if (a_on) {
        mbar_wait(&pfull[0], kt & 1);
        tc_fence_after();
        issue_pv(0, kt);
      }
      if (a_next || b_next) {
        mbar_wait(&kfull[(kt + 1) % kKStages], ((kt + 1) / kKStages) & 1);
        tc_fence_after();
      }
      if (a_next) issue_s(0, kt + 1);
      if (b_on) {
        mbar_wait(&pfull[1], kt & 1);
        tc_fence_after();
        issue_pv(1, kt);
      }
      if (elect_one()) umma_commit(&vempty[sv]);  // both PV(kt) issued before: V(kt) free once they finish
      __syncwarp();
      if (b_next) issue_s(1, kt + 1);
      if (a_next || b_next) {
        if (elect_one()) umma_commit(&kempty[(kt + 1) % kKStages]);
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------- softmax
    const int X = warp >> 2;                       // stream
    const int row = (warp & 3) * 32 + lane;        // TMEM lane = query row of the stream's tile
    const int qrow = q0 + X * kTcTile + row;
    const int nk = X == 0 ? nkA : nkB;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t scol = tmem + lane_off + kTmemS + (uint32_t)X * 128u;
    const uint32_t ocol = tmem + lane_off + kTmemO + (uint32_t)X * 128u;
    const float sl = a.scale_log2;  // raw q.k scores -> log2 domain
    float m_run = -INFINITY, l_run = 0.f;
    for (int kt = 0; kt < nk; ++kt) {
      mbar_wait(&sfull[X], kt & 1);
      tc_fence_after();
      if (lane == 0 && (warp & 3) == 0) pattn_stamp(4 + X, kt);
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(scol + c * 32, v + c * 32);
      tmem_ld_wait();
      if (kt == nk - 1) {  // the stream's diagonal tile (earlier tiles hold keys < its first row)
        const int key0 = kt * kTcTile;
#pragma unroll
        for (int j = 0; j < 128; ++j)
          if (key0 + j > qrow || key0 + j >= n) v[j] = __float_as_uint(-INFINITY);
      }
      // One pass while the running max holds: exp2 against the current max
      // (lazy rescaling keeps it unless a tile's max exceeds it by 2^8),
      // tracking this tile's max alongside.  A row whose max moved (the first
      // tile always) takes the second pass below with the new max, reloading
      // its scores from TMEM (P has not been stored yet).
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (kt > 0) {
        const float msub = m_run;  // finite after the first tile
#pragma unroll
        for (int j = 0; j < 128; j += 2) {
          const float s0 = __uint_as_float(v[j]), s1 = __uint_as_float(v[j + 1]);
          m4[(j >> 1) & 3] = fmaxf(m4[(j >> 1) & 3], fmaxf(s0, s1));
          const float p0 = ex2(fmaf(s0, sl, -msub));
          const float p1 = ex2(fmaf(s1, sl, -msub));
          ps[(j >> 1) & 3] += p0 + p1;
          v[j >> 1] = cvt_bf2(p0, p1);  // packed P, in place (index j/2 <= j)
        }
      } else {
#pragma unroll
        for (int j = 0; j < 128; ++j) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(v[j]));
      }
      const float m_tile = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl;
      const bool move = kt == 0 || m_tile > m_run + kRescaleLog2;
      const float m_new = move ? (m_tile > m_run ? m_tile : m_run) : m_run;
      const float corr = (move && m_run != -INFINITY) ? ex2(m_run - m_new) : 1.f;
      if (kt > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
        // O_X holds PV_X(0 .. kt-1), all complete (covered by this S's commit)
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(ocol + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * corr);
          tmem_st32p(ocol + c0, o);
        }
      }
      if (__any_sync(0xffffffffu, move)) {
        // second pass (rows whose max moved, e.g. every row of the first
        // tile): the scores again from TMEM, 64 columns at a time (registers)
        const float msub = m_new == -INFINITY ? 0.f : m_new;
        if (move) {
#pragma unroll
          for (int k = 0; k < 4; ++k) ps[k] = 0.f;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t w[64];
          tmem_ld32(scol + hh * 64, w);
          tmem_ld32(scol + hh * 64 + 32, w + 32);
          tmem_ld_wait();
          if (move) {
            if (kt == nk - 1) {
              const int key0 = kt * kTcTile + hh * 64;
#pragma unroll
              for (int j = 0; j < 64; ++j)
                if (key0 + j > qrow || key0 + j >= n) w[j] = __float_as_uint(-INFINITY);
            }
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
              const float p0 = ex2(fmaf(__uint_as_float(w[j]), sl, -msub));
              const float p1 = ex2(fmaf(__uint_as_float(w[j + 1]), sl, -msub));
              ps[(j >> 1) & 3] += p0 + p1;
              v[hh * 32 + (j >> 1)] = cvt_bf2(p0, p1);
            }
          }
        }
      }
      m_run = m_new;
      l_run = l_run * corr + ((ps[0] + ps[1]) + (ps[2] + ps[3]));
      tmem_st32p(scol, v);  // P over S: 64 columns of bf16 pairs
      tmem_st32p(scol + 32, v + 32);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[X]);
      if (lane == 0 && (warp & 3) == 0) pattn_stamp(6 + X, kt);
    }
    // ---- epilogue: O / l
    if (nk > 0) {
      mbar_wait(&ofinal[X], 0);
      tc_fence_after();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const int K = a.H * HD;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(ocol + c0, o);
        tmem_ld_wait();
        if (qrow < n) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const int dim = c0 + j;
            uint4 w;
            w.x = cvt_bf2(__uint_as_float(o[j]) * inv, __uint_as_float(o[j + 1]) * inv);
            w.y = cvt_bf2(__uint_as_float(o[j + 2]) * inv, __uint_as_float(o[j + 3]) * inv);
            w.z = cvt_bf2(__uint_as_float(o[j + 4]) * inv, __uint_as_float(o[j + 5]) * inv);
            w.w = cvt_bf2(__uint_as_float(o[j + 6]) * inv, __uint_as_float(o[j + 7]) * inv);
            const size_t off = a.TM > 0 ? act_off(qrow, h * HD + dim, K, a.TM) : (size_t)qrow * K + h * HD + dim;
            *reinterpret_cast<uint4*>(a.out + off) = w;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tmem, 512);
}

// 2-D map over the arena as rows of 256 B (one token of one KV head), boxes of
// {64 dims, 16 tokens} = one column half of one KV block, 128-B swizzled.
static bool prefill_tensor_map(const KvGeom& kv, int64_t arena_bytes, CUtensorMap* out) {
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
  const cuuint64_t dims[2] = {128, (cuuint64_t)(arena_bytes / 256)};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, 16};
  const cuuint32_t estr[2] = {1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.arena, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t prefill_attn_tc_launch(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.kv.block_tokens != 16 || a.kv.head_dim != 128 || a.arena_bytes <= 0) return cudaErrorNotSupported;
  if (a.arena_bytes / 256 >= (int64_t)1 << 31) return cudaErrorNotSupported;  // TMA row coordinate is int32
  static thread_local const char* map_arena = nullptr;
  static thread_local int64_t map_bytes = 0;
  static thread_local CUtensorMap tmap;
  if (map_arena != a.kv.arena || map_bytes != a.arena_bytes) {
    if (!prefill_tensor_map(a.kv, a.arena_bytes, &tmap)) return cudaErrorInvalidValue;
    map_arena = a.kv.arena;
    map_bytes = a.arena_bytes;
  }
  const int qpairs = (a.n + 2 * kTcTile - 1) / (2 * kTcTile);
  const size_t smem = kCtrlBytes + 1024 + (size_t)(2 + kKStages + kVStages) * kOpBytes;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static std::atomic<uint64_t> attr{0};
  max_smem_once(prefill_attn_tc_kernel, 227 * 1024, attr);
  return launch_pdl(prefill_attn_tc_kernel, dim3(a.H * qpairs), dim3(kThreads), smem, stream, a, tmap);
}

}  // namespace ms

#ifdef MS_PATTN_TL
extern "C" int ms_dbg_pattn_tl(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, ms::g_pattn_tl, sizeof(ms::g_pattn_tl)) == cudaSuccess ? 0 : 3;
}
#endif
