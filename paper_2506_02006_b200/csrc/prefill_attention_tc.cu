// prefill_attention_tc.cu -- causal prefill attention on the 5th-gen tensor
// cores (tcgen05 + TMEM), head_dim 128.
//
// Part of `start_prefill` (reference proj/src/engine.cpp:472-485, priced as
// tokens * prefill_ms_per_token at :477-478): the long-prompt prefill of
// BASELINE.json configs[3] (Llama-2-13B, 8k tokens) spends a large share of its
// time in attention.  prefill_attention.cu does it with mma.sync (m16n8k16);
// this kernel issues tcgen05.mma with 128x128 tiles.
//
// CTA = (128-query tile, query head), 11 warps, warp specialised:
//   warps 8, 10  TMA producers for K and for V: per 128-key tile, 8 paged KV
//            blocks x 2 column halves, SWIZZLE_128B boxes {64 dims, 16 keys}
//            from a 2-D tensor map over the arena (rows of 256 B).  That image
//            is directly a K-major SW128 operand for K (S = Q K^T) and an
//            MN-major SW128 operand for V (O += P V): no transpose, no
//            per-thread copies.  K has 3 buffers (freed when S(kt) completes),
//            V 2 (freed when PV(kt) completes); separate warps so neither
//            queue waits behind the other.
//   warp 9   MMA issuer (one elected lane of a converged warp):
//            S(kt) = Q K^T (8 MMAs M128 N128 K16 into one of three TMEM S
//            buffers; Q = bf16(q) unscaled, the attention contract of every
//            path), then O += P(kt) V (8 MMAs, A = P
//            read from TMEM, B = V MN-major).
//            Order S(0), S(1), [S(kt+2), PV(kt)]...: the tensor cores run up to
//            two S tiles ahead of the softmax.
//   warps 0-7 softmax: thread = (query row = TMEM lane, half of the 128 keys);
//            the halves of a row exchange maxima through shared memory under a
//            pairwise named barrier.  Online softmax in the log2 domain (the
//            fp32 scores scaled by log2(e)/sqrt(hd) inside the exp2 FMA) with lazy rescaling: the running max moves only
//            when a tile's max exceeds it by more than 2^8, so O (in TMEM) is
//            rescaled a handful of times per row instead of every tile; the
//            result is the same softmax (exact up to fp32 rounding).  P (bf16)
//            is written over its own S columns.
// TMEM: S/P [0,384) (three buffers), O [384,512).  CTAs run head-major,
// longest query tiles first, so the K/V of the heads in flight stay in L2.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kTcTile = 128;           // queries per CTA and keys per KV tile
constexpr uint32_t kOpBytes = 32768;   // one 128 x 128 bf16 operand
constexpr uint32_t kHalfBytes = 16384; // one 64-column half of it (SW128 image)
constexpr int kKStages = 3, kVStages = 2, kSBufs = 3;  // K / V tile buffers, S (and P) TMEM buffers
constexpr uint32_t kTmemS = 0, kTmemO = 384;            // S: [0, 384), O: [384, 512)
constexpr int kBars = kKStages * 2 + kVStages * 2 + kSBufs * 2 + 3;
constexpr uint32_t kCtrlBytes = 2 * kTcTile * 4 + kBars * 8 + 16;  // row maxima, barriers, TMEM slot
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
  float* sRed = reinterpret_cast<float*>(smem_raw);  // [2 half][128] row maxima / sums
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 2 * kTcTile);
  uint64_t* kfull = bar;                 // [kKStages]
  uint64_t* kempty = kfull + kKStages;   // [kKStages]
  uint64_t* vfull = kempty + kKStages;   // [kVStages]
  uint64_t* vempty = vfull + kVStages;   // [kVStages]
  uint64_t* sfull = vempty + kVStages;   // [kSBufs] S(kt) in TMEM buffer kt % kSBufs
  uint64_t* pfull = sfull + kSBufs;      // [kSBufs] P(kt) written over S(kt) (8 softmax warps)
  // [2] PV(kt) accumulated into O, on odone[kt & 1]: S(kt) is issued before
  // PV(kt-2), so when the softmax of tile kt runs PV(kt-2) may still be in
  // flight -- a single barrier could then be two phases behind and its parity
  // wait for PV(kt-1) would pass early; per parity it is at most one behind
  uint64_t* odone = pfull + kSBufs;
  uint64_t* ofinal = odone + 2;          // every MMA done (single phase)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + kBars);
  // operands: 1024-B aligned (SW128 atoms)
  uint8_t* ops = smem_raw + (((smem_u32(smem_raw) + kCtrlBytes + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint8_t* sQh = ops;                         // canonical no-swizzle, written by the softmax warps
  uint8_t* sK = sQh + kOpBytes;               // [kKStages] SW128 images [dim half][key][128 B]
  uint8_t* sV = sK + kKStages * kOpBytes;     // [kVStages] same

  // head-major, longest query tiles of a head first: the CTAs in flight share
  // the K/V of two or three heads, which stay in L2
  const int qtiles = (a.n + kTcTile - 1) / kTcTile;
  const int h = (int)blockIdx.x / qtiles;
  const int qt = qtiles - 1 - ((int)blockIdx.x - h * qtiles);
  const int kvh = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * kTcTile, n = a.n;
  const int q_last = min(q0 + kTcTile, n) - 1;
  const int n_ktiles = q_last / kTcTile + 1;
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
      for (int i = 0; i < kBars; ++i) mbar_init(&bar[i], (&bar[i] >= pfull && &bar[i] < pfull + kSBufs) ? 8 : 1);
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

  // ---- Q tile (softmax warps): fp32 -> bf16, canonical layout;
  // all 16 loads of a thread in flight at once (the CTA's first S waits on this)
  if (warp < 8) {
    float4 x[8][2];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int idx = threadIdx.x + it * 256, r = idx >> 4, c = idx & 15;
      const int q = min(q0 + r, n - 1);
      const float4* src = reinterpret_cast<const float4*>(a.q + ((size_t)q * a.H + h) * HD + c * 8);
      x[it][0] = __ldg(src);
      x[it][1] = __ldg(src + 1);
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int idx = threadIdx.x + it * 256, r = idx >> 4, c = idx & 15;
      uint32_t hi[4] = {0, 0, 0, 0};
      if (q0 + r < n) {
        const float4 x0 = x[it][0], x1 = x[it][1];
        hi[0] = pack_bf2(x0.x, x0.y);
        hi[1] = pack_bf2(x0.z, x0.w);
        hi[2] = pack_bf2(x1.x, x1.y);
        hi[3] = pack_bf2(x1.z, x1.w);
      }
      *reinterpret_cast<uint4*>(sQh + canon(r, c)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------ K producer
    // K(kt) as soon as S(kt - kKStages) released its buffer
    for (int kt = kKStages; kt < n_ktiles; ++kt) {
      const int rw = row_k;
      if (kt + 1 < n_ktiles) row_k = tile_row(kt + 1);
      mbar_wait(&kempty[kt % kKStages], ((kt / kKStages) - 1) & 1);
      load(kt, false, rw);
    }
    __syncwarp();
  } else if (warp == 10) {
    // ------------------------------------------------------ V producer
    // V(kt) as soon as PV(kt - kVStages) released its buffer
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
    const uint64_t dQh = umma_desc(smem_u32(sQh), 128u, 2048u);
    auto issue_s = [&](int kt) {  // S(kt) = Q K^T into S buffer kt % kSBufs
      const int s = kt % kKStages;
      mbar_wait(&kfull[s], (kt / kKStages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dK = desc_sw128(smem_u32(sK + s * kOpBytes), 16u, 1024u);
        const uint32_t d = tmem + kTmemS + (uint32_t)(kt % kSBufs) * 128u;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t dk = desc_add(dK, (uint32_t)(ks >> 2) * kHalfBytes + (uint32_t)(ks & 3) * 32u);
          umma_bf16(d, desc_add(dQh, ks * 256u), dk, idesc, ks ? 1u : 0u);
        }
        umma_commit(&sfull[kt % kSBufs]);
        umma_commit(&kempty[s]);
      }
      __syncwarp();
    };
    for (int kt = 0; kt < min(kSBufs - 1, n_ktiles); ++kt) issue_s(kt);
    for (int kt = 0; kt < n_ktiles; ++kt) {
      // S buffer (kt+2) % 3 held P(kt-1): its softmax finished (pfull waited
      // last iteration) and PV(kt-1), which reads it, was issued before --
      // tcgen05 MMAs of one CTA execute in issue order
      if (kt + kSBufs - 1 < n_ktiles) issue_s(kt + kSBufs - 1);
      const int sb = kt % kSBufs, sv = kt % kVStages;
      mbar_wait(&pfull[sb], (kt / kSBufs) & 1);
      mbar_wait(&vfull[sv], (kt / kVStages) & 1);
      const int r0 = q_last + 1 - kt * kTcTile;
      if (kt == n_ktiles - 1 && r0 < kTcTile) {
        // keys past the row (the rest of its last block and the clamped
        // duplicates): zero their V rows -- P is 0 there, but the arena bytes
        // past the sequence are arbitrary and 0 * NaN would not be 0
        uint8_t* vb = sV + sv * kOpBytes;
        for (int i = lane; i < (kTcTile - r0) * 16; i += 32) {
          const int r = r0 + (i >> 4), c = i & 15;
          *reinterpret_cast<uint4*>(vb + (c >> 3) * kHalfBytes + r * 128 + (c & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
        __syncwarp();
      }
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dV = desc_sw128(smem_u32(sV + sv * kOpBytes), kHalfBytes, 1024u);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_bf16_ts(tmem + kTmemO, tmem + kTmemS + (uint32_t)sb * 128u + ks * 8u, desc_add(dV, ks * 2048u),
                       idesc_pv, (kt | ks) ? 1u : 0u);
        umma_commit(&vempty[sv]);
        umma_commit(&odone[kt & 1]);
        if (kt == n_ktiles - 1) umma_commit(ofinal);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------- softmax
    const int row = (warp & 3) * 32 + lane;
    const int half = warp >> 2;
    const int qrow = q0 + row;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int pair_bar = 1 + (warp & 3);
    float m_run = -INFINITY, l_half = 0.f;
    for (int kt = 0; kt < n_ktiles; ++kt) {
      const int sb = kt % kSBufs;
      mbar_wait(&sfull[sb], (kt / kSBufs) & 1);
      tc_fence_after();
      uint32_t v[64];
      const uint32_t scol = tmem + lane_off + kTmemS + (uint32_t)sb * 128u + (uint32_t)(half * 64);
      tmem_ld32(scol, v);
      tmem_ld32(scol + 32, v + 32);
      tmem_ld_wait();
      const bool diag = kt == n_ktiles - 1;
      if (diag) {  // earlier tiles hold keys < q0 <= every query row
        const int key0 = kt * kTcTile + half * 64;
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (key0 + j > qrow || key0 + j >= n) v[j] = __float_as_uint(-INFINITY);
      }
      float m4[4];  // four independent chains
#pragma unroll
      for (int k = 0; k < 4; ++k) m4[k] = __uint_as_float(v[k]);
#pragma unroll
      for (int j = 4; j < 64; ++j) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(v[j]));
      const float sl = a.scale_log2;  // raw q.k scores -> log2 domain
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sl;
      if (kt > 0) asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // partner read the last maxima
      sRed[half * kTcTile + row] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
      const float m_tile = fmaxf(sRed[row], sRed[kTcTile + row]);
      const bool move = m_tile > m_run + kRescaleLog2;  // false while both are -inf
      const float m_new = move ? m_tile : m_run;
      const float corr = (move && m_run != -INFINITY) ? ex2(m_run - m_new) : 1.f;
      if (kt > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
        // O holds PV(0 .. kt-1): wait for the last of them, then rescale this row half
        mbar_wait(&odone[(kt - 1) & 1], ((kt - 1) >> 1) & 1);
        tc_fence_after();
        const uint32_t ocol = tmem + lane_off + kTmemO + (uint32_t)(half * 64);
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(ocol + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * corr);
          tmem_st32p(ocol + c0, o);
        }
      }
      m_run = m_new;
      const float msub = m_new == -INFINITY ? 0.f : m_new;
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 64; j += 2) {
        const float p0 = ex2(fmaf(__uint_as_float(v[j]), sl, -msub));
        const float p1 = ex2(fmaf(__uint_as_float(v[j + 1]), sl, -msub));
        ps[(j >> 1) & 3] += p0 + p1;
        pk[j >> 1] = cvt_bf2(p0, p1);
      }
      l_half = l_half * corr + ((ps[0] + ps[1]) + (ps[2] + ps[3]));
      tmem_st32p(tmem + lane_off + kTmemS + (uint32_t)sb * 128u + (uint32_t)(half * 32), pk);  // P over S
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[sb]);
    }
    // ---- epilogue: O / l
    mbar_wait(ofinal, 0);
    tc_fence_after();
    asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");  // partner read the last maxima
    sRed[half * kTcTile + row] = l_half;
    asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
    const float l = sRed[row] + sRed[kTcTile + row];
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int K = a.H * HD;
    const uint32_t ocol = tmem + lane_off + kTmemO + (uint32_t)(half * 64);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(ocol + c0, o);
      tmem_ld_wait();
      if (qrow < n) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          const int dim = half * 64 + c0 + j;
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
  const int qtiles = (a.n + kTcTile - 1) / kTcTile;
  const size_t smem = kCtrlBytes + 1024 + (size_t)(1 + kKStages + kVStages) * kOpBytes;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  return launch_pdl(prefill_attn_tc_kernel, dim3(a.H * qtiles), dim3(kThreads), smem, stream, a, tmap);
}

}  // namespace ms
