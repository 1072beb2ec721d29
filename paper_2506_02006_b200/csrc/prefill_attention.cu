// prefill_attention.cu -- causal attention of one sequence's prefill over its
// paged KV (flash-attention style: each KV tile is read once per 64-query tile).
//
// Part of `start_prefill` (reference proj/src/engine.cpp:472-485, priced as
// tokens * prefill_ms_per_token at :477-478).  The decode kernel handles one
// query per CTA and would re-read the whole prefix per query (O(n^2) bytes);
// this kernel tiles queries so an 8k-token prefill (BASELINE.json config 4)
// reads each K/V tile n/64 times from L2 instead of n times.
//
// CTA = (64-query tile, query head); 4 warps x 16 query rows.  Per 64-token KV
// tile: cp.async 16-B chunks of K and V (4 paged blocks) into XOR-swizzled
// shared memory (double buffered), S = Q K^T and O += P V on the tensor cores
// with mma.sync m16n8k16 bf16 (fp32 accumulate), online softmax in registers
// (log2 domain).  Q enters the MMA rounded to bf16 (unscaled), the score is
// scaled in fp32 afterwards: the attention contract of every path (DESIGN.md
// section 4, oracle ref_attention).
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kQTile = 64;
constexpr int kKTile = 64;

__device__ __forceinline__ uint32_t swz(int row, int chunk, int chunks_per_row) {
  return (uint32_t)(row * chunks_per_row + (chunk ^ (row & 7))) * 16u;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

}  // namespace

template <int HD>
__global__ void __launch_bounds__(128) prefill_attn_kernel(PrefillAttnArgs a) {
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQh = smem;
  uint8_t* sKV = sQh + kQTile * HD * 2;  // [2 buffers][K tile | V tile]
  int32_t* sPage = reinterpret_cast<int32_t*>(sKV + 2 * 2 * kKTile * HD * 2);

  pdl_wait();
  pdl_trigger();
  const int qt = blockIdx.x, h = blockIdx.y;
  const int kvh = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = qt * kQTile;
  const int n = a.n;
  const int q_last = min(q0 + kQTile, n) - 1;
  const int n_ktiles = q_last / kKTile + 1;
  const int n_blocks = q_last / 16 + 1;
  for (int b = threadIdx.x; b < n_blocks; b += 128) sPage[b] = a.pages[b];

  // ---- Q tile: fp32 -> bf16 into swizzled smem
  for (int idx = threadIdx.x; idx < kQTile * CH; idx += 128) {
    const int r = idx / CH, c = idx - r * CH;
    const int q = q0 + r;
    uint32_t hi[4] = {0, 0, 0, 0};
    if (q < n) {
      const float4* src = reinterpret_cast<const float4*>(a.q + ((size_t)q * a.H + h) * HD + c * 8);
      const float4 x0 = src[0], x1 = src[1];
      hi[0] = pack_bf2(x0.x, x0.y);
      hi[1] = pack_bf2(x0.z, x0.w);
      hi[2] = pack_bf2(x1.x, x1.y);
      hi[3] = pack_bf2(x1.z, x1.w);
    }
    *reinterpret_cast<uint4*>(sQh + swz(r, c, CH)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  }
  __syncthreads();

  const int64_t head_off = a.kv.layer_off(a.layer) + (int64_t)kvh * 2 * a.kv.head_bytes();
  auto load_tile = [&](int kt, int buf) {
    uint8_t* sK = sKV + (size_t)buf * 2 * kKTile * HD * 2;
    uint8_t* sV = sK + kKTile * HD * 2;
    const uint32_t sK_u = smem_u32(sK), sV_u = smem_u32(sV);
    for (int idx = threadIdx.x; idx < kKTile * CH; idx += 128) {
      const int r = idx / CH, c = idx - r * CH;
      int t = kt * kKTile + r;
      if (t > q_last) t = q_last;  // clamp: masked anyway, keeps the address valid
      const char* base = a.kv.arena + (int64_t)sPage[t >> 4] * a.kv.page_bytes + head_off + (t & 15) * HD * 2 + c * 16;
      cp_async16(sK_u + swz(r, c, CH), base);
      cp_async16(sV_u + swz(r, c, CH), base + a.kv.head_bytes());
    }
    cp_async_commit();
  };

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int g = lane >> 2, t4 = lane & 3;
  const int qrow0 = q0 + warp * 16 + g;  // this thread's two query rows: qrow0, qrow0 + 8
  const uint32_t sQh_u = smem_u32(sQh);

  load_tile(0, 0);
  for (int kt = 0; kt < n_ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_ktiles) {
      load_tile(kt + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t sK_u = smem_u32(sKV + (size_t)buf * 2 * kKTile * HD * 2);
    const uint32_t sV_u = sK_u + kKTile * HD * 2;

    // ---- S = Q K^T  (16 query rows x 64 tokens per warp)
    float s[kKTile / 8][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ah[4];
      {
        const int r = warp * 16 + (lane & 15), c = kk * 2 + (lane >> 4);
        ldsm_x4(sQh_u + swz(r, c, CH), ah[0], ah[1], ah[2], ah[3]);
      }
#pragma unroll
      for (int jp = 0; jp < kKTile / 16; ++jp) {  // pairs of 8-token n-tiles
        uint32_t b0, b1, b2, b3;
        const int r = jp * 16 + (lane & 7) + ((lane >> 4) << 3), c = kk * 2 + ((lane >> 3) & 1);
        ldsm_x4(sK_u + swz(r, c, CH), b0, b1, b2, b3);
        mma16816(s[2 * jp], ah[0], ah[1], ah[2], ah[3], b0, b1);
        mma16816(s[2 * jp + 1], ah[0], ah[1], ah[2], ah[3], b2, b3);
      }
    }
    // ---- online softmax (log2 domain), causal mask on the diagonal tiles
    const int tok0 = kt * kKTile;
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int tok = tok0 + j * 8 + 2 * t4 + (e & 1);
        const int qr = qrow0 + ((e >> 1) << 3);
        float v = s[j][e] * a.scale_log2;
        if (tok > qr) v = -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
    }
    float corr[2], psum[2] = {0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 2; ++i) corr[i] = mx[i] == -INFINITY ? 1.f : exp2f(mrow[i] - mx[i]);
    uint32_t pa[kKTile / 16][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float m = mx[e >> 1];
        p[e] = m == -INFINITY ? 0.f : exp2f(s[j][e] - m);
        psum[e >> 1] += p[e];
      }
      // A fragment of P for the PV MMA (FA2 register reuse)
      pa[j >> 1][(j & 1) * 2 + 0] = pack_bf2(p[0], p[1]);
      pa[j >> 1][(j & 1) * 2 + 1] = pack_bf2(p[2], p[3]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      psum[i] += __shfl_xor_sync(0xffffffffu, psum[i], 1);
      psum[i] += __shfl_xor_sync(0xffffffffu, psum[i], 2);
      lrow[i] = lrow[i] * corr[i] + psum[i];
      mrow[i] = mx[i];
    }
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
    // ---- O += P V
#pragma unroll
    for (int ks = 0; ks < kKTile / 16; ++ks) {
      // a0 = (row g, tokens 16ks + 2t4..), a1 = (row g+8, ..), a2/a3 = tokens + 8
      const uint32_t a0 = pa[ks][0], a1 = pa[ks][1], a2 = pa[ks][2], a3 = pa[ks][3];
#pragma unroll
      for (int jp = 0; jp < HD / 16; ++jp) {  // pairs of 8-dim n-tiles
        uint32_t b0, b1, b2, b3;
        const int r = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3), c = jp * 2 + (lane >> 4);
        ldsm_x4_t(sV_u + swz(r, c, CH), b0, b1, b2, b3);
        mma16816(o[2 * jp], a0, a1, a2, a3, b0, b1);
        mma16816(o[2 * jp + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();  // buffer `buf` is refilled two iterations later
  }

  // ---- write O / l as bf16 into the packed O-proj activation image
  const int K = a.H * HD;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int q = qrow0 + i * 8;
    if (q >= n) continue;
    const float inv = lrow[i] > 0.f ? 1.f / lrow[i] : 0.f;
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      const int dim = j * 8 + 2 * t4;
      const uint32_t v = pack_bf2(o[j][2 * i] * inv, o[j][2 * i + 1] * inv);
      const size_t off = a.TM > 0 ? act_off(q, h * HD + dim, K, a.TM) : (size_t)q * K + h * HD + dim;
      *reinterpret_cast<uint32_t*>(a.out + off) = v;
    }
  }
}

cudaError_t prefill_attn_launch(const PrefillAttnArgs& a, cudaStream_t stream) {
  if (a.kv.block_tokens != 16) return cudaErrorInvalidValue;
  // head_dim 128: the tcgen05 kernel (prefill_attention_tc.cu); MS_PREFILL_TC=0 keeps mma.sync
  static const bool tc = [] {
    const char* e = std::getenv("MS_PREFILL_TC");
    return !(e && e[0] == '0');
  }();
  if (tc && a.kv.head_dim == 128) {
    const cudaError_t e = prefill_attn_tc_launch(a, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  const int qtiles = (a.n + kQTile - 1) / kQTile;
  const int max_blocks = (a.n + 15) / 16;
  auto smem_for = [&](int hd) { return (size_t)kQTile * hd * 2 + (size_t)2 * 2 * kKTile * hd * 2 + max_blocks * 4 + 16; };
  if (a.kv.head_dim == 128) {
    const size_t sm = smem_for(128);
    static std::atomic<uint64_t> attr{0};
    max_smem_once(prefill_attn_kernel<128>, 227 * 1024, attr);
    return launch_pdl(prefill_attn_kernel<128>, dim3(qtiles, a.H), dim3(128), sm, stream, a);
  }
  if (a.kv.head_dim == 64) {
    const size_t sm = smem_for(64);
    static std::atomic<uint64_t> attr{0};
    max_smem_once(prefill_attn_kernel<64>, 227 * 1024, attr);
    return launch_pdl(prefill_attn_kernel<64>, dim3(qtiles, a.H), dim3(128), sm, stream, a);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ms
