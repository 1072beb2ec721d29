// elementwise.cu -- the row-wise kernels around the GEMMs and attention:
// embedding + RMSNorm, QKV split-K reduction + RoPE + paged KV append,
// residual add + RMSNorm, SiLU*up, logits reduction + greedy argmax, and the
// offline weight tools (synthetic generator, BF16 tile packer, g128 W4
// quantiser/packer).  Each output is written directly in the layout its
// consumer wants (packed activation images for the next GEMM, KV pages for
// attention) so no separate layout pass runs per step.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

// Sum of the first n split-K partial slots of one element, slot order fixed.
// The slot loads are issued together (predicated, unrolled) so their L2
// latencies overlap instead of chaining through the adds.
__device__ __forceinline__ float sum_slots(const float* p, size_t stride, int n) {
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
__device__ __forceinline__ float4 sum_slots4(const float4* p, size_t stride4, int n);
// the GEMM output at (m, col): one slot for whole-tile plans (every long
// prefill), the stream-K partial slots otherwise
__device__ __forceinline__ float4 part_ld4(const GemmPlanDev& plan, const float4* p, size_t stride4, int m, int col) {
  if (plan.aligned) return __ldcg(p);
  return sum_slots4(p, stride4, part_slots(plan, m, col));
}
__device__ __forceinline__ float4 sum_slots4(const float4* p, size_t stride4, int n) {
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

template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// ------------------------------------------------ embedding + RMSNorm (layer 0)
__global__ void __launch_bounds__(256) embed_norm_kernel(const uint16_t* __restrict__ embed,
                                                         const int32_t* __restrict__ tokens,
                                                         const int32_t* __restrict__ hist,
                                                         const int32_t* __restrict__ slot,
                                                         const int32_t* __restrict__ pos, int hist_stride, int d,
                                                         const uint16_t* __restrict__ w, float eps,
                                                         float* __restrict__ h, uint16_t* __restrict__ x, int TM) {
  __shared__ float red[32];
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int tok = tokens ? tokens[m] : hist[(size_t)slot[m] * hist_stride + pos[m]];
  const uint16_t* e = embed + (size_t)tok * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += 256) {
    const float v = bf2f(e[i]);
    h[(size_t)m * d + i] = v;
    ss += v * v;
  }
  ss = block_sum<256>(ss, red);
  const float r = 1.0f / sqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += 256) {
    const float v = h[(size_t)m * d + i];
    x[act_off(m, i, d, TM)] = f2bf((v * r) * bf2f(w[i]));
  }
}

cudaError_t embed_norm_launch(const uint16_t* embed, const int32_t* tokens, const int32_t* hist,
                              const int32_t* slot, const int32_t* pos, int hist_stride, int M, int d,
                              const uint16_t* norm_w, float eps, float* h, uint16_t* x_packed, int TM,
                              cudaStream_t s) {
  return launch_pdl(embed_norm_kernel, dim3(M), dim3(256), 0, s, embed, tokens, hist, slot, pos, hist_stride, d,
                    norm_w, eps, h, x_packed, TM);
}

// --------------------------------- QKV: split-K sum, RoPE, q out, K/V -> KV pages
// One CTA per row; thread item = (head, 4 consecutive rotation pairs): float4
// reads of both halves, float4 q stores, 8-B K/V stores (no per-element index
// arithmetic; a long prefill has M = thousands of rows).
__global__ void __launch_bounds__(256) qkv_post_kernel(const float* __restrict__ part, GemmPlanDev plan, int M, int H,
                                                       int KVH, int hd, const float* __restrict__ rc,
                                                       const float* __restrict__ rs, const int32_t* __restrict__ pos,
                                                       KvGeom kv, int layer, const int32_t* __restrict__ pages,
                                                       const int32_t* __restrict__ page_row, int page_stride,
                                                       float* __restrict__ q_out) {
  pdl_wait();
  pdl_trigger();
  const int heads = H + 2 * KVH;
  const int half = hd >> 1, g_per = half >> 2;
  const int N = heads * hd;
  const size_t stride4 = (size_t)M * N / 4;
  for (int m = blockIdx.x; m < M; m += gridDim.x) {
    const int p = pos[m];
    const int prow = page_row ? page_row[m] : m;
    const int32_t page = pages[(size_t)prow * page_stride + p / kv.block_tokens];
    const int slot = p % kv.block_tokens;
    char* kv_base = kv.arena + (int64_t)page * kv.page_bytes + kv.layer_off(layer) + (int64_t)slot * hd * 2;
    const float4* row4 = reinterpret_cast<const float4*>(part + (size_t)m * N);
    for (int u = threadIdx.x; u < heads * g_per; u += blockDim.x) {
      const int hs = u / g_per, i = (u - hs * g_per) * 4;
      const int c0 = hs * hd + i;
      float4 x0 = part_ld4(plan, row4 + (c0 >> 2), stride4, m, c0);
      float4 x1 = part_ld4(plan, row4 + ((c0 + half) >> 2), stride4, m, c0 + half);
      if (hs < H + KVH) {  // q and k heads are rotated
        const float4 c = *reinterpret_cast<const float4*>(rc + (size_t)p * half + i);
        const float4 sn = *reinterpret_cast<const float4*>(rs + (size_t)p * half + i);
        const float4 y0 = make_float4(x0.x * c.x - x1.x * sn.x, x0.y * c.y - x1.y * sn.y, x0.z * c.z - x1.z * sn.z,
                                      x0.w * c.w - x1.w * sn.w);
        x1 = make_float4(x1.x * c.x + x0.x * sn.x, x1.y * c.y + x0.y * sn.y, x1.z * c.z + x0.z * sn.z,
                         x1.w * c.w + x0.w * sn.w);
        x0 = y0;
      }
      if (hs < H) {
        float* q = q_out + ((size_t)m * H + hs) * hd;
        *reinterpret_cast<float4*>(q + i) = x0;
        *reinterpret_cast<float4*>(q + i + half) = x1;
        continue;
      }
      const bool is_v = hs >= H + KVH;
      const int kh = is_v ? hs - H - KVH : hs - H;
      uint16_t* dst = reinterpret_cast<uint16_t*>(kv_base + (int64_t)kh * 2 * kv.head_bytes() +
                                                  (is_v ? kv.head_bytes() : 0));
      *reinterpret_cast<uint2*>(dst + i) = make_uint2(pack_bf2(x0.x, x0.y), pack_bf2(x0.z, x0.w));
      *reinterpret_cast<uint2*>(dst + i + half) = make_uint2(pack_bf2(x1.x, x1.y), pack_bf2(x1.z, x1.w));
    }
  }
}

cudaError_t qkv_post_launch(const float* part, const GemmPlanDev& plan, int M, int H, int KVH, int hd, const float* rope_cos,
                            const float* rope_sin, const int32_t* pos, const KvGeom& kv, int layer,
                            const int32_t* pages, const int32_t* page_row, int page_stride, float* q_out,
                            cudaStream_t s) {
  if (hd % 8) return cudaErrorInvalidValue;
  const int items = (H + 2 * KVH) * (hd / 8);
  const int threads = items >= 256 ? 256 : (items + 31) / 32 * 32;
  return launch_pdl(qkv_post_kernel, dim3(M < 65535 ? M : 65535), dim3(threads), 0, s, part, plan, M, H, KVH, hd,
                    rope_cos, rope_sin, pos, kv, layer, pages, page_row, page_stride, q_out);
}

// ----------------------------------- residual add (split-K sum) + RMSNorm + pack
// One CTA per row; each thread keeps its (up to 8) float4 of the row in
// registers between the sum of squares and the normalised write, which goes
// straight into the packed activation image of the next GEMM.
// kNormPer float4 per thread at most: 2 for decode-sized CTAs (up to 1024
// threads, one float4 each at d <= 4096), 4 (8 for d > 8192) for long
// prefills (<= 512 threads, registers for all of a thread's loads in flight
// at once).
template <int kNormPer>
__global__ void __launch_bounds__(kNormPer <= 2 ? 1024 : 512)
    residual_norm_kernel(const float* __restrict__ part, GemmPlanDev plan, int M, int d, float* __restrict__ h,
                         const uint16_t* __restrict__ w, float eps, uint16_t* __restrict__ x, int TM,
                         int norm_row_begin) {
  __shared__ float red[32];
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * d;
  const int d4 = d >> 2;
  float4* hr = reinterpret_cast<float4*>(h + (size_t)m * d);
  const float4* pr = reinterpret_cast<const float4*>(part + (size_t)m * d);
  float4 v[kNormPer], a[kNormPer];
  float ss = 0.f;
  // every load of the row first, then the adds and stores: a store between
  // them keeps the compiler from hoisting the next cache-global loads, which
  // had serialised a thread's float4s into one DRAM round trip each
  if (plan.aligned) {  // one partial slot (long prefills): plain loads, nothing dependent in between
#pragma unroll
    for (int k = 0; k < kNormPer; ++k) {
      const int i4 = threadIdx.x + k * blockDim.x;
      if (i4 < d4) {
        v[k] = hr[i4];
        a[k] = __ldcg(pr + i4);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < kNormPer; ++k) {
      const int i4 = threadIdx.x + k * blockDim.x;
      if (i4 < d4) {
        v[k] = hr[i4];
        a[k] = part_ld4(plan, pr + i4, stride / 4, m, i4 * 4);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNormPer; ++k) {
    const int i4 = threadIdx.x + k * blockDim.x;
    if (i4 < d4) {
      v[k].x += a[k].x;
      v[k].y += a[k].y;
      v[k].z += a[k].z;
      v[k].w += a[k].w;
      hr[i4] = v[k];
      ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  if (w == nullptr || m < norm_row_begin) return;  // uniform per block
  // block reduction
  ss = warp_sum(ss);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[wid] = ss;
  __syncthreads();
  if (wid == 0) {
    float t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const float r = 1.0f / sqrtf(red[0] / (float)d + eps);
  const int mo = m - norm_row_begin;
  const uint2* w4 = reinterpret_cast<const uint2*>(w);
  uint16_t* xrow = x + act_row_off(mo, d, TM);
#pragma unroll
  for (int k = 0; k < kNormPer; ++k) {
    const int i4 = threadIdx.x + k * blockDim.x;
    if (i4 < d4) {
      const uint2 wv = w4[i4];
      uint2 o;
      o.x = pack_bf2((v[k].x * r) * __uint_as_float(wv.x << 16), (v[k].y * r) * __uint_as_float(wv.x & 0xFFFF0000u));
      o.y = pack_bf2((v[k].z * r) * __uint_as_float(wv.y << 16), (v[k].w * r) * __uint_as_float(wv.y & 0xFFFF0000u));
      *reinterpret_cast<uint2*>(xrow + act_col_off(i4 * 4, TM)) = o;
    }
  }
}

// A long prefill (thousands of rows) wants 4 float4 per thread; a decode step
// (tens of rows) wants the widest CTA: one float4 per thread.
static cudaError_t norm_launch(const float* part, const GemmPlanDev& plan, int M, int d, float* h,
                               const uint16_t* norm_w, float eps, uint16_t* x_packed, int TM, int norm_row_begin,
                               cudaStream_t s) {
  const int d4 = d / 4;
  int t = M >= 1024 ? (d4 + 3) / 4 : d4;
  t = (std::min(t, 1024) + 31) / 32 * 32;
  if (t <= 1024 && d4 <= 2 * t)
    return launch_pdl(residual_norm_kernel<2>, dim3(M), dim3(t), 0, s, part, plan, M, d, h, norm_w, eps, x_packed,
                      TM, norm_row_begin);
  t = ((d4 + 3) / 4 + 31) / 32 * 32;
  if (t <= 512)
    return launch_pdl(residual_norm_kernel<4>, dim3(M), dim3(t), 0, s, part, plan, M, d, h, norm_w, eps, x_packed,
                      TM, norm_row_begin);
  t = ((d4 + 7) / 8 + 31) / 32 * 32;
  if (t > 512) return cudaErrorInvalidValue;
  return launch_pdl(residual_norm_kernel<8>, dim3(M), dim3(t), 0, s, part, plan, M, d, h, norm_w, eps, x_packed, TM,
                    norm_row_begin);
}

cudaError_t residual_norm_launch(const float* part, const GemmPlanDev& plan, int M, int d, float* h, const uint16_t* norm_w,
                                 float eps, uint16_t* x_packed, int TM, cudaStream_t s) {
  return norm_launch(part, plan, M, d, h, norm_w, eps, x_packed, TM, 0, s);
}

cudaError_t residual_norm_rows_launch(const float* part, const GemmPlanDev& plan, int M, int d, float* h,
                                      const uint16_t* norm_w, float eps, uint16_t* x_packed, int TM,
                                      int norm_row_begin, cudaStream_t s) {
  return norm_launch(part, plan, M, d, h, norm_w, eps, x_packed, TM, norm_row_begin, s);
}

// ------------------------------------------------------------- SiLU(gate)*up
// grid (column blocks, row groups): thread = 4 consecutive columns of `rows`
// rows (8 for a long prefill, which would otherwise launch ~10^5 tiny CTAs;
// 1 for a decode step, where latency wants the widest grid).
__global__ void silu_mul_kernel(const float* __restrict__ part, GemmPlanDev plan, int M, int ffn,
                                uint16_t* __restrict__ x, int TM, int rows) {
  pdl_wait();
  pdl_trigger();
  const int f4 = ffn >> 2;
  const int j4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (j4 >= f4) return;
  const size_t stride4 = (size_t)M * 2 * ffn / 4;
  const float4* p4 = reinterpret_cast<const float4*>(part);
  const int m_end = min(M, (int)(blockIdx.y + 1) * rows);
  const size_t col = act_col_off(j4 * 4, TM);
  // columns 4 j4 .. +3: gate / up interleaved (gate_col), 8 consecutive floats
  const int n0 = gate_col(j4 * 4);
#pragma unroll 2
  for (int m = blockIdx.y * rows; m < m_end; ++m) {
    const size_t base = ((size_t)m * 2 * ffn + n0) >> 2;
    const float4 a = part_ld4(plan, p4 + base, stride4, m, n0);      // g0 u0 g1 u1
    const float4 b = part_ld4(plan, p4 + base + 1, stride4, m, n0);  // g2 u2 g3 u3
    uint2 o;
    o.x = pack_bf2(silu_f(a.x) * a.y, silu_f(a.z) * a.w);
    o.y = pack_bf2(silu_f(b.x) * b.y, silu_f(b.z) * b.w);
    *reinterpret_cast<uint2*>(x + act_row_off(m, ffn, TM) + col) = o;
  }
}

// gate_up rows -> the interleaved storage order (gate_col); run before packing
__global__ void interleave_gate_up_kernel(const uint16_t* __restrict__ w, int ffn, int K, uint16_t* __restrict__ out) {
  const int64_t total = (int64_t)2 * ffn * K / 8;  // 16-B chunks
  const int kc = K / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / kc), c = (int)(i - (int64_t)r * kc);
    const int blk = r >> 7, t = r & 127;
    const int src = (t & 1) * ffn + blk * 64 + (t >> 1);
    reinterpret_cast<uint4*>(out)[i] = reinterpret_cast<const uint4*>(w)[(int64_t)src * kc + c];
  }
}
cudaError_t interleave_gate_up_launch(const uint16_t* w, int ffn, int K, uint16_t* out, cudaStream_t s) {
  if (ffn % 64 || K % 8) return cudaErrorInvalidValue;
  interleave_gate_up_kernel<<<148 * 8, 256, 0, s>>>(w, ffn, K, out);
  return cudaGetLastError();
}

cudaError_t silu_mul_launch(const float* part, const GemmPlanDev& plan, int M, int ffn, uint16_t* x_packed, int TM,
                            cudaStream_t s) {
  const int f4 = ffn / 4;
  const int rows = M >= 1024 ? 8 : 1;
  const int gy = (M + rows - 1) / rows;
  if (gy > 65535) return cudaErrorInvalidValue;
  return launch_pdl(silu_mul_kernel, dim3((f4 + 255) / 256, gy), dim3(256), 0, s, part, plan, M, ffn, x_packed, TM,
                    rows);
}

// ------------------------------------------------------ logits + greedy argmax
__global__ void __launch_bounds__(512) argmax_kernel(const float* __restrict__ part, GemmPlanDev plan, int M, int V,
                                                     float* __restrict__ logits_out, int32_t* __restrict__ next_out,
                                                     int32_t* __restrict__ hist, const int32_t* __restrict__ slot,
                                                     const int32_t* __restrict__ pos, int hist_stride) {
  __shared__ float bv[16];
  __shared__ int bi[16];
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const size_t stride = (size_t)M * V;
  float best = -INFINITY;
  int besti = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += 512) {
    const float x = sum_slots(part + (size_t)m * V + v, stride, part_slots(plan, m, v));
    if (logits_out) logits_out[(size_t)m * V + v] = x;
    if (x > best || (x == best && v < besti)) {
      best = x;
      besti = v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
    if (ov > best || (ov == best && oi < besti)) {
      best = ov;
      besti = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    bv[w] = best;
    bi[w] = besti;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 16; ++i)
      if (bv[i] > best || (bv[i] == best && bi[i] < besti)) {
        best = bv[i];
        besti = bi[i];
      }
    if (next_out) next_out[m] = besti;
    if (hist) hist[(size_t)slot[m] * hist_stride + pos[m] + 1] = besti;
  }
}

// Wide-vocabulary variant: grid (rows, vocab chunks of kArgChunk).  Each CTA
// reduces its chunk to one 64-bit key (orderable value << 32 | ~index, so
// atomicMax picks the largest logit and, among equals, the lowest id -- the
// same tie rule as above, independent of arrival order) and the last CTA of
// the row to arrive writes the token, then resets the row's key and counter.
constexpr int kArgChunk = 4096;

__device__ __forceinline__ unsigned long long argmax_key(float v, int i) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i);
}

__global__ void __launch_bounds__(256) argmax_wide_kernel(const float* __restrict__ part, GemmPlanDev plan, int M, int V,
                                                          float* __restrict__ logits_out, int32_t* __restrict__ next_out,
                                                          int32_t* __restrict__ hist, const int32_t* __restrict__ slot,
                                                          const int32_t* __restrict__ pos, int hist_stride,
                                                          unsigned long long* __restrict__ row_key,
                                                          int* __restrict__ row_cnt) {
  __shared__ unsigned long long bk[8];
  __shared__ int last;
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x, v0 = blockIdx.y * kArgChunk, v1 = min(V, v0 + kArgChunk);
  const size_t stride = (size_t)M * V;
  unsigned long long best = 0;
  for (int v = v0 + threadIdx.x; v < v1; v += 256) {
    const float x = sum_slots(part + (size_t)m * V + v, stride, part_slots(plan, m, v));
    if (logits_out) logits_out[(size_t)m * V + v] = x;
    const unsigned long long k = argmax_key(x, v);
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, best, o);
    best = ok > best ? ok : best;
  }
  if ((threadIdx.x & 31) == 0) bk[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) best = bk[i] > best ? bk[i] : best;
    atomicMax(row_key + m, best);
    __threadfence();
    last = atomicAdd(row_cnt + m, 1) == (int)gridDim.y - 1;
    if (last) {
      __threadfence();
      const unsigned long long k = atomicExch(row_key + m, 0ull);  // read the row's max, reset for the next launch
      row_cnt[m] = 0;
      const int besti = (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
      if (next_out) next_out[m] = besti;
      if (hist) hist[(size_t)slot[m] * hist_stride + pos[m] + 1] = besti;
    }
  }
}

cudaError_t argmax_launch(const float* part, const GemmPlanDev& plan, int M, int V, float* logits_out, int32_t* next_out,
                          int32_t* hist, const int32_t* slot, const int32_t* pos, int hist_stride,
                          cudaStream_t s, unsigned long long* row_key, int* row_cnt) {
  if (row_key && row_cnt && V > 2 * kArgChunk)
    return launch_pdl(argmax_wide_kernel, dim3(M, (V + kArgChunk - 1) / kArgChunk), dim3(256), 0, s, part, plan, M, V,
                      logits_out, next_out, hist, slot, pos, hist_stride, row_key, row_cnt);
  return launch_pdl(argmax_kernel, dim3(M), dim3(512), 0, s, part, plan, M, V, logits_out, next_out, hist, slot, pos,
                    hist_stride);
}

// ------------------------------------------------ synthetic weight generator
// Bit-identical to oracle/ref_llama.c gen_one(): splitmix64 counter RNG,
// fp64 (explicitly rounded, no FMA contraction) -> fp32 -> bf16 RNE.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void gen_weight_kernel(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset,
                                  uint16_t* __restrict__ out) {
  const uint64_t key = seed ^ (tensor * 0xD1B54A32D192ED03ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(key + (uint64_t)i);
    const double u = __dmul_rn((double)(r >> 11), 0x1.0p-53);
    double w = __dadd_rn(__dmul_rn(2.0, u), -1.0);
    w = __dmul_rn(w, scale);
    w = __dadd_rn(w, offset);
    out[i] = f2bf(__double2float_rn(w));
  }
}
cudaError_t gen_weight_launch(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset,
                              uint16_t* out, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  gen_weight_kernel<<<(int)blocks, 256, 0, s>>>(seed, tensor, n, scale, offset, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------ BF16 tile packer
__global__ void pack_bf16_kernel(const uint16_t* __restrict__ w, int N, int K, uint16_t* __restrict__ out) {
  const int64_t total = (int64_t)N * K;
  const int KB = K / 64;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(idx / K), k = (int)(idx - (int64_t)n * K);
    const int nt = n >> 7, rr = n & 127, g = rr >> 3, r = rr & 7;
    const int kb = k >> 6, kk = k & 63, c = kk >> 3, e = kk & 7;
    const int64_t chunk = (int64_t)nt * KB + kb;
    out[chunk * 8192 + ((g * 8 + c) * 8 + r) * 8 + e] = w[idx];
  }
}
cudaError_t pack_bf16_launch(const uint16_t* w, int N, int K, uint16_t* out, cudaStream_t s) {
  pack_bf16_kernel<<<148 * 16, 256, 0, s>>>(w, N, K, out);
  return cudaGetLastError();
}

// --------------------------------- g128 quantiser (8 / 4 / 3 bits) + chunk packer
// One thread per (row, group).  Reference semantics (toy_model.cpp:40-60, for
// every bit width of toy_model.hpp:26): scale = max|w| / (2^(bits-1) - 1) in
// fp64, code = round(w / scale) (half away from zero), all-zero group ->
// scale 1, codes 0.  Stored: 4-bit containers (code + 8) for 4 and 3 bits
// (W4 chunk, 8448 B), bytes (code + 128) for 8 bits (W8 chunk, 16640 B); the
// bf16 scales follow the codes.
__global__ void quant_kernel(const uint16_t* __restrict__ w, int N, int K, int bits, uint8_t* __restrict__ out,
                             int8_t* __restrict__ codes_out) {
  const int G = K / 128;
  const int64_t total = (int64_t)N * G;
  const double qmax = (double)((1 << (bits - 1)) - 1);
  const int chunk_bytes = bits == 8 ? kW8ChunkBytes : kW4ChunkBytes;
  const int code_bytes = bits == 8 ? 16384 : 8192;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(idx / G), g = (int)(idx - (int64_t)n * G);
    const uint16_t* src = w + (size_t)n * K + (size_t)g * 128;
    double mx = 0.0;
    for (int i = 0; i < 128; ++i) mx = fmax(mx, fabs((double)bf2f(src[i])));
    const double scale = mx == 0.0 ? 1.0 : __ddiv_rn(mx, qmax);
    uint8_t* chunk = out + ((int64_t)(n >> 7) * G + g) * chunk_bytes;
    const int row = n & 127;
    auto code_of = [&](int kk) {
      const int code = mx == 0.0 ? 0 : (int)round(__ddiv_rn((double)bf2f(src[kk]), scale));
      if (codes_out) codes_out[(size_t)n * K + (size_t)g * 128 + kk] = (int8_t)code;
      return code;
    };
    if (bits == 8) {
      for (int j = 0; j < 8; ++j) {
        uint32_t words[4];
        for (int q = 0; q < 4; ++q) {
          uint32_t v = 0;
          for (int e = 0; e < 4; ++e) v |= ((uint32_t)(code_of(j * 16 + q * 4 + e) + 128) & 0xFFu) << (8 * e);
          words[q] = v;
        }
        *reinterpret_cast<uint4*>(chunk + (j * 128 + row) * 16) = make_uint4(words[0], words[1], words[2], words[3]);
      }
    } else {
      for (int j = 0; j < 4; ++j) {
        uint32_t words[4];
        for (int q = 0; q < 4; ++q) {
          uint32_t v = 0;
          for (int e = 0; e < 8; ++e)
            v |= ((uint32_t)(code_of(j * 32 + q * 8 + e) + 8) & 0xFu) << ((e & 1) * 16 + (e >> 1) * 4);
          words[q] = v;
        }
        *reinterpret_cast<uint4*>(chunk + (j * 128 + row) * 16) = make_uint4(words[0], words[1], words[2], words[3]);
      }
    }
    *reinterpret_cast<uint16_t*>(chunk + code_bytes + row * 2) = f2bf(__double2float_rn(scale));
  }
}
cudaError_t quant_launch(const uint16_t* w, int N, int K, int bits, uint8_t* out, int8_t* codes_out, cudaStream_t s) {
  if (bits != 8 && bits != 4 && bits != 3) return cudaErrorInvalidValue;
  const int64_t total = (int64_t)N * (K / 128);
  int64_t blocks = (total + 127) / 128;
  if (blocks > 148 * 16) blocks = 148 * 16;
  quant_kernel<<<(int)blocks, 128, 0, s>>>(w, N, K, bits, out, codes_out);
  return cudaGetLastError();
}


// ------------------------------------------------ activation packer (tests / e2e)
__global__ void pack_act_kernel(const uint16_t* __restrict__ x, int M, int K, int TM, uint16_t* __restrict__ out) {
  const int64_t total = (int64_t)M * K;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(idx / K), k = (int)(idx - (int64_t)m * K);
    out[act_off(m, k, K, TM)] = x[idx];
  }
}
cudaError_t pack_act_launch(const uint16_t* x, int M, int K, int TM, uint16_t* out, cudaStream_t s) {
  pack_act_kernel<<<148 * 8, 256, 0, s>>>(x, M, K, TM, out);
  return cudaGetLastError();
}

// ------------------------------------- synthetic KV fill (bench "prefilled" context)
__global__ void fill_kv_kernel(KvGeom kv, const int32_t* __restrict__ page_list, int n_pages, uint64_t seed) {
  const int64_t per_page = kv.page_bytes / 2;
  const int64_t total = per_page * n_pages;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pi = idx / per_page, off = idx - pi * per_page;
    const uint64_t r = splitmix64(seed + (uint64_t)idx);
    const float u = (float)(r >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
    reinterpret_cast<uint16_t*>(kv.arena + (int64_t)page_list[pi] * kv.page_bytes)[off] = f2bf(u);
  }
}
cudaError_t fill_kv_launch(const KvGeom& kv, const int32_t* page_list, int n_pages, uint64_t seed, cudaStream_t s) {
  fill_kv_kernel<<<148 * 32, 256, 0, s>>>(kv, page_list, n_pages, seed);
  return cudaGetLastError();
}

}  // namespace ms
