// mma_rate.cu -- tcgen05.mma issue/execute rate at the decode GEMM shapes
// (experiment, B200 only).  One CTA per SM issues groups of 8
// tcgen05.mma.cta_group::1.kind::f16 M=128 N=n K=16 (one 128-wide K group,
// as in the W4 kernel) into one TMEM accumulator, A from shared memory (SS) or
// tensor memory (TS), with the K-major no-swizzle descriptors the GEMM
// kernels use; operand contents are garbage.  Variants: issue from one
// thread ("thread"), or from a warp-uniform loop with one elected lane
// ("warp"); descriptors are precomputed, offsets are compile-time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o tools/mma_rate.bin
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02006_b200/csrc/ptx.cuh"

using namespace ms;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

template <bool kTS, bool kWarp>
__global__ void mma_kernel(int N, int G, int commit, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)N);
  const uint64_t da0 = umma_desc(smem_u32(smem), 128u, 1024u);
  const uint64_t db0 = umma_desc(smem_u32(smem + 65536), 128u, 1024u);
  if (kWarp ? warp == 1 : threadIdx.x == 32) {
    const long long t0 = clock64();
    for (int g = 0; g < G; ++g) {
      if (!kWarp || elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          // +256 B per K=16 inside a 64-wide chunk, next chunk +16 KB (A) / +N*128 B (B)
          const uint64_t db = db0 + (uint64_t)(((kk & 3) * 256u + (kk >> 2) * (uint32_t)N * 128u) >> 4);
          if (kTS)
            umma_bf16_ts(tmem, tmem + 256u + (uint32_t)kk * 8u, db, idesc, (g | kk) ? 1u : 0u);
          else
            umma_bf16(tmem, da0 + (uint64_t)(((kk & 3) * 256u + (kk >> 2) * 16384u) >> 4), db, idesc,
                      (g | kk) ? 1u : 0u);
        }
        if (commit) umma_commit(&bar);
      }
      if (kWarp) __syncwarp();
    }
    if (!kWarp || elect_one()) umma_commit(&bar2);
    const long long t1 = clock64();
    mbar_wait(&bar2, 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <bool kTS, bool kWarp>
void run(long long* d) {
  cudaFuncSetAttribute(mma_kernel<kTS, kWarp>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int N : {64, 128, 256})
    for (int commit : {0, 1}) {
      const int G = 512;
      mma_kernel<kTS, kWarp><<<148, 128, 160 * 1024>>>(N, G, commit, d);
      mma_kernel<kTS, kWarp><<<148, 128, 160 * 1024>>>(N, G, commit, d);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s %s N=%3d commit/8=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d)\n",
             kWarp ? "warp  " : "thread", kTS ? "TS" : "SS", N, commit, (double)h[0] / (8 * G),
             (double)h[1] / (8 * G), 128 * N / 256);
    }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<false, false>(d);
  run<true, false>(d);
  run<false, true>(d);
  run<true, true>(d);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
