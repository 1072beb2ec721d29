// bulk_stream.cu -- how fast can one producer thread per SM stream HBM with
// 1-D cp.async.bulk into an mbarrier ring?  (experiment, B200 only)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I.. tools/bulk_stream.cu -o /tmp/bulk_stream
//   /tmp/bulk_stream
//
// Grid = 148 CTAs x 1 (or k CTAs per SM); each CTA streams a contiguous slice
// of a 1 GiB buffer in chunks of S bytes through a D-deep ring; one consumer
// thread waits each chunk and releases it (no compute).  Reports GB/s.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../paper_2506_02006_b200/csrc/ptx.cuh"

using namespace ms;

__global__ void stream_kernel(const uint8_t* src, size_t bytes_per_cta, int S, int D, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)D * S);
  uint64_t* empty = full + D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * bytes_per_cta;
  const uint32_t n = (uint32_t)(bytes_per_cta / S);
  if (warp == 0 && lane == 0) {
    for (uint32_t it = 0; it < n; ++it) {
      const int s = it % D;
      if (it >= (uint32_t)D) mbar_wait(&empty[s], ((it / D) & 1) ^ 1);
      mbar_expect_tx(&full[s], S);
      bulk_g2s(smem + (size_t)s * S, base + (size_t)it * S, S, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t acc = 0;
    for (uint32_t it = 0; it < n; ++it) {
      const int s = it % D;
      mbar_wait(&full[s], (it / D) & 1);
      acc += smem[(size_t)s * S];
      mbar_arrive(&empty[s]);
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* buf;
  uint32_t* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int sizes[] = {4096, 8448, 16384, 16896, 32768};
  for (int per_sm : {1, 2}) {
    for (int S : sizes) {
      for (int D : {4, 6, 8, 12, 16, 24}) {
        const size_t smem = (size_t)D * S + 2 * D * 8;
        if (smem * per_sm > 220 * 1024) continue;
        const int ctas = sms * per_sm;
        size_t per = total / ctas / S * S;
        for (int rep = 0; rep < 2; ++rep) stream_kernel<<<ctas, 64, smem>>>(buf, per, S, D, sink);
        cudaEventRecord(a);
        const int R = 10;
        for (int rep = 0; rep < R; ++rep) stream_kernel<<<ctas, 64, smem>>>(buf, per, S, D, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)per * ctas * R / (ms * 1e-3) / 1e9;
        printf("ctas/sm=%d S=%6d D=%3d inflight/SM=%7.0f KB  %7.1f GB/s\n", per_sm, S, D,
               (double)D * S * per_sm / 1024, gbs);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
