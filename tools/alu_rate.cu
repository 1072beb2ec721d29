// alu_rate.cu -- issue-rate microbenchmark for the W4 dequant instruction mix
// (experiments).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_rate.bin tools/alu_rate.cu
//
// Each mode runs 8 independent dependency chains per thread, 2..16 warps per
// SM, and reports cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int kMode>
__global__ void rate_kernel(uint32_t* out, int iters, uint32_t seed) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x01010101u;
  const uint32_t s = 0x3c003c00u ^ (seed & 1);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kMode == 0) {  // HMUL2.BF16
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&v[i]);
        a = __hmul2(a, *reinterpret_cast<const __nv_bfloat162*>(&s));
        v[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (kMode == 1) {  // HMUL2 fp16
        __half2 a = *reinterpret_cast<__half2*>(&v[i]);
        a = __hmul2(a, *reinterpret_cast<const __half2*>(&s));
        v[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (kMode == 2) {  // FMUL
        v[i] = __float_as_uint(__uint_as_float(v[i]) * __uint_as_float(s));
      } else if (kMode == 3) {  // LOP3
        asm("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[i]) : "r"(0x000F000Fu), "r"(s));
      } else if (kMode == 5) {  // MUFU ex2 f32
        float x = __uint_as_float(v[i] & 0x3fffffffu) * -0.5f;
        asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
        v[i] = __float_as_uint(x);
      } else if (kMode == 6) {  // MUFU ex2 f16x2
        uint32_t x = v[i] | 0x80008000u;
        asm("ex2.approx.f16x2 %0, %0;" : "+r"(x));
        v[i] = x;
      } else if (kMode == 7) {  // software exp2 (round-to-nearest split, degree-3 polynomial)
        const float x = __uint_as_float(v[i] & 0x3fffffffu) * -0.5f;
        const float j = x + 12582912.0f;                 // 1.5 * 2^23: nearest integer in the mantissa
        const float f = x - (j - 12582912.0f);           // [-0.5, 0.5]
        float p = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
        v[i] = __float_as_uint(p) + (__float_as_uint(j) << 23);
      } else if (kMode == 4) {  // dequant word: shf + lop3 + hsub2 + hmul2 (bf16)
        uint32_t x;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(v[i] >> 4), "r"(0x000F000Fu), "r"(0x43004300u));
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&x);
        a = __hmul2(__hsub2(a, __floats2bfloat162_rn(136.f, 136.f)), *reinterpret_cast<const __nv_bfloat162*>(&s));
        v[i] ^= *reinterpret_cast<uint32_t*>(&a);
      }
    }
  }
  const long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int kMode>
void run(const char* name, int warps) {
  uint32_t* d;
  const int blocks = 148, threads = warps * 32, iters = 4096;
  cudaMalloc(&d, (size_t)(blocks * threads + blocks) * 4);
  rate_kernel<kMode><<<blocks, threads>>>(d, iters, 7);
  rate_kernel<kMode><<<blocks, threads>>>(d, iters, 7);
  cudaDeviceSynchronize();
  uint32_t cyc;
  cudaMemcpy(&cyc, d + blocks * threads, 4, cudaMemcpyDeviceToHost);
  const int per_iter = kMode == 4 ? 5 : (kMode == 5 ? 3 : (kMode == 6 ? 2 : (kMode == 7 ? 10 : 1)));  // warp-instructions per chain step (mode 4: shf, lop3, hadd2, hmul2, xor)
  const double instr_per_smsp = (double)iters * 8 * per_iter * warps / 4.0;
  printf("%-28s warps %2d: %.2f cycles per warp-instruction per SMSP\n", name, warps, cyc / instr_per_smsp);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("HMUL2.BF16", w);
    run<1>("HMUL2 fp16", w);
    run<2>("FMUL", w);
    run<3>("LOP3", w);
    run<4>("dequant word (5 instr)", w);
    run<5>("ex2.f32 (+lop, fmul)", w);
    run<6>("ex2.f16x2 (+lop)", w);
    run<7>("soft exp2 (10 instr)", w);
  }
  return 0;
}
