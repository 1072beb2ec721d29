// gemm2sm.cu -- long-prefill BF16 GEMM on CTA pairs (tcgen05 cta_group::2).
//
// The prefill linear layers of `start_prefill` (reference proj/src/engine.cpp:
// 472-485) at M = thousands of tokens are tensor-core bound.  gemm_kernel<false>
// (gemm.cu) issues M128 x N256 x K16 MMAs from one SM, reading A (4 KB) and B
// (8 KB) from shared memory per MMA: ~96 B/clk of the ~128 B/clk an SM has,
// which caps it near 75% of the tensor peak.  Here two SMs of a cluster pair
// run one M256 x N256 MMA (cta_group::2): each SM holds 128 weight rows (its
// half of A) and 128 tokens (its half of B), so each SM reads 8 KB per 2x the
// flops.
//
// Cluster = 2 CTAs = one "super tile": weight tiles 2j (rank 0) and 2j+1
// (rank 1) x one 256-token tile.  Per CTA, 6 warps:
//   warp 0     producer: per 64-wide k-step, its 16 KB weight chunk and its
//              16 KB half of the activation chunk (bulk copies) into a ring
//   warp 1     rank 0: MMA issuer (4 x M256 N256 K16 per k-step, commits
//              multicast to both CTAs' barriers); rank 1: forwards "stage
//              landed" to the leader's barrier (the MMA reads both SMs' smem)
//   warps 2-5  epilogue: its own TMEM half (128 weight rows x 256 tokens) ->
//              fp32 out[m][n]; then release the accumulator to the leader
// Whole super tiles per cluster, round-robin through the same grouped raster
// as gemm.cu's whole-tile plans (8 token tiles per group).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {

namespace {

constexpr int kStages2 = 6;
constexpr uint32_t kHalfChunk = 16384;  // 128 rows x 64 k bf16
constexpr uint32_t kStageBytes2 = 2 * kHalfChunk;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  // default .release.cta semantics (as CUTLASS's ClusterBarrier::arrive): the
  // .release.cluster form compiles to a MEMBAR.GPU per arrive, which
  // serialised the per-stage hand-off (the data it guards is written by the
  // async proxy and observed through the local mbarrier first)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma2_bf16(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// arrive once on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

struct SuperIter {  // super tiles (n pair, m tile) of one cluster, round-robin + grouped raster
  int u, total, step, nst, mt_n;
  __device__ SuperIter(int n_tiles, int m_tiles, int pair, int pairs)
      : u(pair), total((n_tiles / 2) * m_tiles), step(pairs), nst(n_tiles / 2), mt_n(m_tiles) {}
  __device__ bool next(int& nsup, int& mt) {
    if (u >= total) return false;
    constexpr int kR = 8;
    const int grp = u / (kR * nst);
    const int r = u - grp * kR * nst;
    const int gm = min(kR, mt_n - grp * kR);
    nsup = r / gm;
    mt = grp * kR + (r - nsup * gm);
    u += step;
    return true;
  }
};

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm_2sm_kernel(GemmWeights W, const uint16_t* __restrict__ X, int M, GemmPlanDev plan, float* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int N = W.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1, pairs = (int)gridDim.x >> 1;
  const int nk = plan.nk;  // 64-wide k-steps
  const int n_tiles = plan.n_tiles, m_tiles = plan.tiles / plan.n_tiles;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages2 * kStageBytes2);
  uint64_t* empty = full + kStages2;
  uint64_t* pfull = full + 2 * kStages2;  // leader: the peer's half of stage s landed
  uint64_t* tfull = full + 3 * kStages2;  // [2] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;           // [2] leader: accumulator drained by both epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  auto sA = [&](int s) { return smem + (size_t)s * kStageBytes2; };
  auto sB = [&](int s) { return smem + (size_t)s * kStageBytes2 + kHalfChunk; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&pfull[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_mbar_init();
  }
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      pdl_wait();
      SuperIter st(n_tiles, m_tiles, pair, pairs);
      int nsup, mt;
      uint32_t it = 0;
      while (st.next(nsup, mt)) {
        const int n_tile = 2 * nsup + (int)rank;
        const uint8_t* xb = reinterpret_cast<const uint8_t*>(X) + (size_t)mt * (W.K / 64) * (2 * kHalfChunk) +
                            rank * kHalfChunk;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kStages2;
          if (it >= (uint32_t)kStages2) mbar_wait(&empty[s], ((it / kStages2) & 1) ^ 1);
          const int64_t ci = W.first_chunk + (int64_t)n_tile * nk + k;
          const int64_t p = ci / W.chunks_per_page, ip = p - W.inl_p0;
          const uint8_t* page = reinterpret_cast<const uint8_t*>(ip >= 0 && ip < W.n_inl ? W.inl[ip] : W.pages[p]);
          mbar_expect_tx(&full[s], kStageBytes2);
          bulk_g2s(sA(s), page + (ci - p * W.chunks_per_page) * kHalfChunk, kHalfChunk, &full[s]);
          bulk_g2s(sB(s), xb + (size_t)k * (2 * kHalfChunk), kHalfChunk, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 1) {
      // ------------------------------------------------ peer: stage landed -> leader
      if (lane == 0) {
        const uint32_t leader_pfull = mapa_rank(smem_u32(pfull), 0);
        SuperIter st(n_tiles, m_tiles, pair, pairs);
        int nsup, mt;
        uint32_t it = 0;
        while (st.next(nsup, mt))
          for (int k = 0; k < nk; ++k, ++it) {
            const int s = it % kStages2;
            mbar_wait(&full[s], (it / kStages2) & 1);
            mbar_arrive_cluster(leader_pfull + (uint32_t)s * 8u);
          }
      }
    } else {
      // ------------------------------------------------------ UMMA issuer (leader)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
      const uint64_t dA0 = umma_desc(smem_u32(sA(0)), 128u, 1024u);
      const uint64_t dB0 = umma_desc(smem_u32(sB(0)), 128u, 1024u);
      SuperIter st(n_tiles, m_tiles, pair, pairs);
      int nsup, mt;
      uint32_t it = 0, u = 0;
      while (st.next(nsup, mt)) {
        const uint32_t acc = u & 1, use = u >> 1;
        if (use > 0) mbar_wait(&tempty[acc], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * 256u;
        for (int k = 0; k < nk; ++k, ++it) {
          const int s = it % kStages2;
          const uint32_t ph = (it / kStages2) & 1;
          mbar_wait(&full[s], ph);
          mbar_wait(&pfull[s], ph);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma2_bf16(d, desc_add(dA0, (uint32_t)s * kStageBytes2 + kk * 256u),
                         desc_add(dB0, (uint32_t)s * kStageBytes2 + kk * 256u), idesc, (k | kk) ? 1u : 0u);
            umma2_commit_both(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) umma2_commit_both(&tfull[acc]);
        __syncwarp();
        ++u;
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    pdl_wait();
    const int quad = warp & 3;
    const uint32_t leader_tempty = mapa_rank(smem_u32(tempty), 0);
    SuperIter st(n_tiles, m_tiles, pair, pairs);
    int nsup, mt;
    uint32_t u = 0;
    while (st.next(nsup, mt)) {
      const uint32_t acc = u & 1, use = u >> 1;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const int n = (2 * nsup + (int)rank) * 128 + quad * 32 + lane;
      const uint32_t d = tmem_base + acc * 256u + ((uint32_t)(quad * 32) << 16);
      for (int c0 = 0; c0 < 256; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(d + (uint32_t)c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = mt * 256 + c0 + j;
          if (m < M) out[(size_t)m * N + n] = __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + acc * 8u);
      ++u;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's smem / TMEM stay valid until the leader's MMAs and both epilogues are done
  if (warp == 1) tmem_dealloc2(tmem_base, 512);
}

bool gemm_2sm_ok(const GemmWeights& w, int TM, const GemmPlanDev& plan) {
  static const bool on = [] {
    const char* e = std::getenv("MS_GEMM_2SM");
    return e && e[0] == '1';
  }();
  return on && plan.aligned && TM == 256 && plan.n_tiles % 2 == 0 && w.K % 64 == 0;
}

cudaError_t gemm_2sm_launch(const GemmWeights& w, const uint16_t* x, int M, const GemmPlanDev& plan, float* out,
                            cudaStream_t stream) {
  const size_t smem = (size_t)kStages2 * kStageBytes2 + (4 * kStages2 + 4) * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int supers = (plan.n_tiles / 2) * (plan.tiles / plan.n_tiles);
  const int pairs = std::min(sms / 2, supers);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = (pdl_enabled() && !pdl_suppress) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemm_2sm_kernel, w, x, M, plan, out);
}

}  // namespace ms
