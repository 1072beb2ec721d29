// kernels.h -- internal launch interface between the runtime (runtime.cu) and
// the CUDA kernels.  Not part of the public C ABI (include/morphserve.h).
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace ms {

// Dynamic shared-memory opt-in for `fn` on the current device.  The attribute
// is per device, so a process driving several GPUs (peer fetch between
// contexts) sets it once per (kernel, device); `done` is the kernel's bit set.
template <typename F>
inline void max_smem_once(F* fn, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_release);
}

// Every hot-path kernel is launched with programmatic dependent launch so its
// launch latency and prologue overlap the tail of the previous kernel
// (MS_PDL=0 disables, for A/B measurements).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Packed weight chunk sizes: one chunk = 128 weight
// rows x one K block (64 for BF16, a 128-wide quantisation group otherwise).
constexpr int kBf16ChunkBytes = 16384;  // [row_group 16][k_chunk 8][row 8][8 bf16]
constexpr int kW4ChunkBytes = 8448;     // [j 4][row 128][16 B of nibbles] + 128 bf16 scales (4- and 3-bit codes)
constexpr int kW8ChunkBytes = 16640;    // [j 8][row 128][16 B of bytes] + 128 bf16 scales
// Weight kinds of the GEMM: 16 = BF16, 8 = int8 codes, 4 = int4 containers
// (the 4- and 3-bit levels share the container format and kernel).
inline int wkind_of_bits(int bits) { return bits == 3 ? 4 : bits; }
inline int chunk_k(int wkind) { return wkind == 16 ? 64 : 128; }
inline int chunk_bytes_of(int wkind) {
  return wkind == 16 ? kBf16ChunkBytes : wkind == 8 ? kW8ChunkBytes : kW4ChunkBytes;
}

// A weight matrix as the GEMM sees it: chunk c of the matrix lives in page
// (first_chunk + c) / chunks_per_page of its variant image.
// The pages a matrix spans are also passed inline in the kernel parameters
// (up to kGemmInlinePages), so the producer's first bulk copy does not wait
// for a dependent global load of the page table.
constexpr int kGemmInlinePages = 48;
struct GemmWeights {
  const uint64_t* pages;  // device array of page base addresses
  int64_t first_chunk;
  int64_t chunks_per_page;
  int N, K;
  int n_inl = 0;          // pages [inl_p0, inl_p0 + n_inl) are inlined below
  int inl_p0 = 0;
  uint64_t inl[kGemmInlinePages] = {};
};
// Fill the inline page table from a host copy of `pages` (host_pages[p] ==
// pages[p]); leaves n_inl = 0 when the matrix spans too many pages.
void gemm_inline_pages(GemmWeights& w, int wkind, const uint64_t* host_pages);

// Stream-K partition of one GEMM: T = tiles * nk k-steps split into C
// contiguous ranges (one persistent CTA each).  CTA c covers global k-steps
// [floor(c*T/C), floor((c+1)*T/C)); a tile t touched by several CTAs gets one
// fp32 partial slot per CTA (slot = c - first CTA of t).  `aligned` = whole
// tiles per CTA (one slot; the value is the raster group, see SegIter).  Consumers sum part_slots() slots of [slot][M][N]
// in slot order, so the result is deterministic.
struct GemmPlanDev {
  int64_t T;
  int C, nk, n_tiles, tiles, TM, aligned, slots;
};
// 32-bit arithmetic: gemm_plan() guarantees (T + 1) * C < 2^31 for stream-K
// plans (larger problems use whole-tile plans, where every count is 1).
__host__ __device__ inline int plan_cta_of(const GemmPlanDev& p, int64_t g) {
  const uint32_t T = (uint32_t)p.T;
  return (int)(((uint32_t)(g + 1) * (uint32_t)p.C + T - 1) / T) - 1;
}
__host__ __device__ inline int plan_count(const GemmPlanDev& p, int t) {
  if (p.aligned) return 1;
  return plan_cta_of(p, (int64_t)(t + 1) * p.nk - 1) - plan_cta_of(p, (int64_t)t * p.nk) + 1;
}
__host__ __device__ inline int part_slots(const GemmPlanDev& p, int m, int n) {
  return plan_count(p, (m / p.TM) * p.n_tiles + (n >> 7));
}

GemmPlanDev gemm_plan(int N, int K, int M, int TM, int wkind, int num_sms, size_t part_elems);

// The gate_up matrix is stored with gate and up rows interleaved per 64
// output columns: packed row 128 c + 2 i = gate row 64 c + i, row 128 c + 2 i + 1
// = up row 64 c + i.  A 128-row weight tile then holds gate AND up of the same
// 64 FFN columns, in adjacent TMEM lanes, so SiLU(gate) * up is tile-local.
__host__ __device__ inline int gate_col(int j) { return ((j >> 6) << 7) + ((j & 63) << 1); }  // up: + 1
cudaError_t interleave_gate_up_launch(const uint16_t* w, int ffn, int K, uint16_t* out, cudaStream_t s);

// Optional fused epilogue of the GEMMs (whole-tile plans, one slot):
// silu_out != nullptr -> the tile's (gate, up) lane pairs become
// bf16(silu(gate) * up) in the packed activation image [M x ffn] (token tile TMo)
// instead of fp32 partials.
struct GemmEpi {
  uint16_t* silu_out = nullptr;
  int ffn = 0, TMo = 0;
};

cudaError_t gemm_launch(const GemmWeights& w, int wkind, const uint16_t* x, int M, int TM, const GemmPlanDev& plan,
                        float* out, cudaStream_t stream, const GemmEpi& epi = GemmEpi());

// Paged KV geometry.  Page p holds one logical KV block (block_tokens tokens of
// every layer): [layer][kv_head][K|V][token][head_dim] bf16.
struct KvGeom {
  char* arena;
  int64_t page_bytes;
  int layers, kv_heads, head_dim, block_tokens;
  __host__ __device__ int64_t head_bytes() const { return (int64_t)block_tokens * head_dim * 2; }
  __host__ __device__ int64_t layer_off(int l) const { return (int64_t)l * kv_heads * 2 * head_bytes(); }
};

struct AttnArgs {
  const float* q;           // [rows][H][hd] fp32, RoPE applied (unused when qkv_part is set)
  // fused QKV post-processing (decode): when qkv_part != nullptr every CTA sums
  // the QKV GEMM's split-K partial slots for its q heads (+ RoPE) itself, and
  // the CTA holding the row's last block also rotates/appends the new K and V
  // token into the paged cache before streaming it (replaces qkv_post_kernel).
  const float* qkv_part;    // [slots][rows][(H + 2 KVH) hd]
  GemmPlanDev qkv_plan;
  const float* rope_cos;    // [max_pos][hd/2]
  const float* rope_sin;
  const int32_t* pos;       // [rows] position of the new token
  KvGeom kv;
  int layer;
  const int32_t* pages;     // page index table, row r uses pages + page_row[r] * page_stride
  const int32_t* page_row;  // nullptr => identity
  int page_stride;
  const int32_t* ctx_len;   // [rows] tokens attended (current token included)
  int rows, H, KVH;
  float scale_log2;         // log2(e) / sqrt(hd)
  int splits;               // split-KV slices (1 => write the final output directly)
  float* part_o;            // [splits][rows][H][hd] (splits > 1)
  float* part_ml;           // [splits][rows][H][2]
  uint16_t* out;            // bf16 output
  int out_packed;           // 1: packed activation image (K = H*hd, TM), 0: row-major [rows][H*hd]
  int TM;
  int stages;               // K/V ring depth (set by attn_decode_launch)
  int64_t arena_bytes;      // size of kv.arena (GQA tensor-core path: TMA tensor map over the arena)
  // CTA -> work item map (set by attn_decode_launch): items (row, kv_head) are
  // numbered row * KVH + kv_head; the first `whole_items` run as one CTA each,
  // every later item is split over `tail_splits` CTAs (merged by the combine kernel).
  int whole_items;
  int tail_splits;
};
cudaError_t attn_decode_launch(const AttnArgs& a, cudaStream_t stream);

// Causal prefill attention of ONE sequence (positions 0..n-1) over its paged KV.
struct PrefillAttnArgs {
  const float* q;         // [n][H][hd] fp32, RoPE applied
  KvGeom kv;
  int layer;
  const int32_t* pages;   // the sequence's page indices (block j -> page)
  int n, H, KVH;
  float scale_log2;
  uint16_t* out;          // packed activation image (TM > 0) or row-major [n][H*hd] (TM == 0)
  int TM;
  int64_t arena_bytes;    // arena extent (tensor map of the tcgen05 kernel); 0 = unknown
};
cudaError_t prefill_attn_launch(const PrefillAttnArgs& a, cudaStream_t stream);
// tcgen05 / TMEM variant (head_dim 128); cudaErrorNotSupported otherwise.
cudaError_t prefill_attn_tc_launch(const PrefillAttnArgs& a, cudaStream_t stream);

// elementwise / row kernels (elementwise.cu)
cudaError_t embed_norm_launch(const uint16_t* embed, const int32_t* tokens, const int32_t* hist,
                              const int32_t* slot, const int32_t* pos, int hist_stride, int M, int d,
                              const uint16_t* norm_w, float eps, float* h, uint16_t* x_packed, int TM,
                              cudaStream_t s);
cudaError_t qkv_post_launch(const float* part, const GemmPlanDev& plan, int M, int H, int KVH, int hd, const float* rope_cos,
                            const float* rope_sin, const int32_t* pos, const KvGeom& kv, int layer,
                            const int32_t* pages, const int32_t* page_row, int page_stride, float* q_out,
                            cudaStream_t s);
cudaError_t residual_norm_launch(const float* part, const GemmPlanDev& plan, int M, int d, float* h, const uint16_t* norm_w,
                                 float eps, uint16_t* x_packed, int TM, cudaStream_t s);
cudaError_t residual_norm_rows_launch(const float* part, const GemmPlanDev& plan, int M, int d, float* h,
                                      const uint16_t* norm_w, float eps, uint16_t* x_packed, int TM,
                                      int norm_row_begin, cudaStream_t s);
cudaError_t silu_mul_launch(const float* part, const GemmPlanDev& plan, int M, int ffn, uint16_t* x_packed, int TM,
                            cudaStream_t s);
// row_key / row_cnt ([M] each, zero between launches): per-row scratch of the
// wide-vocabulary (vocab-chunked) variant; nullptr selects one CTA per row.
cudaError_t argmax_launch(const float* part, const GemmPlanDev& plan, int M, int V, float* logits_out, int32_t* next_out,
                          int32_t* hist, const int32_t* slot, const int32_t* pos, int hist_stride,
                          cudaStream_t s, unsigned long long* row_key = nullptr, int* row_cnt = nullptr);
cudaError_t gen_weight_launch(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset,
                              uint16_t* out, cudaStream_t s);
cudaError_t pack_bf16_launch(const uint16_t* w, int N, int K, uint16_t* out, cudaStream_t s);
// g128 quantiser + packer for 8, 4 or 3 bits (W8 chunks / 4-bit containers)
cudaError_t quant_launch(const uint16_t* w, int N, int K, int bits, uint8_t* out, int8_t* codes_out, cudaStream_t s);
cudaError_t pack_act_launch(const uint16_t* x, int M, int K, int TM, uint16_t* out, cudaStream_t s);
cudaError_t fill_kv_launch(const KvGeom& kv, const int32_t* page_list, int n_pages, uint64_t seed,
                           cudaStream_t s);

}  // namespace ms
