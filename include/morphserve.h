/*
 * morphserve.h -- C ABI of the B200 serving hot path (libmorphserve.so).
 *
 * The reference (morphsim, /root/reference/proj) has no compute FFI: its hot
 * path is priced inside `Simulation` (proj/src/engine.cpp:66-676) through
 * `CostModel` (proj/src/sim_config.cpp:23-33).  This ABI is the device backend
 * those call sites bind to instead; each entry point below names the reference
 * seam it replaces.  The C++ host runtime (paper_2506_02006_b200/csrc/host/)
 * and the Python bindings call only these functions.
 *
 * Conventions (reference proj/include/morphsim/experiment.hpp:16-18):
 *   return 0 = ok, 2 = validation error (std::invalid_argument),
 *   3 = runtime error (CUDA / allocation), 4 = invariant broken (std::logic_error);
 *   the message of the last failure on this thread is ms_last_error().
 *   Plain pointers and sizes only.  "host" pointers are ordinary CPU memory;
 *   `stream` arguments are cudaStream_t passed as void* (NULL = the context's
 *   compute stream).  One context per device, driven from one host thread.
 */
#ifndef MORPHSERVE_H
#define MORPHSERVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MS_OK 0
#define MS_EVALIDATION 2
#define MS_ERUNTIME 3
#define MS_ELOGIC 4

typedef struct ms_ctx ms_ctx;

/* Llama-style decoder shape + device arena.  `block_tokens` tokens of every
 * layer form one KV block = one arena page (reference KvConfig,
 * proj/include/morphsim/kv_pool.hpp:14-18). */
typedef struct {
  int32_t num_layers, hidden, num_heads, num_kv_heads, head_dim, ffn, vocab;
  int32_t block_tokens;       /* 16 */
  int32_t max_batch;          /* decode rows per step */
  int32_t max_prefill_tokens; /* rows per prefill call */
  int32_t max_pos;            /* longest sequence (RoPE table, block-table width) */
  float rms_eps;
  double rope_theta;
  int64_t arena_pages;        /* pages of ms_page_bytes() each: weights images + KV blocks + staging */
} ms_model_desc;

const char* ms_last_error(void);

/* Bytes of one arena page = one KV block (all layers, K and V). */
int64_t ms_page_bytes(const ms_model_desc* desc);
/* Pages one layer's packed image occupies at `bits`: 16 = BF16, 8 / 4 / 3 =
 * the reference's kQ8 / kQ4 / kQ3 levels (proj/include/morphsim/toy_model.hpp:26)
 * as g128 codes + bf16 scales (Q8: one byte per code; Q4 and Q3: 4-bit
 * containers, so a Q3 image occupies the same pages as Q4).
 * page_count * ms_page_bytes() is the value a morphsim config must use for
 * model.layer_bytes[...] so that floor(freed / block_bytes) matches
 * (reference proj/src/engine.cpp:273, SimModelConfig sim_config.hpp:17-28). */
int64_t ms_layer_pages(const ms_model_desc* desc, int bits);

int ms_ctx_create(int device, const ms_model_desc* desc, ms_ctx** out);
int ms_ctx_destroy(ms_ctx* ctx);
int ms_sync(ms_ctx* ctx);
int ms_num_sms(ms_ctx* ctx);

/* ------------------------------------------------------------ weights */
/* Generates every tensor on the device with the counter RNG that
 * oracle/ref_llama.c restates bit for bit, packs the BF16 image of every layer
 * into arena pages (all layers start BF16), and builds the pinned-host variant
 * store the LayerSwapper uploads from: BF16 and Q4 images of every layer, plus
 * Q8 / Q3 when enabled with ms_variant_enable. */
int ms_weights_synthetic(ms_ctx* ctx, uint64_t seed);
/* Row-major bf16 upload of one tensor (layer -1 = global: which 0 embed,
 * 1 final norm, 2 lm_head; layer >= 0: 0 norm1, 1 qkv, 2 o, 3 norm2, 4 gate_up,
 * 5 down).  After all tensors: ms_weights_finalize(). */
int ms_weights_upload(ms_ctx* ctx, int layer, int which, const uint16_t* host_bf16, int64_t count);
int ms_weights_finalize(ms_ctx* ctx);
/* Adds the `bits` level (16, 8, 4, 3) to the variant store built at weight
 * finalisation (BF16 and Q4 are always built; Q8 and Q3 on request, each
 * costs one more pinned image per layer).  Must precede ms_weights_*.
 * Replaces the reference's eager build of every level
 * (proj/src/toy_model.cpp:64-75 materialize_variants). */
int ms_variant_enable(ms_ctx* ctx, int bits);
/* Registers caller-owned host memory as the variant-store image of one layer at
 * `bits` (SURVEY 8(b) ms_variant_register; the LayerSwapper uploads from it).
 * Must precede ms_weights_synthetic / ms_weights_finalize.  The memory is
 * page-locked here (cudaHostRegister, portable) unless already pinned and must
 * outlive the context.  prefilled = 1: it already holds the packed image
 * (ms_variant_bytes(bits) bytes, e.g. built by another replica process over
 * shared memory, or by an offline packer) and finalize skips building it;
 * prefilled = 0: finalize packs the image into it.  One host copy of every
 * variant can thus serve all replica contexts of a box. */
int ms_variant_register(ms_ctx* ctx, int layer, int bits, void* host, int64_t bytes, int prefilled);
/* Copies one layer's packed variant image (from the pinned store) for inspection. */
int64_t ms_variant_bytes(ms_ctx* ctx, int bits);
int ms_variant_export(ms_ctx* ctx, int layer, int bits, void* host_out, int64_t bytes);

/* --------------------------------------------------- LayerSwapper (a5,a6,a7)
 * Replaces MorphState::begin_swap / complete_swap (proj/src/engine.cpp:19-38)
 * and CostModel::swap_duration_ms (proj/src/sim_config.cpp:29-33): the
 * variant image is uploaded from pinned host memory with cudaMemcpyAsync on
 * the copy stream into free arena pages while decode continues on the compute
 * stream; ms_swap_commit is the token-boundary pointer flip (no flush: the
 * compute stream waits on the upload event, old pages are released behind a
 * compute-stream fence).  Validation mirrors begin_swap (range, double swap,
 * no-op) with MS_EVALIDATION. */
int ms_swap_begin(ms_ctx* ctx, int layer, int bits, uint64_t* ticket);
/* Peer fetch: the same swap, with the image copied from
 * `src`, another context of this process with the same model geometry that
 * holds `layer` committed at `bits` (device to device, cudaMemcpyPeerAsync --
 * NVLink 5 between B200s -- instead of the pinned host store over PCIe).
 * src's copy of the layer stays resident until the fetch completes (a later
 * commit on src waits for it).  Poll / wait / commit with the ticket as usual. */
int ms_swap_begin_peer(ms_ctx* ctx, int layer, int bits, ms_ctx* src, uint64_t* ticket);
int ms_swap_poll(ms_ctx* ctx, uint64_t ticket, int* done);
int ms_swap_wait(ms_ctx* ctx, uint64_t ticket, float* upload_ms);
int ms_swap_commit(ms_ctx* ctx, uint64_t ticket, int64_t* pages_freed);
int ms_layer_bits(ms_ctx* ctx, int layer);
/* Between runs: restore every layer to BF16 and unmap every KV block id. */
int ms_reset_state(ms_ctx* ctx);

/* ------------------------------------------------------ KV resizer (a7,a9)
 * Logical block ids stay owned by the host KvBlockPool (bit-exact with
 * proj/src/kv_pool.cpp); the device maps every live id to an arena page.
 * attach = KvBlockPool::attach_blocks (kv_pool.cpp:77-83): ids
 * [first_id, first_id + n) get pages carved from the freed weight pages.
 * detach = KvBlockPool::detach_blocks (kv_pool.cpp:85-100): the listed free ids
 * return their pages.  Because weights are paged too, no live block moves. */
int ms_kv_attach(ms_ctx* ctx, int64_t first_id, int64_t n);
int ms_kv_detach(ms_ctx* ctx, const int64_t* ids, int64_t n);
int64_t ms_free_pages(ms_ctx* ctx);
int64_t ms_kv_page_of(ms_ctx* ctx, int64_t block_id);
/* Copies the KV page of one mapped block (every layer, layout
 * [layer][kv_head][K|V][16 tok][head_dim] bf16, ms_page_bytes() bytes) to host
 * memory, ordered after every step already launched (inspection / tests). */
int ms_kv_export(ms_ctx* ctx, int64_t block_id, void* host_out, int64_t bytes);

/* ------------------------------------------------------- token history */
int ms_hist_reserve(ms_ctx* ctx, int32_t slots, int32_t max_len);
int ms_hist_write(ms_ctx* ctx, int32_t slot, int32_t offset, const int32_t* host_tokens, int32_t n);
int ms_hist_read(ms_ctx* ctx, int32_t slot, int32_t offset, int32_t* host_out, int32_t n);

/* ---------------------------------------------------------------- steps
 * One continuous-batching decode step (replaces CostModel::decode_step_ms at
 * proj/src/engine.cpp:523): row i decodes the token at hist[slots[i]][positions[i]]
 * (or tokens[i] if non-NULL, which is first written there), appends its K/V at
 * that position into the block listed in block_ids[i*max_blocks + pos/bt], and
 * writes the greedy next token to hist[slots[i]][positions[i]+1] and next_out[i]
 * (host, may be NULL).  logits_out (host [n][vocab], may be NULL).  The layer
 * precision of every layer is the committed one at call time (the reference's
 * precision snapshot at step start, engine.cpp:525). */
typedef struct {
  int32_t n;
  const int32_t* slots;
  const int32_t* positions;
  const int32_t* tokens;     /* optional */
  const int64_t* block_ids;  /* [n][max_blocks] logical ids */
  int32_t max_blocks;
} ms_decode_batch;
int ms_decode_step(ms_ctx* ctx, const ms_decode_batch* batch, int32_t* next_out, float* logits_out);
/* Caller-supplied stream: from now on every decode step and
 * prefill is ordered after the work already enqueued on `stream` (a
 * cudaStream_t of the context's device; NULL = none), and `stream` waits for
 * the step's completion, so caller kernels before / after a step see its
 * inputs / outputs without a host synchronisation.  The steps themselves run
 * on the context's compute stream (their CUDA graphs are captured there). */
int ms_set_stream(ms_ctx* ctx, void* stream);
/* Pipelined form of ms_decode_step: submit enqueues the step (its inputs are
 * staged at once, its next tokens copied back asynchronously) and returns; the
 * host may run one step ahead.  collect waits for the OLDEST submitted step and
 * returns its n next tokens.  At most 2 steps may be uncollected (status 2
 * otherwise).  Tokens also land in the device history, so a submitted step
 * can feed the next one without a host round trip. */
int ms_decode_submit(ms_ctx* ctx, const ms_decode_batch* batch);
int ms_decode_collect(ms_ctx* ctx, int32_t* next_out, int32_t* n_out);
/* Single-request prefill of hist[slot][0:n_tokens) (replaces
 * tokens * prefill_ms_per_token at engine.cpp:477-478, incl. re-prefill after
 * preemption); next token -> hist[slot][n_tokens] and *next_out. */
int ms_prefill(ms_ctx* ctx, int32_t slot, int32_t n_tokens, const int64_t* block_ids, int32_t n_blocks,
               int32_t* next_out, float* logits_out);
/* ms_prefill with the residual stream captured for the offline layer profiler
 * (the GPU restatement of profiler.cpp's activation trace,
 * proj/src/profiler.cpp:41-54 / toy_model.cpp forward): h_out (host) receives
 * [num_layers + 1][n_tokens][hidden] fp32 -- the input of every layer, then the
 * output of the last one (before the final norm).  logits_out as ms_prefill. */
int ms_prefill_trace(ms_ctx* ctx, int32_t slot, int32_t n_tokens, const int64_t* block_ids, int32_t n_blocks,
                     float* h_out, float* logits_out);
/* Step timing: CUDA events around the last ms_decode_step / ms_prefill. */
int ms_last_step_ms(ms_ctx* ctx, float* ms);
/* Fill the listed blocks' KV with synthetic values (bench: "prefilled" context). */
int ms_kv_fill_synthetic(ms_ctx* ctx, const int64_t* block_ids, int64_t n, uint64_t seed);

/* ------------------------------------------------------- instrumentation
 * Launch counter (every kernel this context launched), CUDA-event timer on the
 * compute stream, and per-launch timing of the paged attention kernel (events
 * bracketing each attention launch on its own stream). */
int64_t ms_launch_count(ms_ctx* ctx);
/* Decode-step CUDA graphs captured so far (a swap commit does not force a
 * re-capture of shapes already captured at that precision vector). */
int64_t ms_graph_captures(ms_ctx* ctx);
int ms_timer_start(ms_ctx* ctx);
int ms_timer_stop(ms_ctx* ctx, float* ms);
/* Per-kernel-category device time of the decode/prefill steps launched while
 * enabled (an event after every launch on the compute stream; this serialises
 * programmatic-dependent-launch overlap, so totals exceed the unprofiled step).
 * ms_prof_kernels_read fills ms_out[MS_PK_COUNT] / launches_out[MS_PK_COUNT]
 * and resets.  Instrumentation only, not a reference interface. */
enum {
  MS_PK_EMBED = 0, MS_PK_GEMM_QKV, MS_PK_GEMM_QKV_W4, MS_PK_QKV_POST, MS_PK_ATTN, MS_PK_GEMM_O, MS_PK_GEMM_O_W4,
  MS_PK_NORM, MS_PK_GEMM_GU, MS_PK_GEMM_GU_W4, MS_PK_SILU, MS_PK_GEMM_DOWN, MS_PK_GEMM_DOWN_W4, MS_PK_LM_HEAD,
  MS_PK_ARGMAX, MS_PK_COUNT
};
int ms_prof_kernels(ms_ctx* ctx, int enable);
int ms_prof_kernels_read(ms_ctx* ctx, float* ms_out, int64_t* launches_out);
int ms_prof_attention(ms_ctx* ctx, int enable);
int ms_prof_attention_read(ms_ctx* ctx, float* total_ms, int64_t* launches);

/* ------------------------------------------ kernel-level entry points (tests)
 * Device pointers, caller-owned memory, caller stream. */
int ms_k_gen_weight(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset, uint16_t* out,
                    void* stream);
int ms_k_pack_bf16(const uint16_t* w, int N, int K, uint16_t* out, void* stream);
/* g128 quantiser (reference quantize_weights, proj/src/toy_model.cpp:47-60, per
 * 128-wide group) + packer: bits 8 -> W8 chunks (16640 B), 4 / 3 -> 4-bit
 * container chunks (8448 B); codes_out (optional) = int8 codes [N][K]. */
int ms_k_quant(int bits, const uint16_t* w, int N, int K, uint8_t* out, int8_t* codes_out, void* stream);
int ms_k_quant_w4(const uint16_t* w, int N, int K, uint8_t* out, int8_t* codes_out, void* stream);
int ms_k_pack_act(const uint16_t* x, int M, int K, int TM, uint16_t* out, void* stream);
/* out[s][m][n] fp32 partials of W(packed, bits) x X(packed, TM) from the
 * persistent stream-K kernel; `splits` > 0 caps the CTA count (<= 0: one per
 * SM).  *splits_used = partial slots the plan may write; `out` must hold that
 * many [M][N] slots and be zeroed (a tile writes only the slots it uses), the
 * result is the sum over slots. */
int ms_k_gemm(int bits, const void* w_packed, int N, int K, const uint16_t* x_packed, int M, int TM, int splits,
              float* out, int* splits_used, void* stream);
/* Paged decode attention on a caller-provided arena (page_bytes per page,
 * layout [layer][kv_head][K|V][16][head_dim]): q [rows][H][hd] fp32, pages
 * [rows][max_blocks] int32 page indices, ctx_len [rows]; out bf16 [rows][H*hd]. */
int ms_k_attn_decode(const float* q, const void* arena, int64_t page_bytes, int layers, int layer, int H,
                     int KVH, int hd, const int32_t* pages, int max_blocks, const int32_t* ctx_len, int rows,
                     int splits, float* workspace, uint16_t* out, void* stream);

/* Causal prefill attention of one sequence (positions 0..n-1): q [n][H][hd]
 * fp32, pages = that sequence's page index per 16-token block; out bf16
 * [n][H*hd] row-major. */
int ms_k_attn_prefill(const float* q, const void* arena, int64_t page_bytes, int layers, int layer, int H, int KVH,
                      int hd, const int32_t* pages, int n, uint16_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MORPHSERVE_H */
