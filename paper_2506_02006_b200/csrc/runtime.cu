// runtime.cu -- the device context behind include/morphserve.h.
//
// Owns: the page arena (KV blocks and layer weight images share one pool of
// page_bytes pages), the per-layer dispatch table (committed precision +
// double-buffered device page tables), the pinned-host variant store the
// LayerSwapper uploads from, the compute/copy streams, the token history, and
// the per-step driver that strings the kernels together.
//
// Reference seams replaced (see include/morphserve.h for the per-function map):
//   CostModel::decode_step_ms        proj/src/sim_config.cpp:23-27  -> ms_decode_step
//   tokens * prefill_ms_per_token    proj/src/engine.cpp:477-478    -> ms_prefill
//   CostModel::swap_duration_ms      proj/src/sim_config.cpp:29-33  -> ms_swap_begin (+ copy stream)
//   MorphState::complete_swap        proj/src/engine.cpp:30-38      -> ms_swap_commit (pointer flip)
//   KvBlockPool::attach/detach       proj/src/kv_pool.cpp:77-100    -> ms_kv_attach / ms_kv_detach
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/morphserve.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

// live contexts of this process (peer fetches reference each other's layers)
std::mutex g_ctx_mu;
std::set<ms_ctx*> g_ctxs;

struct MsError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw MsError{code, msg}; }

#define CK(x)                                                                                      \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) fail(MS_ERUNTIME, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

template <class F>
int guard(F&& f) {
  try {
    f();
    return MS_OK;
  } catch (const MsError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MS_ERUNTIME;
  }
}

constexpr int kMats = 4;  // qkv, o, gate_up, down
// Precision variants of a layer, in the reference's Precision order
// (proj/include/morphsim/toy_model.hpp:26 kFull, kQ8, kQ4, kQ3).
constexpr int kVariants = 4;
constexpr int kVariantBits[kVariants] = {16, 8, 4, 3};
int variant_of(int bits) { return bits == 16 ? 0 : bits == 8 ? 1 : bits == 4 ? 2 : bits == 3 ? 3 : -1; }
bool valid_bits(int bits) { return variant_of(bits) >= 0; }
constexpr int kRing = 3;  // staging ring depth (host may run this many steps ahead)

struct MatShape {
  int N, K;
};

struct ImageGeom {
  int bits = 16;
  int64_t chunk_bytes = 0, cpp = 0, total_chunks = 0, pages = 0;
  int64_t first_chunk[kMats] = {0, 0, 0, 0};
  MatShape mat[kMats];
};

int64_t page_bytes_of(const ms_model_desc& d) {
  return (int64_t)d.block_tokens * d.num_layers * d.num_kv_heads * 2 * d.head_dim * 2;
}

void validate_desc(const ms_model_desc& d) {
  auto bad = [](const char* m) { fail(MS_EVALIDATION, std::string("model desc: ") + m); };
  if (d.num_layers < 1 || d.hidden < 128 || d.num_heads < 1 || d.num_kv_heads < 1) bad("bad sizes");
  if (d.num_heads % d.num_kv_heads) bad("num_heads must be a multiple of num_kv_heads");
  const int G = d.num_heads / d.num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) bad("GQA group must be 1, 2, 4 or 8");
  if (d.head_dim != 64 && d.head_dim != 128) bad("head_dim must be 64 or 128");
  if (d.block_tokens != 16) bad("block_tokens must be 16");
  if (d.hidden % 128 || d.ffn % 128 || d.vocab % 128 || (d.num_heads * d.head_dim) % 128 ||
      ((d.num_heads + 2 * d.num_kv_heads) * d.head_dim) % 128)
    bad("hidden, ffn, vocab and projection widths must be multiples of 128");
  if (d.max_batch < 1 || d.max_batch > 4096 || d.max_prefill_tokens < 1 || d.max_pos < 1) bad("bad capacities");
  if (d.arena_pages < 1) bad("arena_pages must be >= 1");
}

ImageGeom image_geom(const ms_model_desc& d, int bits) {
  ImageGeom g;
  g.bits = bits;
  g.mat[0] = {(d.num_heads + 2 * d.num_kv_heads) * d.head_dim, d.hidden};
  g.mat[1] = {d.hidden, d.num_heads * d.head_dim};
  g.mat[2] = {2 * d.ffn, d.hidden};
  g.mat[3] = {d.hidden, d.ffn};
  const int wk = ms::wkind_of_bits(bits);
  g.chunk_bytes = ms::chunk_bytes_of(wk);
  const int64_t pb = page_bytes_of(d);
  g.cpp = pb / g.chunk_bytes;
  if (g.cpp < 1) {  // this level cannot be paged at this page size (e.g. Q8 with 16 KiB pages)
    g.pages = -1;
    return g;
  }
  int64_t c = 0;
  for (int i = 0; i < kMats; ++i) {
    g.first_chunk[i] = c;
    c += (int64_t)(g.mat[i].N / 128) * (g.mat[i].K / ms::chunk_k(wk));
  }
  g.total_chunks = c;
  g.pages = (c + g.cpp - 1) / g.cpp;
  return g;
}

struct FreePage {
  int32_t page;
  cudaEvent_t fence;  // compute-stream event that must complete before reuse (may be null)
};

// Device page tables: one per precision variant of the layer, at a fixed
// address for the context's lifetime, holding the page addresses of that
// variant's current image.  A decode step reads the table of the layer's
// committed precision from device memory (nothing about the pages is baked
// into kernel parameters), so a swap commit does not invalidate captured
// CUDA graphs: graphs are keyed by the per-layer precision vector instead.
struct Layer {
  int bits = 16;
  int slot = 0;  // table of the committed precision (variant_of(bits))
  uint64_t* d_table[kVariants] = {};
  uint64_t* h_table[kVariants] = {};  // pinned staging
  cudaEvent_t table_ev[kVariants] = {};  // last H2D copy out of h_table[slot] (host may rewrite after it)
  std::vector<int32_t> pages;
  cudaEvent_t last_release = nullptr;
  // in-flight swap
  bool in_flight = false;
  int to_bits = 0;
  uint64_t ticket = 0;
  std::vector<int32_t> new_pages;
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  // peer fetches reading this layer's resident image (ms_swap_begin_peer on
  // another context): its pages are not released before these complete
  // (event owned by the reading context; dropped when that context dies)
  std::vector<std::pair<cudaEvent_t, const ms_ctx*>> peer_reads;
  // pinned host variant store
  uint8_t* host_img[kVariants] = {};  // by variant_of(bits)
  // caller-registered images (ms_variant_register): not freed here; `ready`
  // = the memory already holds the packed image (another process built it)
  bool host_registered[kVariants] = {};
  bool host_ready[kVariants] = {};
};

struct Staging {  // one slot of the per-step H2D ring
  int32_t* h = nullptr;   // pinned, mapped
  int32_t* hd = nullptr;  // device alias of h (zero-copy)
  int32_t* d = nullptr;   // device
  int32_t* next_h = nullptr;  // pinned: next tokens of a submitted (not yet collected) decode step
  cudaEvent_t done = nullptr;
  int next_n = 0;
  bool pending = false;
  size_t words = 0;
  cudaEvent_t used = nullptr;
  bool armed = false;
};

}  // namespace

struct ms_ctx {
  ms_model_desc desc{};
  int device = 0;
  int num_sms = 148;
  int64_t page_bytes = 0;
  ImageGeom geom[kVariants];                  // by variant_of(bits)
  bool variant_on[kVariants] = {true, false, true, false};  // stores built at weight finalisation (ms_variant_enable)
  cudaStream_t compute = nullptr, copy = nullptr;
  char* arena = nullptr;
  ms::KvGeom kv{};
  std::vector<FreePage> free_pages;
  std::vector<cudaEvent_t> events;      // every event made by new_event (destroyed at the end)
  std::vector<cudaEvent_t> fence_live;  // compute fences that pages / layers may still reference
  std::vector<cudaEvent_t> fence_pool;  // completed fences, free for reuse
  std::vector<int32_t> id_page;     // logical KV block id -> page (-1 unmapped)
  std::vector<Layer> layers;
  uint64_t next_ticket = 1;

  // resident non-morphable weights
  uint16_t* embed = nullptr;     // [V][d] row-major
  uint16_t* normf = nullptr;     // [d]
  uint16_t* norms = nullptr;     // [L][2][d]
  uint16_t* lm_packed = nullptr; // packed [V/128][d/64] chunks
  uint64_t* lm_table = nullptr;  // 1-entry page table
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  bool weights_ready = false;
  // raw uploads awaiting finalize
  std::vector<uint16_t*> raw;  // [L*6 + 3]

  // activations
  int max_rows = 0;
  float* h = nullptr;
  uint16_t* x = nullptr;
  uint16_t* x2 = nullptr;  // SiLU output of a fused gate_up GEMM (its input x is still being read)
  float* part = nullptr;
  size_t part_elems = 0;
  float* q = nullptr;
  float* attn_ws = nullptr;
  size_t attn_ws_elems = 0;
  unsigned long long* am_key = nullptr;  // wide argmax: per-row best key (self-resetting)
  int* am_cnt = nullptr;                 // wide argmax: per-row arrival counter (self-resetting)
  std::vector<int> submitted;  // ring slots of submitted decode steps, oldest first
  // decode-step CUDA graphs (MS_GRAPH=1): keyed by staging slot / batch shape, dropped when
  // anything baked into the kernel parameters changes (layer tables, arena mappings)
  struct StepGraph {
    const int32_t* st_d;
    int n, mb, asplits, want_logits, has_tokens;
    std::vector<int8_t> bits;  // per-layer precision the graph's kernels were chosen for
    int64_t launches;
    cudaGraphExec_t exec;
  };
  std::vector<StepGraph> graphs;
  std::vector<std::array<int64_t, 6>> graph_seen;  // shapes seen once (captured on the second sighting)
  int64_t graph_captures = 0;
  uint64_t graph_gen = 0, graph_gen_built = 0;
  float* trace_h = nullptr;  // ms_prefill_trace: device [L+1][n][d] residual stream snapshots (lazy)
  size_t trace_elems = 0;
  bool tracing = false;
  int64_t tl_counter = 0;
  int32_t* next = nullptr;
  float* logits = nullptr;
  int max_blocks = 0;
  Staging ring[kRing];
  int ring_i = 0;
  int32_t* h_next = nullptr;   // pinned
  float* h_logits = nullptr;   // pinned
  cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr;
  // caller stream (ms_set_stream): steps order after its prior work and it
  // waits for each step's completion
  cudaStream_t user = nullptr;
  cudaEvent_t ev_user_in = nullptr, ev_user_out = nullptr;

  int32_t* hist = nullptr;
  int32_t hist_slots = 0, hist_len = 0;

  // instrumentation: launch counter and per-launch attention timing
  int64_t launches = 0;
  bool prof_attn = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  size_t prof_used = 0;
  // per-kernel-category step profile (ms_prof_kernels): an event after every launch
  bool prof_all = false;
  std::vector<cudaEvent_t> pk_ev;
  std::vector<int> pk_cat;
  size_t pk_used = 0;
  cudaEvent_t tm0 = nullptr, tm1 = nullptr;
};

namespace {

cudaEvent_t new_event(ms_ctx* c, bool timing = false) {
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  c->events.push_back(e);
  return e;
}

std::vector<int32_t> take_pages(ms_ctx* c, int64_t n, cudaStream_t user) {
  if ((int64_t)c->free_pages.size() < n)
    fail(MS_ERUNTIME, "arena exhausted: need " + std::to_string(n) + " pages, " +
                          std::to_string(c->free_pages.size()) + " free");
  std::vector<int32_t> out;
  out.reserve(n);
  cudaEvent_t last = nullptr;
  for (int64_t i = 0; i < n; ++i) {
    FreePage fp = c->free_pages.back();
    c->free_pages.pop_back();
    if (fp.fence && fp.fence != last && user != c->compute) {
      CK(cudaStreamWaitEvent(user, fp.fence, 0));
      last = fp.fence;
    }
    out.push_back(fp.page);
  }
  return out;
}

void give_pages(ms_ctx* c, const std::vector<int32_t>& pages, cudaEvent_t fence) {
  for (auto it = pages.rbegin(); it != pages.rend(); ++it) c->free_pages.push_back({*it, fence});
}

// Fence events are recycled: once a fence has completed, every free page and
// layer that references it drops the reference, and the event returns to the
// pool (a long serving run records one per detach / commit / reset).
void reclaim_fences(ms_ctx* c) {
  if (c->fence_live.size() < 8) return;  // amortised sweep
  std::vector<cudaEvent_t> done, live;
  for (cudaEvent_t e : c->fence_live) (cudaEventQuery(e) == cudaSuccess ? done : live).push_back(e);
  if (done.empty()) return;
  std::sort(done.begin(), done.end());
  auto is_done = [&](cudaEvent_t e) { return e && std::binary_search(done.begin(), done.end(), e); };
  for (auto& fp : c->free_pages)
    if (is_done(fp.fence)) fp.fence = nullptr;
  for (auto& L : c->layers)
    if (is_done(L.last_release)) L.last_release = nullptr;
  c->fence_live.swap(live);
  c->fence_pool.insert(c->fence_pool.end(), done.begin(), done.end());
}

cudaEvent_t compute_fence(ms_ctx* c) {
  reclaim_fences(c);
  cudaEvent_t e;
  if (!c->fence_pool.empty()) {
    e = c->fence_pool.back();
    c->fence_pool.pop_back();
  } else {
    e = new_event(c);
  }
  CK(cudaEventRecord(e, c->compute));
  c->fence_live.push_back(e);
  return e;
}

const ImageGeom& geom_of(ms_ctx* c, int bits) { return c->geom[variant_of(bits)]; }

// Write the page-address table of `pages` into layer slot `slot` (on stream s).
void write_table(ms_ctx* c, Layer& L, int slot, const std::vector<int32_t>& pages, cudaStream_t s) {
  if (L.table_ev[slot]) CK(cudaEventSynchronize(L.table_ev[slot]));  // the previous copy out of h_table[slot]
  else L.table_ev[slot] = new_event(c);
  for (size_t i = 0; i < pages.size(); ++i)
    L.h_table[slot][i] = (uint64_t)(c->arena + (int64_t)pages[i] * c->page_bytes);
  CK(cudaMemcpyAsync(L.d_table[slot], L.h_table[slot], pages.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  CK(cudaEventRecord(L.table_ev[slot], s));
}

// Upload granularity: the LayerSwapper's H2D copies share the copy engines
// with each decode step's small metadata upload, so they are issued in
// pieces of at most this many bytes (MS_UPLOAD_CHUNK; default 0 = whole pages:
// measured, smaller pieces do not reduce the decode stall).
int64_t upload_piece_bytes() {
  static const int64_t v = [] {
    const char* e = std::getenv("MS_UPLOAD_CHUNK");
    return e ? (int64_t)std::atoll(e) : (int64_t)0;
  }();
  return v;
}

void upload_image(ms_ctx* c, const uint8_t* img, const ImageGeom& g, const std::vector<int32_t>& pages,
                  cudaStream_t s) {
  const int64_t piece = upload_piece_bytes();
  for (int64_t p = 0; p < g.pages; ++p) {
    const int64_t chunks = std::min<int64_t>(g.cpp, g.total_chunks - p * g.cpp);
    const int64_t bytes = chunks * g.chunk_bytes;
    char* dst = c->arena + (int64_t)pages[p] * c->page_bytes;
    const uint8_t* src = img + p * c->page_bytes;
    const int64_t step = piece > 0 ? piece : bytes;
    for (int64_t off = 0; off < bytes; off += step)
      CK(cudaMemcpyAsync(dst + off, src + off, std::min(step, bytes - off), cudaMemcpyHostToDevice, s));
  }
}

// Scatter a contiguous packed matrix (device) into a pinned host image.
void scatter_to_image(ms_ctx* c, const ImageGeom& g, int mat, const uint8_t* packed_dev, uint8_t* img) {
  const int64_t n = (int64_t)(g.mat[mat].N / 128) * (g.mat[mat].K / ms::chunk_k(ms::wkind_of_bits(g.bits)));
  int64_t ci = 0;
  while (ci < n) {
    const int64_t c_abs = g.first_chunk[mat] + ci;
    const int64_t page = c_abs / g.cpp, inpage = c_abs % g.cpp;
    const int64_t run = std::min<int64_t>(n - ci, g.cpp - inpage);
    CK(cudaMemcpyAsync(img + page * c->page_bytes + inpage * g.chunk_bytes, packed_dev + ci * g.chunk_bytes,
                       run * g.chunk_bytes, cudaMemcpyDeviceToHost, c->compute));
    ci += run;
  }
}

int round16(int m) { return (m + 15) / 16 * 16; }

void build_images(ms_ctx* c, int l, uint16_t* w_dev[kMats], uint8_t* tmp) {
  Layer& L = c->layers[l];
  // gate_up rows into the interleaved storage order (kernels.h gate_col) once,
  // before any variant is packed: tmp <- raw, raw <- interleave(tmp)
  {
    const ms_model_desc& D = c->desc;
    CK(cudaMemcpyAsync(tmp, w_dev[2], (size_t)2 * D.ffn * D.hidden * 2, cudaMemcpyDeviceToDevice, c->compute));
    CK(ms::interleave_gate_up_launch(reinterpret_cast<const uint16_t*>(tmp), D.ffn, D.hidden, w_dev[2], c->compute));
  }
  for (int bi = 0; bi < kVariants; ++bi) {
    if (!c->variant_on[bi]) continue;
    const ImageGeom& g = c->geom[bi];
    if (L.host_ready[bi]) continue;  // pre-packed image registered by the caller
    if (!L.host_img[bi]) {
      CK(cudaHostAlloc(&L.host_img[bi], g.pages * c->page_bytes, cudaHostAllocPortable));
      std::memset(L.host_img[bi], 0, g.pages * c->page_bytes);
    }
    for (int m = 0; m < kMats; ++m) {
      if (bi == 0)
        CK(ms::pack_bf16_launch(w_dev[m], g.mat[m].N, g.mat[m].K, reinterpret_cast<uint16_t*>(tmp), c->compute));
      else
        CK(ms::quant_launch(w_dev[m], g.mat[m].N, g.mat[m].K, g.bits, tmp, nullptr, c->compute));
      scatter_to_image(c, g, m, tmp, L.host_img[bi]);
      CK(cudaStreamSynchronize(c->compute));  // tmp reused
    }
  }
}

void make_resident_bf16(ms_ctx* c) {
  for (int l = 0; l < c->desc.num_layers; ++l) {
    Layer& L = c->layers[l];
    if (!L.pages.empty()) give_pages(c, L.pages, nullptr);
    L.pages = take_pages(c, c->geom[0].pages, c->compute);
    L.bits = 16;
    L.slot = 0;
    upload_image(c, L.host_img[0], c->geom[0], L.pages, c->compute);
    write_table(c, L, L.slot, L.pages, c->compute);
  }
  CK(cudaStreamSynchronize(c->compute));
  c->weights_ready = true;
}

// The layer's matrix as the GEMM reads it: through the device page table of
// its committed precision (never inlined: the table's content changes on swaps
// while captured graphs keep their parameters).
ms::GemmWeights mat_weights(ms_ctx* c, int l, int mat) {
  Layer& L = c->layers[l];
  const ImageGeom& g = geom_of(c, L.bits);
  return ms::GemmWeights{L.d_table[L.slot], g.first_chunk[mat], g.cpp, g.mat[mat].N, g.mat[mat].K};
}

// Quantised layers (Q8 / Q4 / Q3) at every M run the fused kernel (codes ->
// bf16 dequantised into TMEM in the GEMM's staging path); no dequantised copy
// of a matrix exists.  wkind: 16 BF16, 8 int8 codes, 4 int4 containers.
// MS_FUSED_SILU=0 (experiments / A-B): keep the separate SiLU kernel at long prefills
bool fused_silu_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MS_FUSED_SILU");
    return !(e && e[0] == '0');
  }();
  return on;
}

// fuse_silu (the gate_up GEMM): when the plan takes whole tiles and the layer
// is BF16, the epilogue writes bf16(silu(gate) * up) straight into the next
// GEMM's activation image and *fused is set (no fp32 output, no SiLU launch).
ms::GemmPlanDev gemm(ms_ctx* c, const ms::GemmWeights& w, int wkind, int M, int TM, bool fuse_silu = false,
                     bool* fused = nullptr, const uint16_t* x_in = nullptr) {
  if ((size_t)M * w.N > c->part_elems) fail(MS_EVALIDATION, "GEMM rows x N exceed the partial buffer");
  const ms::GemmPlanDev plan = ms::gemm_plan(w.N, w.K, M, TM, wkind, c->num_sms, c->part_elems);
  ms::GemmEpi epi;
  // BF16 only: the quantised kernel's 256-token tiles have a single
  // accumulator, so its epilogue is not hidden behind the next tile's MMAs
  // and the fused SiLU measured slower there (13B 8k, 10 W4 layers: gate_up
  // 20.4 -> 29.4 ms vs 2.2 ms of SiLU kernel)
  const bool fuse = fuse_silu && wkind == 16 && plan.aligned && fused_silu_enabled();
  if (fuse) {
    epi.silu_out = c->x2;
    epi.ffn = w.N / 2;
    epi.TMo = TM;
  }
  if (fused) *fused = fuse;
  CK(ms::gemm_launch(w, wkind, x_in ? x_in : c->x, M, TM, plan, c->part, c->compute, epi));
  c->launches += 1;
  return plan;
}

// categories of ms_prof_kernels_read (include/morphserve.h MS_PK_*)
void pk_mark(ms_ctx* c, int cat) {
  if (!c->prof_all) return;
  if (c->pk_used == c->pk_ev.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->pk_ev.push_back(e);
    c->pk_cat.push_back(0);
  }
  c->pk_cat[c->pk_used] = cat;
  CK(cudaEventRecord(c->pk_ev[c->pk_used++], c->compute));
}

void prof_mark(ms_ctx* c) {
  if (!c->prof_attn) return;
  if (c->prof_used == c->prof_ev.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->prof_ev.push_back(e);
  }
  CK(cudaEventRecord(c->prof_ev[c->prof_used++], c->compute));
}

constexpr int kAttnMaxSplits = 16;

// Decode steps replay from captured CUDA graphs (MS_GRAPH=0 disables): a shape
// is captured the second time it is seen, at most kMaxGraphs are kept.
constexpr size_t kMaxGraphs = 64;
bool graphs_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("MS_GRAPH");
    return !(e && e[0] == '0');
  }();
  return v;
}

void drop_graphs(ms_ctx* c) {
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  c->graph_seen.clear();
}

int attn_splits(ms_ctx* c, int rows, int max_ctx) {
  static const int forced = [] {  // MS_ATTN_SPLITS (experiments)
    const char* e = std::getenv("MS_ATTN_SPLITS");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  const int ctas = rows * c->desc.num_kv_heads;
  // the GQA tensor-core kernel (G >= 2, hd 128) runs 2 CTAs/SM and splitting
  // its items (partials + a combine launch) cost more than its tail wave:
  // Llama-3-8B B=64 step 7.38 -> 6.79 ms unsplit; the MHA kernel keeps 4x
  const bool gqa = c->desc.num_heads / c->desc.num_kv_heads >= 2 && c->desc.head_dim == 128;
  const int target = c->num_sms * (gqa ? 2 : 4);
  int s = 1;
  const int nb = (max_ctx + 15) / 16;
  // at most kAttnMaxSplits: forward() lays the workspace out for that many
  // split slots (part_o [kAttnMaxSplits][rows][H][hd], then part_ml)
  while (ctas * s < target && s < kAttnMaxSplits && nb / (s * 2) >= 8) s *= 2;
  return s;
}

// The decoder over M rows whose per-row metadata already sits in device memory.
void forward(ms_ctx* c, int M, int TM, const int32_t* d_slot, const int32_t* d_pos, const int32_t* d_ctx,
             const int32_t* d_tokens, const int32_t* d_pages, const int32_t* d_page_row, int page_stride,
             int max_ctx, int final_row_begin, bool want_logits) {
  const ms_model_desc& D = c->desc;
  const int d = D.hidden, H = D.num_heads, KVH = D.num_kv_heads, hd = D.head_dim;
  pk_mark(c, -1);
  CK(ms::embed_norm_launch(c->embed, d_tokens, c->hist, d_slot, d_pos, c->hist_len, M, d, c->norms, D.rms_eps,
                           c->h, c->x, TM, c->compute));
  c->launches += 1;
  pk_mark(c, MS_PK_EMBED);
  const int asplits = attn_splits(c, M, max_ctx);
  for (int l = 0; l < D.num_layers; ++l) {
    if (c->tracing)  // residual stream entering layer l
      CK(cudaMemcpyAsync(c->trace_h + (size_t)l * M * d, c->h, (size_t)M * d * sizeof(float), cudaMemcpyDeviceToDevice,
                         c->compute));
    const int wk = ms::wkind_of_bits(c->layers[l].bits);
    const bool w4 = wk != 16;  // profile category: quantised layer
    ms::GemmPlanDev s = gemm(c, mat_weights(c, l, 0), wk, M, TM);
    pk_mark(c, w4 ? MS_PK_GEMM_QKV_W4 : MS_PK_GEMM_QKV);
    prof_mark(c);
    if (d_page_row != nullptr) {
      // prefill: one sequence, QKV post-processing (RoPE + K/V append) then
      // tiled causal attention (page table row 0)
      CK(ms::qkv_post_launch(c->part, s, M, H, KVH, hd, c->rope_cos, c->rope_sin, d_pos, c->kv, l, d_pages,
                             d_page_row, page_stride, c->q, c->compute));
      c->launches += 1;
      pk_mark(c, MS_PK_QKV_POST);
      ms::PrefillAttnArgs pa{};
      pa.q = c->q;
      pa.kv = c->kv;
      pa.layer = l;
      pa.pages = d_pages;
      pa.n = M;
      pa.H = H;
      pa.KVH = KVH;
      pa.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
      pa.out = c->x;
      pa.TM = TM;
      pa.arena_bytes = (int64_t)c->desc.arena_pages * c->page_bytes;
      CK(ms::prefill_attn_launch(pa, c->compute));
      c->launches += 1;
    } else {
      // decode: the attention kernel does the QKV post-processing itself
      ms::AttnArgs a{};
      a.kv = c->kv;
      a.layer = l;
      a.pages = d_pages;
      a.page_row = nullptr;
      a.page_stride = page_stride;
      a.ctx_len = d_ctx;
      a.rows = M;
      a.H = H;
      a.KVH = KVH;
      a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
      a.splits = asplits;
      // workspace laid out for kAttnMaxSplits split slots
      a.part_o = c->attn_ws;
      a.part_ml = c->attn_ws + (size_t)kAttnMaxSplits * M * H * hd;
      a.qkv_part = c->part;
      a.qkv_plan = s;
      a.rope_cos = c->rope_cos;
      a.rope_sin = c->rope_sin;
      a.pos = d_pos;
      a.out = c->x;
      a.out_packed = 1;
      a.TM = TM;
      a.arena_bytes = (int64_t)c->desc.arena_pages * c->page_bytes;
      CK(ms::attn_decode_launch(a, c->compute));
      c->launches += asplits > 1 ? 2 : 1;
    }
    pk_mark(c, MS_PK_ATTN);
    prof_mark(c);
    const uint16_t* n2 = c->norms + ((size_t)l * 2 + 1) * d;
    const bool last = l == D.num_layers - 1;
    const uint16_t* nw = last ? c->normf : c->norms + ((size_t)(l + 1) * 2) * d;
    const int tm_out = last ? round16(M - final_row_begin) > 256 ? 256 : round16(M - final_row_begin) : TM;
    const int row_begin = last ? final_row_begin : 0;
    s = gemm(c, mat_weights(c, l, 1), wk, M, TM);
    pk_mark(c, w4 ? MS_PK_GEMM_O_W4 : MS_PK_GEMM_O);
    CK(ms::residual_norm_launch(c->part, s, M, d, c->h, n2, D.rms_eps, c->x, TM, c->compute));
    c->launches += 1;
    pk_mark(c, MS_PK_NORM);
    bool silu_done = false;
    s = gemm(c, mat_weights(c, l, 2), wk, M, TM, true, &silu_done);
    pk_mark(c, w4 ? MS_PK_GEMM_GU_W4 : MS_PK_GEMM_GU);
    if (!silu_done) {
      CK(ms::silu_mul_launch(c->part, s, M, D.ffn, c->x, TM, c->compute));
      c->launches += 1;
      pk_mark(c, MS_PK_SILU);
    }
    s = gemm(c, mat_weights(c, l, 3), wk, M, TM, false, nullptr, silu_done ? c->x2 : c->x);
    pk_mark(c, w4 ? MS_PK_GEMM_DOWN_W4 : MS_PK_GEMM_DOWN);
    CK(ms::residual_norm_rows_launch(c->part, s, M, d, c->h, nw, D.rms_eps, c->x, tm_out, row_begin, c->compute));
    c->launches += 1;
    pk_mark(c, MS_PK_NORM);
  }
  if (c->tracing)  // after the last layer (before the final norm)
    CK(cudaMemcpyAsync(c->trace_h + (size_t)D.num_layers * M * d, c->h, (size_t)M * d * sizeof(float),
                       cudaMemcpyDeviceToDevice, c->compute));
  const int Mo = M - final_row_begin;
  const int TMo = round16(Mo) > 256 ? 256 : round16(Mo);
  ms::GemmWeights lw{c->lm_table, 0, (int64_t)1 << 40, D.vocab, d};
  const uint64_t lm_addr = (uint64_t)c->lm_packed;
  ms::gemm_inline_pages(lw, 16, &lm_addr);
  const ms::GemmPlanDev s = gemm(c, lw, 16, Mo, TMo);
  pk_mark(c, MS_PK_LM_HEAD);
  CK(ms::argmax_launch(c->part, s, Mo, D.vocab, want_logits ? c->logits : nullptr, c->next, c->hist,
                       d_slot + final_row_begin, d_pos + final_row_begin, c->hist_len, c->compute, c->am_key,
                       c->am_cnt));
  c->launches += 1;
  pk_mark(c, MS_PK_ARGMAX);
}

Staging& next_staging(ms_ctx* c, size_t words) {
  Staging& st = c->ring[c->ring_i];
  c->ring_i = (c->ring_i + 1) % kRing;
  if (st.armed) CK(cudaEventSynchronize(st.used));
  if (st.words < words) {
    if (st.h) cudaFreeHost(st.h);
    if (st.d) cudaFree(st.d);
    st.words = words * 2 + 4;
    CK(cudaHostAlloc(&st.h, st.words * 4, cudaHostAllocMapped | cudaHostAllocPortable));
    CK(cudaHostGetDevicePointer(&st.hd, st.h, 0));
    CK(cudaMalloc(&st.d, st.words * 4));
  }
  return st;
}

int32_t page_of(ms_ctx* c, int64_t id) {
  if (id < 0 || id >= (int64_t)c->id_page.size() || c->id_page[id] < 0)
    fail(MS_EVALIDATION, "block id " + std::to_string(id) + " is not mapped to a page");
  return c->id_page[id];
}

void check_ready(ms_ctx* c) {
  if (!c->weights_ready) fail(MS_EVALIDATION, "weights not initialised");
  if (!c->hist) fail(MS_EVALIDATION, "token history not reserved (ms_hist_reserve)");
}

// Per-step metadata upload by zero-copy reads of the mapped staging buffer:
// the step never queues behind LayerSwapper uploads in the copy engines
// (a cudaMemcpyAsync H2D on the compute stream waits for every H2D copy
// submitted before it, i.e. for a whole in-flight layer image).
__global__ void stage_in_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void hist_in_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

void stage_in(ms_ctx* c, Staging& st, size_t words) {
  const int64_t n16 = (int64_t)((words * 4 + 15) / 16);
  const int blocks = (int)std::min<int64_t>(64, (n16 + 255) / 256);
  stage_in_kernel<<<blocks, 256, 0, c->compute>>>(reinterpret_cast<const int4*>(st.hd), reinterpret_cast<int4*>(st.d),
                                                  n16);
  CK(cudaGetLastError());
  c->launches += 1;
}

__global__ void hist_scatter_kernel(int32_t* hist, int stride, const int32_t* slot, const int32_t* pos,
                                    const int32_t* tok, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) hist[(size_t)slot[i] * stride + pos[i]] = tok[i];
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* ms_last_error(void) { return g_err.c_str(); }

int64_t ms_page_bytes(const ms_model_desc* desc) { return desc ? page_bytes_of(*desc) : -1; }

int64_t ms_layer_pages(const ms_model_desc* desc, int bits) {
  int64_t out = -1;
  guard([&] {
    if (!desc || !valid_bits(bits)) fail(MS_EVALIDATION, "bits must be 16, 8, 4 or 3");
    out = image_geom(*desc, bits).pages;
    if (out < 0) fail(MS_EVALIDATION, "page smaller than one weight chunk at this precision");
  });
  return out;
}

int ms_ctx_create(int device, const ms_model_desc* desc, ms_ctx** out) {
  return guard([&] {
    if (!desc || !out) fail(MS_EVALIDATION, "null argument");
    validate_desc(*desc);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(MS_EVALIDATION, "no such CUDA device");
    CK(cudaSetDevice(device));
    auto* c = new ms_ctx();
    try {
      c->desc = *desc;
      c->device = device;
      cudaDeviceProp prop;
      CK(cudaGetDeviceProperties(&prop, device));
      c->num_sms = prop.multiProcessorCount;
      if (prop.major != 10) fail(MS_ERUNTIME, "libmorphserve is built for sm_100a (B200) only");
      c->page_bytes = page_bytes_of(*desc);
      for (int v = 0; v < kVariants; ++v) c->geom[v] = image_geom(*desc, kVariantBits[v]);
      for (int v : {0, 2})  // BF16 and Q4 are always built
        if (c->geom[v].pages < 0) fail(MS_EVALIDATION, "page smaller than one weight chunk");
      CK(cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
      CK(cudaMalloc(&c->arena, (size_t)desc->arena_pages * c->page_bytes));
      c->kv = ms::KvGeom{c->arena, c->page_bytes, desc->num_layers, desc->num_kv_heads, desc->head_dim,
                         desc->block_tokens};
      c->free_pages.reserve(desc->arena_pages);
      for (int64_t p = desc->arena_pages - 1; p >= 0; --p) c->free_pages.push_back({(int32_t)p, nullptr});
      c->layers.resize(desc->num_layers);
      int64_t max_img_pages = 0;
      for (int v = 0; v < kVariants; ++v) max_img_pages = std::max(max_img_pages, c->geom[v].pages);
      for (auto& L : c->layers) {
        for (int s = 0; s < kVariants; ++s) {
          CK(cudaMalloc(&L.d_table[s], max_img_pages * sizeof(uint64_t)));
          CK(cudaHostAlloc(&L.h_table[s], max_img_pages * sizeof(uint64_t), cudaHostAllocDefault));
        }
        CK(cudaEventCreateWithFlags(&L.ev_start, cudaEventDefault));
        CK(cudaEventCreateWithFlags(&L.ev_done, cudaEventDefault));
      }
      const int d = desc->hidden, H = desc->num_heads, hd = desc->head_dim;
      const int qkv_n = (H + 2 * desc->num_kv_heads) * hd;
      c->max_rows = std::max(desc->max_batch, desc->max_prefill_tokens);
      const int rows_pad = (c->max_rows + 255) / 256 * 256;
      const int kmax = std::max(std::max(d, H * hd), desc->ffn);
      const int nmax = std::max(std::max(qkv_n, 2 * desc->ffn), std::max(d, desc->vocab));
      CK(cudaMalloc(&c->h, (size_t)c->max_rows * d * sizeof(float)));
      CK(cudaMalloc(&c->x, (size_t)rows_pad * kmax * sizeof(uint16_t)));
      CK(cudaMemset(c->x, 0, (size_t)rows_pad * kmax * sizeof(uint16_t)));
      // second image for the fused gate_up -> SiLU output (whole-tile plans)
      const size_t x2_elems = (size_t)rows_pad * desc->ffn;
      CK(cudaMalloc(&c->x2, x2_elems * sizeof(uint16_t)));
      CK(cudaMemset(c->x2, 0, x2_elems * sizeof(uint16_t)));
      c->part_elems = std::max((size_t)desc->max_prefill_tokens * std::max(qkv_n, 2 * desc->ffn),
                               (size_t)std::min(desc->max_batch * 16, 4096) * nmax);
      c->part_elems = std::max(c->part_elems, (size_t)std::min(desc->max_prefill_tokens, 256) * desc->vocab);
      CK(cudaMalloc(&c->part, c->part_elems * sizeof(float)));
      CK(cudaMalloc(&c->q, (size_t)c->max_rows * H * hd * sizeof(float)));
      c->attn_ws_elems = (size_t)16 * desc->max_batch * H * (hd + 2);
      CK(cudaMalloc(&c->attn_ws, c->attn_ws_elems * sizeof(float)));
      CK(cudaMalloc(&c->am_key, (size_t)c->max_rows * sizeof(unsigned long long)));
      CK(cudaMemset(c->am_key, 0, (size_t)c->max_rows * sizeof(unsigned long long)));
      CK(cudaMalloc(&c->am_cnt, (size_t)c->max_rows * sizeof(int)));
      CK(cudaMemset(c->am_cnt, 0, (size_t)c->max_rows * sizeof(int)));
      CK(cudaMalloc(&c->next, (size_t)c->max_rows * sizeof(int32_t)));
      CK(cudaMalloc(&c->logits, (size_t)desc->max_batch * desc->vocab * sizeof(float)));
      CK(cudaHostAlloc(&c->h_next, (size_t)c->max_rows * sizeof(int32_t), cudaHostAllocDefault));
      CK(cudaHostAlloc(&c->h_logits, (size_t)desc->max_batch * desc->vocab * sizeof(float), cudaHostAllocDefault));
      c->max_blocks = (desc->max_pos + desc->block_tokens - 1) / desc->block_tokens;
      for (auto& st : c->ring) CK(cudaEventCreateWithFlags(&st.used, cudaEventDisableTiming));
      CK(cudaEventCreate(&c->ev_step0));
      CK(cudaEventCreate(&c->ev_step1));
      // RoPE table (fp64 -> fp32), same formula as oracle/ref_llama.c ref_rope_table
      const int half = hd / 2;
      std::vector<float> cs((size_t)desc->max_pos * half), sn((size_t)desc->max_pos * half);
      for (int p = 0; p < desc->max_pos; ++p)
        for (int i = 0; i < half; ++i) {
          const double inv = std::pow(desc->rope_theta, -2.0 * (double)i / (double)hd);
          const double a = (double)p * inv;
          cs[(size_t)p * half + i] = (float)std::cos(a);
          sn[(size_t)p * half + i] = (float)std::sin(a);
        }
      CK(cudaMalloc(&c->rope_cos, cs.size() * sizeof(float)));
      CK(cudaMalloc(&c->rope_sin, sn.size() * sizeof(float)));
      CK(cudaMemcpy(c->rope_cos, cs.data(), cs.size() * sizeof(float), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->rope_sin, sn.data(), sn.size() * sizeof(float), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&c->embed, (size_t)desc->vocab * d * 2));
      CK(cudaMalloc(&c->normf, (size_t)d * 2));
      CK(cudaMalloc(&c->norms, (size_t)desc->num_layers * 2 * d * 2));
      CK(cudaMalloc(&c->lm_packed, (size_t)desc->vocab * d * 2));
      CK(cudaMalloc(&c->lm_table, sizeof(uint64_t)));
      const uint64_t lm_addr = (uint64_t)c->lm_packed;
      CK(cudaMemcpy(c->lm_table, &lm_addr, sizeof(uint64_t), cudaMemcpyHostToDevice));
      c->raw.assign((size_t)desc->num_layers * 6 + 3, nullptr);
    } catch (...) {
      ms_ctx_destroy(c);
      throw;
    }
    {
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      g_ctxs.insert(c);
    }
    *out = c;
  });
}

int ms_ctx_destroy(ms_ctx* c) {
  if (!c) return MS_OK;
  cudaSetDevice(c->device);
  if (c->compute) cudaStreamSynchronize(c->compute);
  if (c->copy) cudaStreamSynchronize(c->copy);
  {
    // peer fetches: this context's copies are done (copy stream synced); drop
    // its read events from the layers it read, and wait for other contexts
    // still reading this context's layers
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    g_ctxs.erase(c);
    for (ms_ctx* o : g_ctxs)
      for (auto& L : o->layers)
        L.peer_reads.erase(std::remove_if(L.peer_reads.begin(), L.peer_reads.end(),
                                          [c](const std::pair<cudaEvent_t, const ms_ctx*>& pr) { return pr.second == c; }),
                           L.peer_reads.end());
    for (auto& L : c->layers)
      for (auto& pr : L.peer_reads) cudaEventSynchronize(pr.first);
  }
  for (auto& L : c->layers) {
    for (int s = 0; s < kVariants; ++s) {
      cudaFree(L.d_table[s]);
      cudaFreeHost(L.h_table[s]);
      if (L.host_registered[s]) cudaHostUnregister(L.host_img[s]);
      else cudaFreeHost(L.host_img[s]);
    }
    if (L.ev_start) cudaEventDestroy(L.ev_start);
    if (L.ev_done) cudaEventDestroy(L.ev_done);
  }
  for (auto* p : c->raw) cudaFree(p);
  for (auto& st : c->ring) {
    cudaFreeHost(st.h);
    if (st.next_h) cudaFreeHost(st.next_h);
    if (st.done) cudaEventDestroy(st.done);
    cudaFree(st.d);
    if (st.used) cudaEventDestroy(st.used);
  }
  for (auto e : c->events) cudaEventDestroy(e);
  drop_graphs(c);
  for (auto e : c->prof_ev) cudaEventDestroy(e);
  if (c->trace_h) cudaFree(c->trace_h);
  if (c->tm0) cudaEventDestroy(c->tm0);
  if (c->tm1) cudaEventDestroy(c->tm1);
  if (c->ev_user_in) cudaEventDestroy(c->ev_user_in);
  if (c->ev_user_out) cudaEventDestroy(c->ev_user_out);
  if (c->ev_step0) cudaEventDestroy(c->ev_step0);
  if (c->ev_step1) cudaEventDestroy(c->ev_step1);
  void* dev[] = {c->arena, c->embed, c->normf, c->norms, c->lm_packed, c->lm_table, c->rope_cos, c->rope_sin,
                 c->h, c->x, c->x2, c->part, c->q, c->attn_ws, c->am_key, c->am_cnt, c->next, c->logits, c->hist};
  for (void* p : dev) cudaFree(p);
  cudaFreeHost(c->h_next);
  cudaFreeHost(c->h_logits);
  if (c->compute) cudaStreamDestroy(c->compute);
  if (c->copy) cudaStreamDestroy(c->copy);
  delete c;
  return MS_OK;
}

int ms_sync(ms_ctx* c) {
  return guard([&] {
    CK(cudaStreamSynchronize(c->compute));
    CK(cudaStreamSynchronize(c->copy));
  });
}

int ms_num_sms(ms_ctx* c) { return c ? c->num_sms : 0; }

// ------------------------------------------------------------------ weights
namespace {
struct TensorSpec {
  int64_t n;
  double scale, offset;
};
TensorSpec layer_tensor(const ms_model_desc& D, int which) {
  const int64_t d = D.hidden, qkv_n = (int64_t)(D.num_heads + 2 * D.num_kv_heads) * D.head_dim;
  switch (which) {
    case 0: case 3: return {d, 0.1, 1.0};
    case 1: return {qkv_n * d, 1.0 / std::sqrt((double)d), 0.0};
    case 2: return {d * D.num_heads * D.head_dim, 1.0 / std::sqrt((double)(D.num_heads * D.head_dim)), 0.0};
    case 4: return {2LL * D.ffn * d, 1.0 / std::sqrt((double)d), 0.0};
    default: return {d * D.ffn, 1.0 / std::sqrt((double)D.ffn), 0.0};
  }
}
int64_t expected_count(const ms_model_desc& D, int layer, int which) {
  if (layer < 0) return which == 1 ? D.hidden : (int64_t)D.vocab * D.hidden;
  return layer_tensor(D, which).n;
}
void finalize_weights(ms_ctx* c, bool synthetic, uint64_t seed) {
  const ms_model_desc& D = c->desc;
  const int d = D.hidden;
  const int64_t tmp_elems = std::max<int64_t>((int64_t)2 * D.ffn * d,
                                              (int64_t)(D.num_heads + 2 * D.num_kv_heads) * D.head_dim * d);
  uint16_t* wtmp[kMats] = {nullptr, nullptr, nullptr, nullptr};
  uint8_t* ptmp = nullptr;
  try {
    if (synthetic) {
      CK(ms::gen_weight_launch(seed, 0, (int64_t)D.vocab * d, 1.0, 0.0, c->embed, c->compute));
      CK(ms::gen_weight_launch(seed, 1, d, 0.1, 1.0, c->normf, c->compute));
      uint16_t* lm = nullptr;
      CK(cudaMalloc(&lm, (size_t)D.vocab * d * 2));
      CK(ms::gen_weight_launch(seed, 2, (int64_t)D.vocab * d, 1.0 / std::sqrt((double)d), 0.0, lm, c->compute));
      CK(ms::pack_bf16_launch(lm, D.vocab, d, c->lm_packed, c->compute));
      CK(cudaStreamSynchronize(c->compute));
      cudaFree(lm);
    } else {
      for (int w = 0; w < 3; ++w)
        if (!c->raw[(size_t)D.num_layers * 6 + w]) fail(MS_EVALIDATION, "missing global tensor upload");
      CK(cudaMemcpyAsync(c->embed, c->raw[(size_t)D.num_layers * 6 + 0], (size_t)D.vocab * d * 2,
                         cudaMemcpyDeviceToDevice, c->compute));
      CK(cudaMemcpyAsync(c->normf, c->raw[(size_t)D.num_layers * 6 + 1], (size_t)d * 2, cudaMemcpyDeviceToDevice,
                         c->compute));
      CK(ms::pack_bf16_launch(c->raw[(size_t)D.num_layers * 6 + 2], D.vocab, d, c->lm_packed, c->compute));
    }
    for (int m = 0; m < kMats; ++m) CK(cudaMalloc(&wtmp[m], (size_t)tmp_elems * 2));
    CK(cudaMalloc(&ptmp, (size_t)tmp_elems * 2));
    static const int mat_which[kMats] = {1, 2, 4, 5};
    for (int l = 0; l < D.num_layers; ++l) {
      for (int nrm = 0; nrm < 2; ++nrm) {
        uint16_t* dst = c->norms + ((size_t)l * 2 + nrm) * d;
        const int which = nrm == 0 ? 0 : 3;
        if (synthetic) {
          CK(ms::gen_weight_launch(seed, 16 + (uint64_t)l * 8 + which, d, 0.1, 1.0, dst, c->compute));
        } else {
          uint16_t* r = c->raw[(size_t)l * 6 + which];
          if (!r) fail(MS_EVALIDATION, "missing norm upload");
          CK(cudaMemcpyAsync(dst, r, (size_t)d * 2, cudaMemcpyDeviceToDevice, c->compute));
        }
      }
      for (int m = 0; m < kMats; ++m) {
        const int which = mat_which[m];
        if (synthetic) {
          const TensorSpec t = layer_tensor(D, which);
          CK(ms::gen_weight_launch(seed, 16 + (uint64_t)l * 8 + which, t.n, t.scale, t.offset, wtmp[m],
                                   c->compute));
        } else {
          uint16_t* r = c->raw[(size_t)l * 6 + which];
          if (!r) fail(MS_EVALIDATION, "missing layer tensor upload");
          CK(cudaMemcpyAsync(wtmp[m], r, (size_t)layer_tensor(D, which).n * 2, cudaMemcpyDeviceToDevice,
                             c->compute));
        }
      }
      build_images(c, l, wtmp, ptmp);
    }
    make_resident_bf16(c);
  } catch (...) {
    for (auto* p : wtmp) cudaFree(p);
    cudaFree(ptmp);
    throw;
  }
  for (auto* p : wtmp) cudaFree(p);
  cudaFree(ptmp);
  for (auto*& p : c->raw) {
    cudaFree(p);
    p = nullptr;
  }
}
}  // namespace

int ms_weights_synthetic(ms_ctx* c, uint64_t seed) {
  return guard([&] {
    c->graph_gen++;
    CK(cudaSetDevice(c->device));
    finalize_weights(c, true, seed);
  });
}

int ms_weights_upload(ms_ctx* c, int layer, int which, const uint16_t* host_bf16, int64_t count) {
  return guard([&] {
    const ms_model_desc& D = c->desc;
    if (layer < -1 || layer >= D.num_layers) fail(MS_EVALIDATION, "layer out of range");
    if (layer < 0 ? (which < 0 || which > 2) : (which < 0 || which > 5)) fail(MS_EVALIDATION, "bad tensor id");
    if (count != expected_count(D, layer, which)) fail(MS_EVALIDATION, "tensor element count mismatch");
    const size_t idx = layer < 0 ? (size_t)D.num_layers * 6 + which : (size_t)layer * 6 + which;
    if (!c->raw[idx]) CK(cudaMalloc(&c->raw[idx], (size_t)count * 2));
    CK(cudaMemcpy(c->raw[idx], host_bf16, (size_t)count * 2, cudaMemcpyHostToDevice));
  });
}

int ms_weights_finalize(ms_ctx* c) {
  return guard([&] {
    c->graph_gen++;
    CK(cudaSetDevice(c->device));
    finalize_weights(c, false, 0);
  });
}

int64_t ms_variant_bytes(ms_ctx* c, int bits) {
  if (!c || !valid_bits(bits) || c->geom[variant_of(bits)].pages < 0) return -1;
  return c->geom[variant_of(bits)].pages * c->page_bytes;
}

int ms_variant_enable(ms_ctx* c, int bits) {
  return guard([&] {
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "variant enable: bits must be 16, 8, 4 or 3");
    if (c->weights_ready) fail(MS_EVALIDATION, "variant enable: weights already finalized");
    if (c->geom[variant_of(bits)].pages < 0)
      fail(MS_EVALIDATION, "variant enable: page smaller than one " + std::to_string(bits) + "-bit weight chunk");
    c->variant_on[variant_of(bits)] = true;
  });
}

int ms_variant_export(ms_ctx* c, int layer, int bits, void* host_out, int64_t bytes) {
  return guard([&] {
    if (layer < 0 || layer >= c->desc.num_layers) fail(MS_EVALIDATION, "layer out of range");
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "bits must be 16, 8, 4 or 3");
    const Layer& L = c->layers[layer];
    const uint8_t* img = L.host_img[variant_of(bits)];
    if (!img) fail(MS_EVALIDATION, "variant store not built");
    const int64_t n = std::min<int64_t>(bytes, ms_variant_bytes(c, bits));
    std::memcpy(host_out, img, (size_t)n);
  });
}

int ms_variant_register(ms_ctx* c, int layer, int bits, void* host, int64_t bytes, int prefilled) {
  return guard([&] {
    if (layer < 0 || layer >= c->desc.num_layers) fail(MS_EVALIDATION, "variant register: layer out of range");
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "variant register: bits must be 16, 8, 4 or 3");
    if (!host || bytes < ms_variant_bytes(c, bits)) fail(MS_EVALIDATION, "variant register: buffer too small");
    if (c->weights_ready) fail(MS_EVALIDATION, "variant register: weights already finalized");
    Layer& L = c->layers[layer];
    const int bi = variant_of(bits);
    if (c->geom[bi].pages < 0) fail(MS_EVALIDATION, "variant register: page smaller than one weight chunk");
    if (L.host_img[bi]) fail(MS_EVALIDATION, "variant register: image already present");
    c->variant_on[bi] = true;
    CK(cudaSetDevice(c->device));
    const cudaError_t e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      cudaGetLastError();  // pinned already (e.g. cudaHostAlloc'd by the caller): use as is
    } else {
      CK(e);
      L.host_registered[bi] = true;
    }
    L.host_img[bi] = static_cast<uint8_t*>(host);
    L.host_ready[bi] = prefilled != 0;
  });
}

// ------------------------------------------------------------- LayerSwapper
int ms_swap_begin(ms_ctx* c, int layer, int bits, uint64_t* ticket) {
  return guard([&] {
    if (layer < 0 || layer >= c->desc.num_layers) fail(MS_EVALIDATION, "begin_swap: layer out of range");
    Layer& L = c->layers[layer];
    if (L.in_flight) fail(MS_EVALIDATION, "begin_swap: swap already in flight on layer");
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "begin_swap: bits must be 16, 8, 4 or 3");
    if (L.bits == bits) fail(MS_EVALIDATION, "begin_swap: layer already at target precision");
    if (!c->weights_ready) fail(MS_EVALIDATION, "weights not initialised");
    if (!L.host_img[variant_of(bits)])
      fail(MS_EVALIDATION, "begin_swap: no " + std::to_string(bits) + "-bit variant store (ms_variant_enable)");
    const ImageGeom& g = geom_of(c, bits);
    CK(cudaSetDevice(c->device));
    // the inactive table slot may still be read by steps launched before the
    // previous commit of this layer
    if (L.last_release) CK(cudaStreamWaitEvent(c->copy, L.last_release, 0));
    L.new_pages = take_pages(c, g.pages, c->copy);
    CK(cudaEventRecord(L.ev_start, c->copy));
    write_table(c, L, variant_of(bits), L.new_pages, c->copy);
    upload_image(c, L.host_img[variant_of(bits)], g, L.new_pages, c->copy);
    CK(cudaEventRecord(L.ev_done, c->copy));
    L.in_flight = true;
    L.to_bits = bits;
    L.ticket = (c->next_ticket++ << 16) | (uint64_t)layer;
    *ticket = L.ticket;
  });
}

// LayerSwapper, peer fetch: the variant image is copied
// from another context that holds this layer committed at `bits` (device to
// device, cudaMemcpyPeerAsync: NVLink between GPUs of one process) instead of
// uploaded from pinned host memory.  Poll / wait / commit as for ms_swap_begin.
int ms_swap_begin_peer(ms_ctx* c, int layer, int bits, ms_ctx* src, uint64_t* ticket) {
  return guard([&] {
    if (!src || src == c) fail(MS_EVALIDATION, "begin_swap_peer: bad source context");
    if (layer < 0 || layer >= c->desc.num_layers) fail(MS_EVALIDATION, "begin_swap_peer: layer out of range");
    const ms_model_desc &a = c->desc, &b = src->desc;
    if (a.num_layers != b.num_layers || a.hidden != b.hidden || a.num_heads != b.num_heads ||
        a.num_kv_heads != b.num_kv_heads || a.head_dim != b.head_dim || a.ffn != b.ffn ||
        a.block_tokens != b.block_tokens || c->page_bytes != src->page_bytes)
      fail(MS_EVALIDATION, "begin_swap_peer: source context has a different model geometry");
    Layer& L = c->layers[layer];
    Layer& S = src->layers[layer];
    if (L.in_flight) fail(MS_EVALIDATION, "begin_swap: swap already in flight on layer");
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "begin_swap: bits must be 16, 8, 4 or 3");
    if (L.bits == bits) fail(MS_EVALIDATION, "begin_swap: layer already at target precision");
    if (!c->weights_ready || !src->weights_ready) fail(MS_EVALIDATION, "weights not initialised");
    if (S.in_flight || S.bits != bits)
      fail(MS_EVALIDATION, "begin_swap_peer: source layer is not committed at " + std::to_string(bits) + " bits");
    CK(cudaSetDevice(c->device));
    if (src->device != c->device) {
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, c->device, src->device));
      if (!ok) fail(MS_ERUNTIME, "begin_swap_peer: no peer access between the devices");
      const cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else CK(e);
    }
    const ImageGeom& g = geom_of(c, bits);
    if (L.last_release) CK(cudaStreamWaitEvent(c->copy, L.last_release, 0));
    L.new_pages = take_pages(c, g.pages, c->copy);
    CK(cudaEventRecord(L.ev_start, c->copy));
    write_table(c, L, variant_of(bits), L.new_pages, c->copy);
    for (int64_t p = 0; p < g.pages; ++p) {
      const int64_t bytes = std::min<int64_t>(g.cpp, g.total_chunks - p * g.cpp) * g.chunk_bytes;
      CK(cudaMemcpyPeerAsync(c->arena + (int64_t)L.new_pages[p] * c->page_bytes, c->device,
                             src->arena + (int64_t)S.pages[p] * src->page_bytes, src->device, (size_t)bytes, c->copy));
    }
    CK(cudaEventRecord(L.ev_done, c->copy));
    cudaEvent_t rd = new_event(c);
    CK(cudaEventRecord(rd, c->copy));
    {
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      S.peer_reads.push_back({rd, c});
    }
    L.in_flight = true;
    L.to_bits = bits;
    L.ticket = (c->next_ticket++ << 16) | (uint64_t)layer;
    *ticket = L.ticket;
  });
}

namespace {
Layer& ticket_layer(ms_ctx* c, uint64_t ticket) {
  const int layer = (int)(ticket & 0xFFFF);
  if (layer >= c->desc.num_layers) fail(MS_EVALIDATION, "bad swap ticket");
  Layer& L = c->layers[layer];
  if (!L.in_flight || L.ticket != ticket) fail(MS_ELOGIC, "complete_swap: no swap in flight on layer");
  return L;
}
}  // namespace

int ms_swap_poll(ms_ctx* c, uint64_t ticket, int* done) {
  return guard([&] {
    Layer& L = ticket_layer(c, ticket);
    const cudaError_t e = cudaEventQuery(L.ev_done);
    if (e == cudaErrorNotReady) {
      *done = 0;
      return;
    }
    CK(e);
    *done = 1;
  });
}

int ms_swap_wait(ms_ctx* c, uint64_t ticket, float* upload_ms) {
  return guard([&] {
    Layer& L = ticket_layer(c, ticket);
    CK(cudaEventSynchronize(L.ev_done));
    if (upload_ms) CK(cudaEventElapsedTime(upload_ms, L.ev_start, L.ev_done));
  });
}

int ms_swap_commit(ms_ctx* c, uint64_t ticket, int64_t* pages_freed) {
  return guard([&] {
    // no graph invalidation: steps read the layer's page table from device
    // memory and graphs are keyed by the precision vector (see struct Layer)
    Layer& L = ticket_layer(c, ticket);
    CK(cudaSetDevice(c->device));
    // Token-boundary flip: steps launched from now on use the new image; the
    // compute stream orders them after the upload (no host sync, no flush).
    CK(cudaStreamWaitEvent(c->compute, L.ev_done, 0));
    {  // another context may still be copying the old image
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      for (auto& pr : L.peer_reads) CK(cudaEventSynchronize(pr.first));
      L.peer_reads.clear();
    }
    cudaEvent_t fence = compute_fence(c);  // after every step that read the old image
    const int64_t freed = (int64_t)L.pages.size();
    give_pages(c, L.pages, fence);
    L.pages = std::move(L.new_pages);
    L.new_pages.clear();
    L.bits = L.to_bits;
    L.slot = variant_of(L.bits);
    L.in_flight = false;
    L.last_release = fence;
    if (pages_freed) *pages_freed = freed;
  });
}

int ms_reset_state(ms_ctx* c) {
  return guard([&] {
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->compute));
    CK(cudaStreamSynchronize(c->copy));
    for (int l = 0; l < c->desc.num_layers; ++l)
      if (c->layers[l].in_flight) fail(MS_ELOGIC, "reset: swap in flight");
    // KV pages first: the BF16 restores below may need the pages the KV
    // resizer carved out of the W4 layers' freed images
    std::vector<int32_t> pages;
    for (auto& p : c->id_page)
      if (p >= 0) {
        pages.push_back(p);
        p = -1;
      }
    give_pages(c, pages, compute_fence(c));
    CK(cudaStreamSynchronize(c->compute));
    for (int l = 0; l < c->desc.num_layers; ++l) {
      if (c->layers[l].bits == 16) continue;
      uint64_t t = 0;
      if (ms_swap_begin(c, l, 16, &t) != MS_OK) fail(MS_ERUNTIME, g_err);
      CK(cudaStreamSynchronize(c->copy));
      if (ms_swap_commit(c, t, nullptr) != MS_OK) fail(MS_ERUNTIME, g_err);
    }
    CK(cudaStreamSynchronize(c->compute));
  });
}

int ms_layer_bits(ms_ctx* c, int layer) {
  if (!c || layer < 0 || layer >= c->desc.num_layers) return -1;
  return c->layers[layer].bits;
}

// ---------------------------------------------------------------- KV resizer
int ms_kv_attach(ms_ctx* c, int64_t first_id, int64_t n) {
  return guard([&] {
    if (n < 1) fail(MS_EVALIDATION, "kv attach: count must be >= 1");
    if (first_id < 0) fail(MS_EVALIDATION, "kv attach: negative id");
    for (int64_t id = first_id; id < first_id + n; ++id)
      if (id < (int64_t)c->id_page.size() && c->id_page[id] >= 0) fail(MS_EVALIDATION, "kv attach: id already mapped");
    std::vector<int32_t> pages = take_pages(c, n, c->compute);
    if ((int64_t)c->id_page.size() < first_id + n) c->id_page.resize(first_id + n, -1);
    for (int64_t i = 0; i < n; ++i) c->id_page[first_id + i] = pages[i];
  });
}

int ms_kv_detach(ms_ctx* c, const int64_t* ids, int64_t n) {
  return guard([&] {
    if (n < 0 || (n > 0 && !ids)) fail(MS_EVALIDATION, "kv detach: bad id list");
    // validate every id (mapped, no duplicates) before unmapping any of them
    std::vector<int32_t> pages;
    pages.reserve(n);
    for (int64_t i = 0; i < n; ++i) pages.push_back(page_of(c, ids[i]));
    std::vector<int64_t> sorted(ids, ids + n);
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
      fail(MS_EVALIDATION, "kv detach: duplicate block id");
    for (int64_t i = 0; i < n; ++i) c->id_page[ids[i]] = -1;
    give_pages(c, pages, compute_fence(c));
  });
}

int64_t ms_free_pages(ms_ctx* c) { return c ? (int64_t)c->free_pages.size() : -1; }

int64_t ms_kv_page_of(ms_ctx* c, int64_t id) {
  if (!c || id < 0 || id >= (int64_t)c->id_page.size()) return -1;
  return c->id_page[id];
}

int ms_kv_export(ms_ctx* c, int64_t id, void* host_out, int64_t bytes) {
  return guard([&] {
    if (!host_out || bytes < c->page_bytes) fail(MS_EVALIDATION, "kv export: buffer smaller than one page");
    const int32_t page = page_of(c, id);
    CK(cudaMemcpyAsync(host_out, c->arena + (int64_t)page * c->page_bytes, c->page_bytes, cudaMemcpyDeviceToHost,
                       c->compute));
    CK(cudaStreamSynchronize(c->compute));
  });
}

// ------------------------------------------------------------ token history
int ms_hist_reserve(ms_ctx* c, int32_t slots, int32_t max_len) {
  return guard([&] {
    c->graph_gen++;  // the token history is re-allocated
    if (slots < 1 || max_len < 2) fail(MS_EVALIDATION, "bad history shape");
    if (max_len > c->desc.max_pos + 1) fail(MS_EVALIDATION, "history longer than max_pos");
    CK(cudaStreamSynchronize(c->compute));
    if (c->hist) cudaFree(c->hist);
    c->hist = nullptr;
    CK(cudaMalloc(&c->hist, (size_t)slots * max_len * sizeof(int32_t)));
    CK(cudaMemset(c->hist, 0, (size_t)slots * max_len * sizeof(int32_t)));
    c->hist_slots = slots;
    c->hist_len = max_len;
  });
}

int ms_hist_write(ms_ctx* c, int32_t slot, int32_t offset, const int32_t* host_tokens, int32_t n) {
  return guard([&] {
    if (!c->hist || slot < 0 || slot >= c->hist_slots || offset < 0 || offset + n > c->hist_len)
      fail(MS_EVALIDATION, "history write out of range");
    for (int i = 0; i < n; ++i)
      if (host_tokens[i] < 0 || host_tokens[i] >= c->desc.vocab) fail(MS_EVALIDATION, "token id out of vocab");
    Staging& st = next_staging(c, (size_t)n);
    std::memcpy(st.h, host_tokens, (size_t)n * 4);
    hist_in_kernel<<<(n + 255) / 256, 256, 0, c->compute>>>(st.hd, c->hist + (size_t)slot * c->hist_len + offset, n);
    CK(cudaGetLastError());
    c->launches += 1;
    CK(cudaEventRecord(st.used, c->compute));
    st.armed = true;
  });
}

int ms_hist_read(ms_ctx* c, int32_t slot, int32_t offset, int32_t* host_out, int32_t n) {
  return guard([&] {
    if (!c->hist || slot < 0 || slot >= c->hist_slots || offset < 0 || offset + n > c->hist_len)
      fail(MS_EVALIDATION, "history read out of range");
    CK(cudaMemcpyAsync(host_out, c->hist + (size_t)slot * c->hist_len + offset, (size_t)n * 4,
                       cudaMemcpyDeviceToHost, c->compute));
    CK(cudaStreamSynchronize(c->compute));
  });
}

// -------------------------------------------------------------------- steps
namespace {
// Enqueue one decode step; returns the staging slot used.
// caller-stream ordering around a step (no-ops without ms_set_stream)
void user_enter(ms_ctx* c) {
  if (!c->user) return;
  CK(cudaEventRecord(c->ev_user_in, c->user));
  CK(cudaStreamWaitEvent(c->compute, c->ev_user_in, 0));
}
void user_leave(ms_ctx* c) {
  if (!c->user) return;
  CK(cudaEventRecord(c->ev_user_out, c->compute));
  CK(cudaStreamWaitEvent(c->user, c->ev_user_out, 0));
}

int decode_enqueue(ms_ctx* c, const ms_decode_batch* b, bool want_logits) {
    check_ready(c);
    const int n = b->n;
    if (n < 1 || n > c->desc.max_batch) fail(MS_EVALIDATION, "decode batch size out of range");
    const int mb = c->max_blocks;
    // staging: slot[n] pos[n] ctx[n] tok[n] pages[n][mb]
    Staging& st = next_staging(c, (size_t)n * (4 + mb));
    int32_t* hs = st.h;
    int max_ctx = 0;
    for (int i = 0; i < n; ++i) {
      const int slot = b->slots[i], pos = b->positions[i];
      if (slot < 0 || slot >= c->hist_slots) fail(MS_EVALIDATION, "slot out of range");
      if (pos < 0 || pos + 1 >= c->hist_len || pos >= c->desc.max_pos) fail(MS_EVALIDATION, "position out of range");
      hs[i] = slot;
      hs[n + i] = pos;
      hs[2 * n + i] = pos + 1;
      hs[3 * n + i] = b->tokens ? b->tokens[i] : 0;
      if (b->tokens && (b->tokens[i] < 0 || b->tokens[i] >= c->desc.vocab)) fail(MS_EVALIDATION, "token out of vocab");
      max_ctx = std::max(max_ctx, pos + 1);
      const int nb = pos / c->desc.block_tokens + 1;
      if (nb > b->max_blocks) fail(MS_EVALIDATION, "block table narrower than the context");
      int32_t* row = hs + 4 * n + (size_t)i * mb;
      for (int j = 0; j < nb; ++j) row[j] = page_of(c, b->block_ids[(size_t)i * b->max_blocks + j]);
    }
    CK(cudaSetDevice(c->device));
    user_enter(c);
    CK(cudaEventRecord(c->ev_step0, c->compute));
    stage_in(c, st, (size_t)n * (4 + mb));
    CK(cudaEventRecord(st.used, c->compute));
    st.armed = true;
    const int32_t* d_slot = st.d;
    const int32_t* d_pos = st.d + n;
    const int32_t* d_ctx = st.d + 2 * n;
    const int32_t* d_tok = st.d + 3 * n;
    const int32_t* d_pages = st.d + 4 * n;
    if (b->tokens) {
      hist_scatter_kernel<<<(n + 127) / 128, 128, 0, c->compute>>>(c->hist, c->hist_len, d_slot, d_pos, d_tok, n);
      CK(cudaGetLastError());
      c->launches += 1;
    }
    const int TM = std::min(256, round16(n));
    if (graphs_enabled() && !c->prof_attn && !c->prof_all && !c->tracing) {
      if (c->graph_gen != c->graph_gen_built) {
        drop_graphs(c);
        c->graph_gen_built = c->graph_gen;
      }
      const int asplits = attn_splits(c, n, max_ctx);
      const int wl = want_logits;
      std::vector<int8_t> bits(c->layers.size());
      uint64_t bits_hash = 1469598103934665603ull;
      for (size_t l = 0; l < bits.size(); ++l) {
        bits[l] = (int8_t)c->layers[l].bits;
        bits_hash = (bits_hash ^ (uint64_t)(uint8_t)bits[l]) * 1099511628211ull;
      }
      ms_ctx::StepGraph* g = nullptr;
      for (auto& x : c->graphs)
        if (x.st_d == st.d && x.n == n && x.mb == mb && x.asplits == asplits && x.want_logits == wl &&
            x.has_tokens == 0 && x.bits == bits)
          g = &x;
      bool capture = false;
      if (!g) {
        const std::array<int64_t, 6> key{(int64_t)st.d, n, mb, asplits, wl, (int64_t)bits_hash};
        auto it = std::find(c->graph_seen.begin(), c->graph_seen.end(), key);
        if (it == c->graph_seen.end()) {
          if (c->graph_seen.size() >= 4 * kMaxGraphs) c->graph_seen.clear();
          c->graph_seen.push_back(key);
        } else {
          capture = true;
          if (c->graphs.size() >= kMaxGraphs) drop_graphs(c);
        }
      }
      if (!g && !capture) {
        forward(c, n, TM, d_slot, d_pos, d_ctx, nullptr, d_pages, nullptr, mb, max_ctx, 0, wl != 0);
      } else if (!g) {  // capture the forward once for this shape / staging slot
        cudaGraph_t graph;
        const int64_t l0 = c->launches;
        CK(cudaStreamBeginCapture(c->compute, cudaStreamCaptureModeThreadLocal));
        forward(c, n, TM, d_slot, d_pos, d_ctx, nullptr, d_pages, nullptr, mb, max_ctx, 0, wl != 0);
        CK(cudaStreamEndCapture(c->compute, &graph));
        cudaGraphExec_t exec;
        CK(cudaGraphInstantiate(&exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        c->graphs.push_back({st.d, n, mb, asplits, wl, 0, bits, c->launches - l0, exec});
        c->graph_captures += 1;
        c->launches = l0;
        g = &c->graphs.back();
      }
      if (g) {
        CK(cudaGraphLaunch(g->exec, c->compute));
        c->launches += g->launches;
      }
    } else {
      forward(c, n, TM, d_slot, d_pos, d_ctx, nullptr, d_pages, nullptr, mb, max_ctx, 0, want_logits);
    }
    CK(cudaEventRecord(c->ev_step1, c->compute));
    user_leave(c);
    return (int)(&st - c->ring);
}
}  // namespace

int ms_set_stream(ms_ctx* c, void* stream) {
  return guard([&] {
    CK(cudaSetDevice(c->device));
    if (!c->ev_user_in) {
      CK(cudaEventCreateWithFlags(&c->ev_user_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_user_out, cudaEventDisableTiming));
    }
    c->user = static_cast<cudaStream_t>(stream);
  });
}

int ms_decode_step(ms_ctx* c, const ms_decode_batch* b, int32_t* next_out, float* logits_out) {
  return guard([&] {
    const int n = b->n;
    decode_enqueue(c, b, logits_out != nullptr);
    if (next_out || logits_out) {
      if (next_out) CK(cudaMemcpyAsync(c->h_next, c->next, (size_t)n * 4, cudaMemcpyDeviceToHost, c->compute));
      if (logits_out)
        CK(cudaMemcpyAsync(c->h_logits, c->logits, (size_t)n * c->desc.vocab * 4, cudaMemcpyDeviceToHost,
                           c->compute));
      CK(cudaStreamSynchronize(c->compute));
      if (next_out) std::memcpy(next_out, c->h_next, (size_t)n * 4);
      if (logits_out) std::memcpy(logits_out, c->h_logits, (size_t)n * c->desc.vocab * 4);
    }
  });
}

int ms_decode_submit(ms_ctx* c, const ms_decode_batch* b) {
  return guard([&] {
    if ((int)c->submitted.size() >= kRing - 1 || c->ring[c->ring_i].pending)
      fail(MS_EVALIDATION, "decode_submit: collect the oldest step first (at most 2 in flight)");
    const int i = decode_enqueue(c, b, false);
    Staging& st = c->ring[i];
    if (!st.next_h) {
      CK(cudaHostAlloc(&st.next_h, (size_t)c->max_rows * sizeof(int32_t), cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
    }
    CK(cudaMemcpyAsync(st.next_h, c->next, (size_t)b->n * 4, cudaMemcpyDeviceToHost, c->compute));
    CK(cudaEventRecord(st.done, c->compute));
    st.next_n = b->n;
    st.pending = true;
    c->submitted.push_back(i);
  });
}

int ms_decode_collect(ms_ctx* c, int32_t* next_out, int32_t* n_out) {
  return guard([&] {
    if (c->submitted.empty()) fail(MS_EVALIDATION, "decode_collect: no submitted step");
    Staging& st = c->ring[c->submitted.front()];
    c->submitted.erase(c->submitted.begin());
    CK(cudaEventSynchronize(st.done));
    if (next_out) std::memcpy(next_out, st.next_h, (size_t)st.next_n * 4);
    if (n_out) *n_out = st.next_n;
    st.pending = false;
  });
}

int ms_prefill(ms_ctx* c, int32_t slot, int32_t n_tokens, const int64_t* block_ids, int32_t n_blocks,
               int32_t* next_out, float* logits_out) {
  return guard([&] {
    check_ready(c);
    const int n = n_tokens;
    if (n < 1 || n > c->desc.max_prefill_tokens) fail(MS_EVALIDATION, "prefill length out of range");
    if (slot < 0 || slot >= c->hist_slots || n + 1 > c->hist_len) fail(MS_EVALIDATION, "prefill slot/length");
    const int nb = (n + c->desc.block_tokens - 1) / c->desc.block_tokens;
    if (n_blocks < nb) fail(MS_EVALIDATION, "prefill needs more blocks");
    const int mb = c->max_blocks;
    Staging& st = next_staging(c, (size_t)n * 4 + mb);
    int32_t* hs = st.h;
    for (int i = 0; i < n; ++i) {
      hs[i] = slot;
      hs[n + i] = i;
      hs[2 * n + i] = i + 1;
      hs[3 * n + i] = 0;  // page_row
    }
    int32_t* row = hs + 4 * n;
    for (int j = 0; j < nb; ++j) row[j] = page_of(c, block_ids[j]);
    CK(cudaSetDevice(c->device));
    user_enter(c);
    CK(cudaEventRecord(c->ev_step0, c->compute));
    stage_in(c, st, (size_t)n * 4 + mb);
    CK(cudaEventRecord(st.used, c->compute));
    st.armed = true;
    const int TM = std::min(256, round16(n));
    forward(c, n, TM, st.d, st.d + n, st.d + 2 * n, nullptr, st.d + 4 * n, st.d + 3 * n, 0, n, n - 1,
            logits_out != nullptr);
    CK(cudaEventRecord(c->ev_step1, c->compute));
    user_leave(c);
    if (next_out || logits_out) {
      if (next_out) CK(cudaMemcpyAsync(c->h_next, c->next, 4, cudaMemcpyDeviceToHost, c->compute));
      if (logits_out)
        CK(cudaMemcpyAsync(c->h_logits, c->logits, (size_t)c->desc.vocab * 4, cudaMemcpyDeviceToHost, c->compute));
      CK(cudaStreamSynchronize(c->compute));
      if (next_out) *next_out = c->h_next[0];
      if (logits_out) std::memcpy(logits_out, c->h_logits, (size_t)c->desc.vocab * 4);
    }
  });
}

int ms_prefill_trace(ms_ctx* c, int32_t slot, int32_t n_tokens, const int64_t* block_ids, int32_t n_blocks,
                     float* h_out, float* logits_out) {
  return guard([&] {
    if (!h_out) fail(MS_EVALIDATION, "prefill_trace: h_out is required");
    const size_t need = (size_t)(c->desc.num_layers + 1) * n_tokens * c->desc.hidden;
    if (n_tokens < 1 || n_tokens > c->desc.max_prefill_tokens) fail(MS_EVALIDATION, "prefill length out of range");
    CK(cudaSetDevice(c->device));
    if (c->trace_elems < need) {
      if (c->trace_h) CK(cudaFree(c->trace_h));
      CK(cudaMalloc(&c->trace_h, need * sizeof(float)));
      c->trace_elems = need;
    }
    c->tracing = true;
    const int rc = ms_prefill(c, slot, n_tokens, block_ids, n_blocks, nullptr, logits_out);
    c->tracing = false;
    if (rc != MS_OK) fail(rc, ms_last_error());
    // on the compute stream: a plain cudaMemcpy would not wait for the (non-blocking) compute stream
    CK(cudaMemcpyAsync(h_out, c->trace_h, need * sizeof(float), cudaMemcpyDeviceToHost, c->compute));
    CK(cudaStreamSynchronize(c->compute));
  });
}

int ms_last_step_ms(ms_ctx* c, float* ms_out) {
  return guard([&] {
    CK(cudaEventSynchronize(c->ev_step1));
    CK(cudaEventElapsedTime(ms_out, c->ev_step0, c->ev_step1));
  });
}

int ms_kv_fill_synthetic(ms_ctx* c, const int64_t* ids, int64_t n, uint64_t seed) {
  return guard([&] {
    std::vector<int32_t> pages(n);
    for (int64_t i = 0; i < n; ++i) pages[i] = page_of(c, ids[i]);
    int32_t* d = nullptr;
    CK(cudaMalloc(&d, (size_t)n * 4));
    CK(cudaMemcpyAsync(d, pages.data(), (size_t)n * 4, cudaMemcpyHostToDevice, c->compute));
    CK(ms::fill_kv_launch(c->kv, d, (int)n, seed, c->compute));
    CK(cudaStreamSynchronize(c->compute));
    cudaFree(d);
  });
}

// ------------------------------------------------------------ instrumentation
int64_t ms_launch_count(ms_ctx* c) { return c ? c->launches : -1; }
int64_t ms_graph_captures(ms_ctx* c) { return c ? c->graph_captures : -1; }

int ms_timer_start(ms_ctx* c) {
  return guard([&] {
    if (!c->tm0) {
      CK(cudaEventCreate(&c->tm0));
      CK(cudaEventCreate(&c->tm1));
    }
    CK(cudaEventRecord(c->tm0, c->compute));
  });
}

int ms_timer_stop(ms_ctx* c, float* ms_out) {
  return guard([&] {
    CK(cudaEventRecord(c->tm1, c->compute));
    CK(cudaEventSynchronize(c->tm1));
    CK(cudaEventElapsedTime(ms_out, c->tm0, c->tm1));
  });
}

int ms_prof_kernels(ms_ctx* c, int enable) {
  return guard([&] {
    c->prof_all = enable != 0;
    c->pk_used = 0;
  });
}

int ms_prof_kernels_read(ms_ctx* c, float* ms_out, int64_t* launches_out) {
  return guard([&] {
    CK(cudaStreamSynchronize(c->compute));
    for (int k = 0; k < MS_PK_COUNT; ++k) {
      ms_out[k] = 0.f;
      launches_out[k] = 0;
    }
    for (size_t i = 1; i < c->pk_used; ++i) {
      const int cat = c->pk_cat[i];
      if (cat < 0 || c->pk_cat[i - 1] == MS_PK_ARGMAX) continue;  // step start: gap between steps not counted
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->pk_ev[i - 1], c->pk_ev[i]));
      ms_out[cat] += ms;
      launches_out[cat] += 1;
    }
    c->pk_used = 0;
  });
}

int ms_prof_attention(ms_ctx* c, int enable) {
  return guard([&] {
    c->prof_attn = enable != 0;
    c->prof_used = 0;
  });
}

int ms_prof_attention_read(ms_ctx* c, float* total_ms, int64_t* launches) {
  return guard([&] {
    CK(cudaStreamSynchronize(c->compute));
    double t = 0.0;
    for (size_t i = 0; i + 1 < c->prof_used; i += 2) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->prof_ev[i], c->prof_ev[i + 1]));
      t += ms;
    }
    *total_ms = (float)t;
    *launches = (int64_t)(c->prof_used / 2);
  });
}

// ------------------------------------------------------ kernel-level (tests)
int ms_k_gen_weight(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset, uint16_t* out,
                    void* stream) {
  return guard([&] { CK(ms::gen_weight_launch(seed, tensor, n, scale, offset, out, (cudaStream_t)stream)); });
}
int ms_k_pack_bf16(const uint16_t* w, int N, int K, uint16_t* out, void* stream) {
  return guard([&] {
    if (N % 128 || K % 64) fail(MS_EVALIDATION, "pack_bf16: N%128, K%64");
    CK(ms::pack_bf16_launch(w, N, K, out, (cudaStream_t)stream));
  });
}
int ms_k_quant(int bits, const uint16_t* w, int N, int K, uint8_t* out, int8_t* codes_out, void* stream) {
  return guard([&] {
    if (bits != 8 && bits != 4 && bits != 3) fail(MS_EVALIDATION, "quant: bits must be 8, 4 or 3");
    if (N % 128 || K % 128) fail(MS_EVALIDATION, "quant: N%128, K%128");
    CK(ms::quant_launch(w, N, K, bits, out, codes_out, (cudaStream_t)stream));
  });
}

int ms_k_quant_w4(const uint16_t* w, int N, int K, uint8_t* out, int8_t* codes_out, void* stream) {
  return guard([&] {
    if (N % 128 || K % 128) fail(MS_EVALIDATION, "quant_w4: N%128, K%128");
    CK(ms::quant_launch(w, N, K, 4, out, codes_out, (cudaStream_t)stream));
  });
}
int ms_k_pack_act(const uint16_t* x, int M, int K, int TM, uint16_t* out, void* stream) {
  return guard([&] {
    if (K % 64 || TM % 16 || TM < 16 || TM > 256) fail(MS_EVALIDATION, "pack_act: K%64, TM in 16..256 step 16");
    CK(ms::pack_act_launch(x, M, K, TM, out, (cudaStream_t)stream));
  });
}
int ms_k_gemm(int bits, const void* w_packed, int N, int K, const uint16_t* x_packed, int M, int TM, int splits,
              float* out, int* splits_used, void* stream) {
  return guard([&] {
    if (!valid_bits(bits)) fail(MS_EVALIDATION, "gemm: bits must be 16, 8, 4 or 3");
    if (N % 128 || K % 128 || M < 1 || TM % 16 || TM < 16 || TM > 256) fail(MS_EVALIDATION, "gemm: bad shape");
    // one-entry page table per contiguous packed matrix (up to 1024 distinct
    // matrices; written once, so later calls may be graph-captured)
    static thread_local uint64_t* tables = nullptr;
    static thread_local std::vector<uint64_t> known;
    if (!tables) CK(cudaMalloc(&tables, 1024 * sizeof(uint64_t)));
    const uint64_t addr = (uint64_t)w_packed;
    size_t idx = std::find(known.begin(), known.end(), addr) - known.begin();
    if (idx == known.size()) {
      if (known.size() == 1024) fail(MS_EVALIDATION, "gemm: more than 1024 distinct weight matrices");
      CK(cudaMemcpyAsync(tables + idx, &addr, sizeof(addr), cudaMemcpyHostToDevice, (cudaStream_t)stream));
      CK(cudaStreamSynchronize((cudaStream_t)stream));
      known.push_back(addr);
    }
    uint64_t* table = tables + idx;
    ms::GemmWeights w{table, 0, (int64_t)1 << 40, N, K};
    const int wk = ms::wkind_of_bits(bits);
    ms::gemm_inline_pages(w, wk, &addr);
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // `splits` > 0 caps the persistent CTA count (exercises other partitions)
    const int ctas = splits > 0 ? std::min(splits, sms) : sms;
    ms::GemmPlanDev plan = ms::gemm_plan(N, K, M, TM, wk, ctas, (size_t)16 * M * N);
    CK(ms::gemm_launch(w, wk, x_packed, M, TM, plan, out, (cudaStream_t)stream));
    // slots actually written per tile are part_slots() <= plan.slots; slots a
    // tile does not use are left untouched (callers pass a zeroed buffer)
    if (splits_used) *splits_used = plan.aligned ? 1 : plan.slots;
  });
}

int ms_k_attn_decode(const float* q, const void* arena, int64_t page_bytes, int layers, int layer, int H, int KVH,
                     int hd, const int32_t* pages, int max_blocks, const int32_t* ctx_len, int rows, int splits,
                     float* workspace, uint16_t* out, void* stream) {
  return guard([&] {
    ms::AttnArgs a{};
    a.q = q;
    a.kv = ms::KvGeom{(char*)arena, page_bytes, layers, KVH, hd, 16};
    a.layer = layer;
    a.pages = pages;
    a.page_row = nullptr;
    a.page_stride = max_blocks;
    a.ctx_len = ctx_len;
    a.rows = rows;
    a.H = H;
    a.KVH = KVH;
    a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    a.splits = splits < 1 ? 1 : splits;
    a.part_o = workspace;
    a.part_ml = workspace ? workspace + (size_t)a.splits * rows * H * hd : nullptr;
    a.out = out;
    a.out_packed = 0;
    a.TM = 16;
    {  // arena extent for the GQA path's tensor map: pages referenced by the table
      std::vector<int32_t> hp((size_t)rows * max_blocks);
      CK(cudaMemcpy(hp.data(), pages, hp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
      int32_t mx = 0;
      for (int32_t v : hp) mx = std::max(mx, v);
      a.arena_bytes = (int64_t)(mx + 1) * page_bytes;
    }
    if (a.splits > 1 && !workspace) fail(MS_EVALIDATION, "attn: split-KV needs a workspace");
    CK(ms::attn_decode_launch(a, (cudaStream_t)stream));
  });
}

int ms_k_attn_prefill(const float* q, const void* arena, int64_t page_bytes, int layers, int layer, int H, int KVH,
                      int hd, const int32_t* pages, int n, uint16_t* out, void* stream) {
  return guard([&] {
    ms::PrefillAttnArgs a{};
    a.q = q;
    a.kv = ms::KvGeom{(char*)arena, page_bytes, layers, KVH, hd, 16};
    a.layer = layer;
    a.pages = pages;
    a.n = n;
    a.H = H;
    a.KVH = KVH;
    a.scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
    a.out = out;
    a.TM = 0;
    if (n < 1 || H % KVH) fail(MS_EVALIDATION, "attn_prefill: bad shape");
    {  // arena extent for the tensor map: pages the sequence references
      std::vector<int32_t> hp((size_t)(n + 15) / 16);
      CK(cudaMemcpy(hp.data(), pages, hp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
      int32_t mx = 0;
      for (int32_t v : hp) mx = std::max(mx, v);
      a.arena_bytes = (int64_t)(mx + 1) * page_bytes;
    }
    CK(ms::prefill_attn_launch(a, (cudaStream_t)stream));
  });
}

}  // extern "C"
