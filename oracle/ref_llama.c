/*
 * oracle/ref_llama.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this file's library (oracle/_lib/libref_llama.so), and only as the checker.
 * The product (paper_2506_02006_b200/) never links, imports or calls it.
 *
 * What it restates:
 *  - The reference's quantizer (proj/src/toy_model.cpp:40-60,
 *    quantize_row_scale / quantize_weights): symmetric round-to-nearest,
 *    scale = max|w| / (2^(b-1) - 1) in fp64, code = std::round(w / scale)
 *    (half away from zero), all-zero group => scale 1, codes 0.  The group is
 *    128 consecutive K elements of a row instead of the whole row (SURVEY
 *    8(c): "g128 grouping").  Pinned against the compiled reference via
 *    tests/golden (see tests/golden/make_golden.py).
 *  - The reference's per-layer precision dispatch inside one forward
 *    (proj/src/toy_model.cpp:139-168, `model.weights(p, config.tags[p])` at
 *    :153): every layer picks its BF16 or dequantized-W4 weights from its tag.
 *  - The reference has NO Llama forward (SPEC.md:14 puts kernels out of
 *    scope).  The Llama-style decoder below is this repo's own definition of
 *    the math the GPU path must compute: it is
 *    "parity unpinned" against the reference and pinned only by the frozen
 *    fixtures under tests/golden.  Rounding points mirror the GPU kernels:
 *      residual stream fp32; GEMM inputs rounded to bf16; fp64 accumulation;
 *      RoPE (rotate-half) in fp32 from a host fp64 table; K/V cached as bf16;
 *      softmax fp32; attention output rounded to bf16; SiLU(g)*u rounded to
 *      bf16; greedy argmax with ties to the lowest index.
 *  - A counter-based weight generator (splitmix64 of (seed, tensor, index))
 *    that the GPU generator reproduces bit for bit.
 *
 * Plain C11 + OpenMP, no dependencies.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ bf16 */
static inline float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
  uint32_t r = ((u >> 16) & 1u) + 0x7fffu;
  return (uint16_t)((u + r) >> 16);
}
float ref_bf16_to_float(uint16_t b) { return bf2f(b); }
uint16_t ref_float_to_bf16(float f) { return f2bf(f); }

/* ------------------------------------------------------- weight generator */
static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
/* value = offset + scale * u,  u uniform in [-1, 1): fp64 then fp32 then bf16 */
static inline uint16_t gen_one(uint64_t seed, uint64_t tensor, uint64_t idx, double scale,
                               double offset) {
  uint64_t key = seed ^ (tensor * 0xD1B54A32D192ED03ull);
  uint64_t r = splitmix64(key + idx);
  double u = (double)(r >> 11) * 0x1.0p-53;
  double w = 2.0 * u - 1.0;
  w = w * scale;
  w = w + offset;
  return f2bf((float)w);
}
void ref_gen_weight(uint64_t seed, uint64_t tensor, int64_t n, double scale, double offset,
                    uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = gen_one(seed, tensor, (uint64_t)i, scale, offset);
}

/* Tensor ids (shared convention with the GPU generator). */
enum { T_EMBED = 0, T_NORMF = 1, T_LMHEAD = 2 };
static inline uint64_t t_layer(int l, int which) { return 16u + (uint64_t)l * 8u + (uint64_t)which; }
enum { W_NORM1 = 0, W_QKV = 1, W_O = 2, W_NORM2 = 3, W_GU = 4, W_DOWN = 5 };

/* ----------------------------------------------------------- quantizer */
/* Per group of `group` K-elements of each row of a row-major [N][K] bf16
 * matrix.  Mirrors toy_model.cpp:40-60 (per row there, per group here). */
void ref_quantize_groups(const uint16_t* w, int64_t N, int64_t K, int group, int bits,
                         int8_t* codes, double* scales_f64, uint16_t* scales_bf16) {
  const int64_t G = K / group;
  const double qmax = (double)((1 << (bits - 1)) - 1);
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    for (int64_t g = 0; g < G; ++g) {
      const uint16_t* src = w + n * K + g * group;
      double max_abs = 0.0;
      for (int i = 0; i < group; ++i) {
        double a = fabs((double)bf2f(src[i]));
        if (a > max_abs) max_abs = a;
      }
      double scale = 1.0;
      int8_t* dst = codes + n * K + g * group;
      if (max_abs == 0.0) {
        for (int i = 0; i < group; ++i) dst[i] = 0;
      } else {
        scale = max_abs / qmax;
        for (int i = 0; i < group; ++i) dst[i] = (int8_t)round((double)bf2f(src[i]) / scale);
      }
      if (scales_f64) scales_f64[n * G + g] = scale;
      if (scales_bf16) scales_bf16[n * G + g] = f2bf((float)scale);
    }
  }
}

/* W4A16 dequantization contract: bf16(code * float(scale_bf16)), one RNE. */
void ref_dequant_w4(const int8_t* codes, const uint16_t* scales_bf16, int64_t N, int64_t K,
                    int group, uint16_t* out) {
  const int64_t G = K / group;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < K; ++k)
      out[n * K + k] = f2bf((float)codes[n * K + k] * bf2f(scales_bf16[n * G + k / group]));
}

/* ----------------------------------------------- device layout restatement */
/* BF16 weight chunk layout: chunk (n_tile, kb)
 * holds rows [128*n_tile, +128) x cols [64*kb, +64) as
 * [row_group 16][k_chunk 8][row 8][8 elems]; chunks ordered n_tile-major. */
void ref_pack_bf16(const uint16_t* w, int64_t N, int64_t K, uint16_t* out) {
  const int64_t KB = K / 64;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    const int64_t nt = n / 128, rr = n % 128, g = rr / 8, r = rr % 8;
    for (int64_t k = 0; k < K; ++k) {
      const int64_t kb = k / 64, kk = k % 64, c = kk / 8, e = kk % 8;
      const int64_t chunk = nt * KB + kb;
      out[chunk * 8192 + ((g * 8 + c) * 8 + r) * 8 + e] = w[n * K + k];
    }
  }
}

/* W4 chunk layout: chunk (n_tile, group g of 128 K) = 8448 bytes:
 *   bytes [0, 8192): codes as [j 4][row 128][16 B]; the 16 B of (j,row) hold
 *   K-elements [32j, 32j+32) of the group, 4 u32 words, word w holds elements
 *   32j+8w .. +7 stored as (code + 8): even elements e=2i in the low half at
 *   bits 4i, odd elements e=2i+1 in the high half at bits 16+4i (so that
 *   (word >> 4i) & 0x000F000F is the bf16x2 pair (e_2i, e_2i+1)).
 *   bytes [8192, 8448): 128 bf16 scales, one per row. */
void ref_pack_w4(const int8_t* codes, const uint16_t* scales_bf16, int64_t N, int64_t K,
                 uint8_t* out) {
  const int64_t G = K / 128;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    const int64_t nt = n / 128, row = n % 128;
    for (int64_t g = 0; g < G; ++g) {
      uint8_t* chunk = out + (nt * G + g) * 8448;
      for (int j = 0; j < 4; ++j) {
        uint32_t words[4];
        for (int w = 0; w < 4; ++w) {
          uint32_t v = 0;
          for (int e = 0; e < 8; ++e) {
            int k = g * 128 + j * 32 + w * 8 + e;
            uint32_t nib = (uint32_t)(codes[n * K + k] + 8) & 0xFu;
            v |= nib << ((e & 1) * 16 + (e >> 1) * 4);
          }
          words[w] = v;
        }
        memcpy(chunk + (j * 128 + row) * 16, words, 16);
      }
      uint16_t s = scales_bf16[n * G + g];
      memcpy(chunk + 8192 + row * 2, &s, 2);
    }
  }
}

/* W8 chunk layout: chunk (n_tile, group g of 128 K) = 16640 bytes:
 *   bytes [0, 16384): codes as [j 8][row 128][16 B]; the 16 B of (j,row) hold
 *   K-elements [16j, 16j+16) of the group in order, one byte each, stored as
 *   (code + 128) (codes are in [-127, 127], so 1..255);
 *   bytes [16384, 16640): 128 bf16 scales, one per row.
 * Q3 (codes in [-3, 3]) uses the W4 layout above (4-bit containers). */
void ref_pack_w8(const int8_t* codes, const uint16_t* scales_bf16, int64_t N, int64_t K,
                 uint8_t* out) {
  const int64_t G = K / 128;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    const int64_t nt = n / 128, row = n % 128;
    for (int64_t g = 0; g < G; ++g) {
      uint8_t* chunk = out + (nt * G + g) * 16640;
      for (int j = 0; j < 8; ++j)
        for (int e = 0; e < 16; ++e)
          chunk[(j * 128 + row) * 16 + e] = (uint8_t)(codes[n * K + g * 128 + j * 16 + e] + 128);
      uint16_t s = scales_bf16[n * G + g];
      memcpy(chunk + 16384 + row * 2, &s, 2);
    }
  }
}

/* --------------------------------------------------------------- model */
typedef struct {
  int L, d, H, KVH, hd, ffn, V, max_pos;
  float eps;
  double theta;
} ref_cfg;

typedef struct {
  ref_cfg c;
  uint64_t seed;
  uint16_t *embed, *normf, *lm_head;
  uint16_t **norm1, **norm2;
  uint16_t **wqkv, **wo, **wgu, **wd;       /* effective bf16 weights */
  uint16_t **bqkv, **bo, **bgu, **bd;       /* pristine BF16 copies (for restore) */
  int* tag;                                  /* 0 = BF16, else the quantised bits (8, 4, 3) */
  float *rope_cos, *rope_sin;                /* [max_pos][hd/2] */
} ref_model;

typedef struct {
  int len, cap;
  uint16_t** k; /* [L] -> [cap][KVH][hd] */
  uint16_t** v;
} ref_seq;

static uint16_t* gen_alloc(uint64_t seed, uint64_t tensor, int64_t n, double scale, double off) {
  uint16_t* p = (uint16_t*)malloc((size_t)n * 2);
  ref_gen_weight(seed, tensor, n, scale, off, p);
  return p;
}

/* RoPE table: angle = pos * theta^(-2i/hd) computed in fp64, stored fp32. */
void ref_rope_table(int max_pos, int hd, double theta, float* cos_out, float* sin_out) {
  const int half = hd / 2;
  for (int p = 0; p < max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      double inv = pow(theta, -2.0 * (double)i / (double)hd);
      double a = (double)p * inv;
      cos_out[(int64_t)p * half + i] = (float)cos(a);
      sin_out[(int64_t)p * half + i] = (float)sin(a);
    }
}

ref_model* ref_model_create(const ref_cfg* cfg, uint64_t seed) {
  ref_model* m = (ref_model*)calloc(1, sizeof(ref_model));
  m->c = *cfg;
  m->seed = seed;
  const ref_cfg* c = cfg;
  const int64_t qkv_n = (int64_t)(c->H + 2 * c->KVH) * c->hd;
  m->embed = gen_alloc(seed, T_EMBED, (int64_t)c->V * c->d, 1.0, 0.0);
  m->normf = gen_alloc(seed, T_NORMF, c->d, 0.1, 1.0);
  m->lm_head = gen_alloc(seed, T_LMHEAD, (int64_t)c->V * c->d, 1.0 / sqrt((double)c->d), 0.0);
#define ALLOC_L(f) m->f = (uint16_t**)calloc(c->L, sizeof(uint16_t*))
  ALLOC_L(norm1); ALLOC_L(norm2); ALLOC_L(wqkv); ALLOC_L(wo); ALLOC_L(wgu); ALLOC_L(wd);
  ALLOC_L(bqkv); ALLOC_L(bo); ALLOC_L(bgu); ALLOC_L(bd);
#undef ALLOC_L
  m->tag = (int*)calloc(c->L, sizeof(int));
  for (int l = 0; l < c->L; ++l) {
    m->norm1[l] = gen_alloc(seed, t_layer(l, W_NORM1), c->d, 0.1, 1.0);
    m->norm2[l] = gen_alloc(seed, t_layer(l, W_NORM2), c->d, 0.1, 1.0);
    m->bqkv[l] = gen_alloc(seed, t_layer(l, W_QKV), qkv_n * c->d, 1.0 / sqrt((double)c->d), 0.0);
    m->bo[l] = gen_alloc(seed, t_layer(l, W_O), (int64_t)c->d * c->H * c->hd,
                         1.0 / sqrt((double)(c->H * c->hd)), 0.0);
    m->bgu[l] = gen_alloc(seed, t_layer(l, W_GU), (int64_t)2 * c->ffn * c->d,
                          1.0 / sqrt((double)c->d), 0.0);
    m->bd[l] = gen_alloc(seed, t_layer(l, W_DOWN), (int64_t)c->d * c->ffn,
                         1.0 / sqrt((double)c->ffn), 0.0);
    m->wqkv[l] = m->bqkv[l]; m->wo[l] = m->bo[l]; m->wgu[l] = m->bgu[l]; m->wd[l] = m->bd[l];
  }
  const int half = c->hd / 2;
  m->rope_cos = (float*)malloc((size_t)c->max_pos * half * sizeof(float));
  m->rope_sin = (float*)malloc((size_t)c->max_pos * half * sizeof(float));
  ref_rope_table(c->max_pos, c->hd, c->theta, m->rope_cos, m->rope_sin);
  return m;
}

static uint16_t* dequant_copy(const uint16_t* w, int64_t N, int64_t K, int bits) {
  int8_t* codes = (int8_t*)malloc((size_t)N * K);
  uint16_t* sc = (uint16_t*)malloc((size_t)N * (K / 128) * 2);
  ref_quantize_groups(w, N, K, 128, bits, codes, NULL, sc);
  uint16_t* out = (uint16_t*)malloc((size_t)N * K * 2);
  ref_dequant_w4(codes, sc, N, K, 128, out);
  free(codes);
  free(sc);
  return out;
}

/* Per-layer precision dispatch (toy_model.cpp:153; precision levels
 * toy_model.hpp:26 kFull/kQ8/kQ4/kQ3): bits 16, 8, 4 or 3, every quantised
 * level through the same g128 quantiser and bf16(code * scale) contract. */
void ref_model_set_precision(ref_model* m, int layer, int bits) {
  const ref_cfg* c = &m->c;
  const int64_t qkv_n = (int64_t)(c->H + 2 * c->KVH) * c->hd;
  if (m->tag[layer] != 0) {
    free(m->wqkv[layer]); free(m->wo[layer]); free(m->wgu[layer]); free(m->wd[layer]);
  }
  if (bits == 8 || bits == 4 || bits == 3) {
    m->wqkv[layer] = dequant_copy(m->bqkv[layer], qkv_n, c->d, bits);
    m->wo[layer] = dequant_copy(m->bo[layer], c->d, (int64_t)c->H * c->hd, bits);
    m->wgu[layer] = dequant_copy(m->bgu[layer], (int64_t)2 * c->ffn, c->d, bits);
    m->wd[layer] = dequant_copy(m->bd[layer], c->d, c->ffn, bits);
    m->tag[layer] = bits;
  } else {
    m->wqkv[layer] = m->bqkv[layer]; m->wo[layer] = m->bo[layer];
    m->wgu[layer] = m->bgu[layer]; m->wd[layer] = m->bd[layer];
    m->tag[layer] = 0;
  }
}

/* Accessors so the harness can hand the exact same weights to the GPU. */
uint16_t* ref_model_tensor(ref_model* m, int layer, int which) {
  if (layer < 0) {
    if (which == T_EMBED) return m->embed;
    if (which == T_NORMF) return m->normf;
    return m->lm_head;
  }
  switch (which) {
    case W_NORM1: return m->norm1[layer];
    case W_QKV: return m->bqkv[layer];
    case W_O: return m->bo[layer];
    case W_NORM2: return m->norm2[layer];
    case W_GU: return m->bgu[layer];
    default: return m->bd[layer];
  }
}

void ref_model_destroy(ref_model* m) {
  if (!m) return;
  for (int l = 0; l < m->c.L; ++l) {
    if (m->tag[l] != 0) ref_model_set_precision(m, l, 16);
    free(m->norm1[l]); free(m->norm2[l]);
    free(m->bqkv[l]); free(m->bo[l]); free(m->bgu[l]); free(m->bd[l]);
  }
  free(m->norm1); free(m->norm2); free(m->wqkv); free(m->wo); free(m->wgu); free(m->wd);
  free(m->bqkv); free(m->bo); free(m->bgu); free(m->bd); free(m->tag);
  free(m->embed); free(m->normf); free(m->lm_head); free(m->rope_cos); free(m->rope_sin);
  free(m);
}

ref_seq* ref_seq_create(const ref_model* m, int cap) {
  ref_seq* s = (ref_seq*)calloc(1, sizeof(ref_seq));
  s->cap = cap;
  s->k = (uint16_t**)calloc(m->c.L, sizeof(uint16_t*));
  s->v = (uint16_t**)calloc(m->c.L, sizeof(uint16_t*));
  const size_t per = (size_t)cap * m->c.KVH * m->c.hd;
  for (int l = 0; l < m->c.L; ++l) {
    s->k[l] = (uint16_t*)calloc(per, 2);
    s->v[l] = (uint16_t*)calloc(per, 2);
  }
  return s;
}
void ref_seq_destroy(const ref_model* m, ref_seq* s) {
  if (!s) return;
  for (int l = 0; l < m->c.L; ++l) { free(s->k[l]); free(s->v[l]); }
  free(s->k); free(s->v); free(s);
}
int ref_seq_len(const ref_seq* s) { return s->len; }
/* Direct KV access for kernel-level tests (positions [0,len) of one layer). */
uint16_t* ref_seq_k(ref_seq* s, int layer) { return s->k[layer]; }
uint16_t* ref_seq_v(ref_seq* s, int layer) { return s->v[layer]; }

/* y[b][n] = sum_k W[n][k] * x[b][k]   (bf16 inputs, fp64 accumulation, fp32 out)
 *
 * Every output element is ONE fp64 chain acc = acc + w[k] * x[k] in ascending
 * k, with the product and the sum rounded separately (-ffp-contract=off): the
 * result is bit-identical to the plain triple loop.  The loops are blocked so
 * that the chains of GB columns of b advance together (vectorised across b,
 * never across k), which keeps the oracle fast enough for the full-size
 * parity tests (7B/8B decode steps, the 13B 8192-token prefill). */
#define GB 16 /* b columns per register block */
#define GN 4  /* W rows per register block */
#define BS 256 /* b rows per cache super-block (X^T of BS rows stays in cache) */
#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target_clones("avx512f", "avx2", "default")))
#endif
static void gemm_tile(const uint16_t* W, const double* XT /*[K][GB]*/, int64_t K, int64_t n0, int nn, int nb,
                      int64_t N, int64_t b0, float* Y) {
  double acc[GN][GB];
  for (int i = 0; i < GN; ++i)
    for (int j = 0; j < GB; ++j) acc[i][j] = 0.0;
  if (nn == GN) {
    const uint16_t* w0 = W + (n0 + 0) * K;
    const uint16_t* w1 = W + (n0 + 1) * K;
    const uint16_t* w2 = W + (n0 + 2) * K;
    const uint16_t* w3 = W + (n0 + 3) * K;
    for (int64_t k = 0; k < K; ++k) {
      const double* x = XT + k * GB;
      const double a0 = (double)bf2f(w0[k]), a1 = (double)bf2f(w1[k]);
      const double a2 = (double)bf2f(w2[k]), a3 = (double)bf2f(w3[k]);
      for (int j = 0; j < GB; ++j) {
        acc[0][j] = acc[0][j] + a0 * x[j];
        acc[1][j] = acc[1][j] + a1 * x[j];
        acc[2][j] = acc[2][j] + a2 * x[j];
        acc[3][j] = acc[3][j] + a3 * x[j];
      }
    }
  } else {
    for (int i = 0; i < nn; ++i) {
      const uint16_t* wr = W + (n0 + i) * K;
      for (int64_t k = 0; k < K; ++k) {
        const double a = (double)bf2f(wr[k]);
        const double* x = XT + k * GB;
        for (int j = 0; j < GB; ++j) acc[i][j] = acc[i][j] + a * x[j];
      }
    }
  }
  for (int i = 0; i < nn; ++i)
    for (int j = 0; j < nb; ++j) Y[(b0 + j) * N + n0 + i] = (float)acc[i][j];
}

void ref_gemm_bf16(const uint16_t* W, const uint16_t* X, int64_t B, int64_t N, int64_t K,
                   float* Y) {
  if (B <= 0 || N <= 0) return;
  const int64_t nbb = (B + GB - 1) / GB;
  for (int64_t s0 = 0; s0 < nbb; s0 += BS / GB) {  /* b super-block: X^T blocks reused by every W row */
    const int64_t s1 = s0 + BS / GB < nbb ? s0 + BS / GB : nbb;
    double* XT = (double*)malloc((size_t)(s1 - s0) * K * GB * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t bb = s0; bb < s1; ++bb) {
      double* xt = XT + (bb - s0) * K * GB;
      for (int j = 0; j < GB; ++j) {
        const int64_t b = bb * GB + j;
        for (int64_t k = 0; k < K; ++k) xt[k * GB + j] = b < B ? (double)bf2f(X[b * K + k]) : 0.0;
      }
    }
    const int64_t nnb = (N + GN - 1) / GN;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < nnb * (s1 - s0); ++t) {
      const int64_t nbk = t / (s1 - s0), bb = s0 + t % (s1 - s0);
      const int64_t n0 = nbk * GN, b0 = bb * GB;
      const int nn = (int)(N - n0 < GN ? N - n0 : GN);
      const int nb = (int)(B - b0 < GB ? B - b0 : GB);
      gemm_tile(W, XT + (bb - s0) * K * GB, K, n0, nn, nb, N, b0, Y);
    }
    free(XT);
  }
}

/* xn = bf16((h * inv_rms) * w), inv_rms = 1/sqrt(mean(h^2) + eps) */
void ref_rmsnorm(const float* h, const uint16_t* w, int64_t B, int64_t d, float eps,
                 uint16_t* out) {
  for (int64_t b = 0; b < B; ++b) {
    double ss = 0.0;
    for (int64_t i = 0; i < d; ++i) ss += (double)h[b * d + i] * (double)h[b * d + i];
    const float r = 1.0f / sqrtf((float)(ss / (double)d) + eps);
    for (int64_t i = 0; i < d; ++i) out[b * d + i] = f2bf((h[b * d + i] * r) * bf2f(w[i]));
  }
}

static void rope_inplace(float* x, int hd, const float* cs, const float* sn) {
  const int half = hd / 2;
  for (int i = 0; i < half; ++i) {
    const float x0 = x[i], x1 = x[i + half];
    x[i] = x0 * cs[i] - x1 * sn[i];
    x[i + half] = x1 * cs[i] + x0 * sn[i];
  }
}

/* One attention query (all heads) against seq positions [0, ctx). */
void ref_attention(const float* q /*[H][hd]*/, const uint16_t* kc, const uint16_t* vc,
                   int ctx, int H, int KVH, int hd, uint16_t* out /*[H][hd] bf16*/,
                   float* out_f32) {
  const int G = H / KVH;
  const float scale = 1.0f / sqrtf((float)hd);
  float* s = (float*)malloc((size_t)ctx * sizeof(float));
  for (int h = 0; h < H; ++h) {
    const int kh = h / G;
    float mx = -INFINITY;
    for (int t = 0; t < ctx; ++t) {
      double acc = 0.0;
      const uint16_t* kr = kc + ((int64_t)t * KVH + kh) * hd;
      /* q enters q.k rounded to bf16 (every device attention path), fp32 scale after */
      for (int i = 0; i < hd; ++i) acc += (double)bf2f(f2bf(q[h * hd + i])) * (double)bf2f(kr[i]);
      s[t] = (float)acc * scale;
      if (s[t] > mx) mx = s[t];
    }
    double l = 0.0;
    for (int t = 0; t < ctx; ++t) {
      s[t] = expf(s[t] - mx);
      l += s[t];
    }
    for (int i = 0; i < hd; ++i) {
      double acc = 0.0;
      for (int t = 0; t < ctx; ++t)
        acc += (double)s[t] * (double)bf2f(vc[((int64_t)t * KVH + kh) * hd + i]);
      const float o = (float)(acc / l);
      if (out) out[h * hd + i] = f2bf(o);
      if (out_f32) out_f32[h * hd + i] = o;
    }
  }
  free(s);
}

static inline float silu(float x) { return x / (1.0f + expf(-x)); }

/* One decode token for each of B sequences: tokens[b] enters at position
 * seqs[b]->len; its K/V are appended; logits[b][V] (may be NULL) and
 * next[b] = argmax are returned.  This is also the prefill math: a prefill of
 * n tokens is n such positions (causal attention makes them identical). */
static void forward_impl(ref_model* m, ref_seq** seqs, const int32_t* tokens, int B, float* logits,
                         int32_t* next, float* trace, int64_t trace_layer_stride);

void ref_forward(ref_model* m, ref_seq** seqs, const int32_t* tokens, int B, float* logits,
                 int32_t* next) {
  forward_impl(m, seqs, tokens, B, logits, next, NULL, 0);
}

/* trace (optional): the residual stream [B][d] entering layer l is written at
 * trace + l * trace_layer_stride, the one leaving the last layer at L * stride
 * (the activation trace of the layer profiler, profiler.cpp:41-103). */
static void forward_impl(ref_model* m, ref_seq** seqs, const int32_t* tokens, int B, float* logits,
                         int32_t* next, float* trace, int64_t trace_layer_stride) {
  const ref_cfg* c = &m->c;
  const int d = c->d, hd = c->hd, H = c->H, KVH = c->KVH, half = hd / 2;
  const int qkv_n = (H + 2 * KVH) * hd;
  float* h = (float*)malloc((size_t)B * d * sizeof(float));
  uint16_t* xn = (uint16_t*)malloc((size_t)B * (c->ffn > d ? c->ffn : d) * 2);
  float* y = (float*)malloc((size_t)B * 2 * (c->ffn > qkv_n ? c->ffn : qkv_n) * sizeof(float) +
                            (size_t)B * c->V * sizeof(float));
  uint16_t* att = (uint16_t*)malloc((size_t)B * H * hd * 2);
  float* q = (float*)malloc((size_t)H * hd * sizeof(float));
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < d; ++i) h[(int64_t)b * d + i] = bf2f(m->embed[(int64_t)tokens[b] * d + i]);

  for (int l = 0; l < c->L; ++l) {
    if (trace) memcpy(trace + (int64_t)l * trace_layer_stride, h, (size_t)B * d * sizeof(float));
    ref_rmsnorm(h, m->norm1[l], B, d, c->eps, xn);
    ref_gemm_bf16(m->wqkv[l], xn, B, qkv_n, d, y);
    for (int b = 0; b < B; ++b) {
      ref_seq* s = seqs[b];
      const int pos = s->len;
      float* row = y + (int64_t)b * qkv_n;
      const float* cs = m->rope_cos + (int64_t)pos * half;
      const float* sn = m->rope_sin + (int64_t)pos * half;
      for (int hh = 0; hh < H; ++hh) rope_inplace(row + hh * hd, hd, cs, sn);
      for (int hh = 0; hh < KVH; ++hh) rope_inplace(row + (H + hh) * hd, hd, cs, sn);
      for (int hh = 0; hh < KVH; ++hh)
        for (int i = 0; i < hd; ++i) {
          s->k[l][((int64_t)pos * KVH + hh) * hd + i] = f2bf(row[(H + hh) * hd + i]);
          s->v[l][((int64_t)pos * KVH + hh) * hd + i] = f2bf(row[(H + KVH + hh) * hd + i]);
        }
      memcpy(q, row, (size_t)H * hd * sizeof(float));
      ref_attention(q, s->k[l], s->v[l], pos + 1, H, KVH, hd, att + (int64_t)b * H * hd, NULL);
    }
    ref_gemm_bf16(m->wo[l], att, B, d, (int64_t)H * hd, y);
    for (int64_t i = 0; i < (int64_t)B * d; ++i) h[i] = h[i] + y[i];
    ref_rmsnorm(h, m->norm2[l], B, d, c->eps, xn);
    ref_gemm_bf16(m->wgu[l], xn, B, 2 * c->ffn, d, y);
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < c->ffn; ++j) {
        const float g = y[(int64_t)b * 2 * c->ffn + j];
        const float u = y[(int64_t)b * 2 * c->ffn + c->ffn + j];
        xn[(int64_t)b * c->ffn + j] = f2bf(silu(g) * u);
      }
    ref_gemm_bf16(m->wd[l], xn, B, d, c->ffn, y);
    for (int64_t i = 0; i < (int64_t)B * d; ++i) h[i] = h[i] + y[i];
  }
  if (trace) memcpy(trace + (int64_t)c->L * trace_layer_stride, h, (size_t)B * d * sizeof(float));
  for (int b = 0; b < B; ++b) seqs[b]->len += 1;
  ref_rmsnorm(h, m->normf, B, d, c->eps, xn);
  float* lg = logits ? logits : y;
  ref_gemm_bf16(m->lm_head, xn, B, c->V, d, lg);
  for (int b = 0; b < B; ++b) {
    const float* r = lg + (int64_t)b * c->V;
    int best = 0;
    for (int v = 1; v < c->V; ++v)
      if (r[v] > r[best]) best = v;
    if (next) next[b] = best;
  }
  free(h); free(xn); free(y); free(att); free(q);
}

/* Prefill helper: runs n positions of one sequence; returns argmax after the
 * last one (and its logits if requested). */
int32_t ref_prefill(ref_model* m, ref_seq* s, const int32_t* tokens, int n, float* logits) {
  int32_t nxt = -1;
  for (int i = 0; i < n; ++i) ref_forward(m, &s, tokens + i, 1, (i == n - 1) ? logits : NULL, &nxt);
  return nxt;
}

/* Prefill with the per-layer residual stream: trace [L+1][n][d] (the GPU
 * counterpart is ms_prefill_trace). */
int32_t ref_prefill_trace(ref_model* m, ref_seq* s, const int32_t* tokens, int n, float* logits, float* trace) {
  int32_t nxt = -1;
  for (int i = 0; i < n; ++i)
    forward_impl(m, &s, tokens + i, 1, (i == n - 1) ? logits : NULL, &nxt, trace + (int64_t)i * m->c.d,
                 (int64_t)n * m->c.d);
  return nxt;
}

/* Batched prefill: the same math as ref_prefill (token by token through
 * forward_impl), evaluated layer by layer over all n tokens at once.  Every
 * per-token operation and its order is unchanged (row-wise GEMM chains in
 * ascending k, causal attention of token i over positions [0, len + i]), so
 * the result is bit-identical to ref_prefill / ref_prefill_trace; only the
 * loops are reordered so that the GEMMs see n rows (fast enough for the
 * 8192-token Llama-2-13B parity test).
 *   rows / n_rows (optional): in the LAST layer only these token rows are
 *   carried past the QKV projection (every row's K/V is still appended); the
 *   trace and the logits are then defined for those rows only (the last token
 *   must be among them when logits are requested).
 *   trace (optional): [L+1][n][d] residual stream, as ref_prefill_trace. */
int32_t ref_prefill_rows(ref_model* m, ref_seq* s, const int32_t* tokens, int n, const int32_t* rows, int n_rows,
                         float* logits, float* trace) {
  const ref_cfg* c = &m->c;
  const int d = c->d, hd = c->hd, H = c->H, KVH = c->KVH, half = hd / 2, ffn = c->ffn;
  const int qkv_n = (H + 2 * KVH) * hd;
  const int pos0 = s->len;
  int* sel = (int*)malloc((size_t)n * sizeof(int));
  int nsel = 0;
  if (rows) {
    for (int i = 0; i < n_rows; ++i) sel[nsel++] = rows[i];
  } else {
    for (int i = 0; i < n; ++i) sel[nsel++] = i;
  }
  float* h = (float*)malloc((size_t)n * d * sizeof(float));
  uint16_t* xn = (uint16_t*)malloc((size_t)n * (ffn > d ? ffn : d) * 2);
  float* y = (float*)malloc((size_t)n * (2 * ffn > qkv_n ? 2 * ffn : qkv_n) * sizeof(float));
  uint16_t* att = (uint16_t*)malloc((size_t)n * H * hd * 2);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) h[(int64_t)i * d + j] = bf2f(m->embed[(int64_t)tokens[i] * d + j]);
  for (int l = 0; l < c->L; ++l) {
    const int last = l == c->L - 1;
    if (trace) memcpy(trace + (int64_t)l * n * d, h, (size_t)n * d * sizeof(float));
    ref_rmsnorm(h, m->norm1[l], n, d, c->eps, xn);
    ref_gemm_bf16(m->wqkv[l], xn, n, qkv_n, d, y);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      const int pos = pos0 + i;
      float* row = y + (int64_t)i * qkv_n;
      const float* cs = m->rope_cos + (int64_t)pos * half;
      const float* sn = m->rope_sin + (int64_t)pos * half;
      for (int hh = 0; hh < H; ++hh) rope_inplace(row + hh * hd, hd, cs, sn);
      for (int hh = 0; hh < KVH; ++hh) rope_inplace(row + (H + hh) * hd, hd, cs, sn);
      for (int hh = 0; hh < KVH; ++hh)
        for (int j = 0; j < hd; ++j) {
          s->k[l][((int64_t)pos * KVH + hh) * hd + j] = f2bf(row[(H + hh) * hd + j]);
          s->v[l][((int64_t)pos * KVH + hh) * hd + j] = f2bf(row[(H + KVH + hh) * hd + j]);
        }
    }
    const int nr = last ? nsel : n;
    /* rows carried on: all of them, or the selected ones in the last layer
     * (compacted to the front of h / att / xn / y) */
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < nr; ++r) {
      const int i = last ? sel[r] : r;
      ref_attention(y + (int64_t)i * qkv_n, s->k[l], s->v[l], pos0 + i + 1, H, KVH, hd,
                    att + (int64_t)r * H * hd, NULL);
    }
    if (last && rows) {
      for (int r = 0; r < nr; ++r)
        memmove(h + (int64_t)r * d, h + (int64_t)sel[r] * d, (size_t)d * sizeof(float));
    }
    ref_gemm_bf16(m->wo[l], att, nr, d, (int64_t)H * hd, y);
    for (int64_t i = 0; i < (int64_t)nr * d; ++i) h[i] = h[i] + y[i];
    ref_rmsnorm(h, m->norm2[l], nr, d, c->eps, xn);
    ref_gemm_bf16(m->wgu[l], xn, nr, 2 * ffn, d, y);
    for (int r = 0; r < nr; ++r)
      for (int j = 0; j < ffn; ++j) {
        const float g = y[(int64_t)r * 2 * ffn + j];
        const float u = y[(int64_t)r * 2 * ffn + ffn + j];
        xn[(int64_t)r * ffn + j] = f2bf(silu(g) * u);
      }
    ref_gemm_bf16(m->wd[l], xn, nr, d, ffn, y);
    for (int64_t i = 0; i < (int64_t)nr * d; ++i) h[i] = h[i] + y[i];
    if (trace && last) {
      float* t = trace + (int64_t)c->L * n * d;
      for (int r = 0; r < nr; ++r)
        memcpy(t + (int64_t)(rows ? sel[r] : r) * d, h + (int64_t)r * d, (size_t)d * sizeof(float));
    }
  }
  s->len += n;
  /* the last token's logits (row n - 1 must have been carried) */
  int lr = -1;
  for (int r = 0; r < nsel; ++r)
    if (sel[r] == n - 1) lr = r;
  int32_t best = -1;
  if (lr >= 0) {
    ref_rmsnorm(h + (int64_t)lr * d, m->normf, 1, d, c->eps, xn);
    float* lg = logits ? logits : (float*)malloc((size_t)c->V * sizeof(float));
    ref_gemm_bf16(m->lm_head, xn, 1, c->V, d, lg);
    best = 0;
    for (int v = 1; v < c->V; ++v)
      if (lg[v] > lg[best]) best = v;
    if (!logits) free(lg);
  }
  free(sel); free(h); free(xn); free(y); free(att);
  return best;
}

void ref_seq_set_len(ref_seq* s, int len) { s->len = len; }

/* Restatement of the device's synthetic KV fill (runtime ms_kv_fill_synthetic
 * -> elementwise.cu fill_kv_kernel): element `off` of the pi-th listed page is
 * bf16(u), u = (r >> 40) * 2^-24 * 2 - 1, r = splitmix64(seed + pi * per_page
 * + off), page layout [layer][kv_head][K|V][16 tok][head_dim].  Fills this
 * sequence's cache for positions [0, 16 * nblocks), block j being the
 * page_index[j]-th page of the fill list. */
void ref_seq_fill_pages(const ref_model* m, ref_seq* s, const int64_t* page_index, int nblocks, uint64_t seed) {
  const ref_cfg* c = &m->c;
  const int64_t hd = c->hd, KVH = c->KVH;
  const int64_t per_page = 16 * (int64_t)c->L * KVH * 2 * hd;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < nblocks; ++j) {
    for (int l = 0; l < c->L; ++l)
      for (int64_t kh = 0; kh < KVH; ++kh)
        for (int kv = 0; kv < 2; ++kv)
          for (int t = 0; t < 16; ++t)
            for (int64_t i = 0; i < hd; ++i) {
              const int64_t off = (((int64_t)l * KVH + kh) * 2 + kv) * 16 * hd + t * hd + i;
              const uint64_t r = splitmix64(seed + (uint64_t)(page_index[j] * per_page + off));
              const float u = (float)(r >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
              uint16_t* dst = kv ? s->v[l] : s->k[l];
              dst[(((int64_t)j * 16 + t) * KVH + kh) * hd + i] = f2bf(u);
            }
  }
}

int ref_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------ CPU baseline sample */
/* Times one decoder-layer decode step for B sequences at context `ctx`
 * (weights from the shared generator, KV filled with random bf16) plus the
 * final norm + lm_head + argmax for B rows.  Used by bench.py's cpu_baseline
 * and --impl reference legs as a BOUNDED sample of the 7B decode step (the
 * full step is L layer-steps + one lm_head).  Returns layer seconds. */
#include <time.h>
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
double ref_bench_decode_sample(const ref_cfg* c, int B, int ctx, int w4, uint64_t seed, double* lm_seconds) {
  const int d = c->d, hd = c->hd, H = c->H, KVH = c->KVH, half = hd / 2, ffn = c->ffn;
  const int64_t qkv_n = (int64_t)(H + 2 * KVH) * hd;
  uint16_t* n1 = gen_alloc(seed, t_layer(0, W_NORM1), d, 0.1, 1.0);
  uint16_t* n2 = gen_alloc(seed, t_layer(0, W_NORM2), d, 0.1, 1.0);
  uint16_t* wqkv = gen_alloc(seed, t_layer(0, W_QKV), qkv_n * d, 1.0 / sqrt((double)d), 0.0);
  uint16_t* wo = gen_alloc(seed, t_layer(0, W_O), (int64_t)d * H * hd, 1.0 / sqrt((double)(H * hd)), 0.0);
  uint16_t* wgu = gen_alloc(seed, t_layer(0, W_GU), (int64_t)2 * ffn * d, 1.0 / sqrt((double)d), 0.0);
  uint16_t* wd = gen_alloc(seed, t_layer(0, W_DOWN), (int64_t)d * ffn, 1.0 / sqrt((double)ffn), 0.0);
  if (w4) {
    uint16_t* t;
    t = dequant_copy(wqkv, qkv_n, d, 4); free(wqkv); wqkv = t;
    t = dequant_copy(wo, d, (int64_t)H * hd, 4); free(wo); wo = t;
    t = dequant_copy(wgu, (int64_t)2 * ffn, d, 4); free(wgu); wgu = t;
    t = dequant_copy(wd, d, ffn, 4); free(wd); wd = t;
  }
  const size_t per_seq = (size_t)ctx * KVH * hd;
  uint16_t* kc = gen_alloc(seed ^ 0x55, 1000, (int64_t)(per_seq * B), 1.0, 0.0);
  uint16_t* vc = gen_alloc(seed ^ 0xAA, 1001, (int64_t)(per_seq * B), 1.0, 0.0);
  float* h = (float*)malloc((size_t)B * d * sizeof(float));
  uint16_t* embed_row = gen_alloc(seed, T_EMBED, (int64_t)B * d, 1.0, 0.0);
  for (int64_t i = 0; i < (int64_t)B * d; ++i) h[i] = bf2f(embed_row[i]);
  uint16_t* xn = (uint16_t*)malloc((size_t)B * (ffn > d ? ffn : d) * 2);
  float* y = (float*)malloc((size_t)B * (2 * ffn > qkv_n ? 2 * ffn : qkv_n) * sizeof(float));
  uint16_t* att = (uint16_t*)malloc((size_t)B * H * hd * 2);
  float* cs = (float*)malloc((size_t)half * sizeof(float));
  float* sn = (float*)malloc((size_t)half * sizeof(float));
  for (int i = 0; i < half; ++i) {
    double a = (double)(ctx - 1) * pow(c->theta, -2.0 * (double)i / (double)hd);
    cs[i] = (float)cos(a);
    sn[i] = (float)sin(a);
  }
  const double t0 = now_s();
  ref_rmsnorm(h, n1, B, d, c->eps, xn);
  ref_gemm_bf16(wqkv, xn, B, qkv_n, d, y);
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < B; ++b) {
    float* row = y + (int64_t)b * qkv_n;
    for (int hh = 0; hh < H + KVH; ++hh) rope_inplace(row + hh * hd, hd, cs, sn);
    uint16_t* kb = kc + (size_t)b * per_seq;
    uint16_t* vb = vc + (size_t)b * per_seq;
    for (int hh = 0; hh < KVH; ++hh)
      for (int i = 0; i < hd; ++i) {
        kb[((size_t)(ctx - 1) * KVH + hh) * hd + i] = f2bf(row[(H + hh) * hd + i]);
        vb[((size_t)(ctx - 1) * KVH + hh) * hd + i] = f2bf(row[(H + KVH + hh) * hd + i]);
      }
    ref_attention(row, kb, vb, ctx, H, KVH, hd, att + (int64_t)b * H * hd, NULL);
  }
  ref_gemm_bf16(wo, att, B, d, (int64_t)H * hd, y);
  for (int64_t i = 0; i < (int64_t)B * d; ++i) h[i] += y[i];
  ref_rmsnorm(h, n2, B, d, c->eps, xn);
  ref_gemm_bf16(wgu, xn, B, 2 * ffn, d, y);
  for (int b = 0; b < B; ++b)
    for (int j = 0; j < ffn; ++j)
      xn[(int64_t)b * ffn + j] = f2bf(silu(y[(int64_t)b * 2 * ffn + j]) * y[(int64_t)b * 2 * ffn + ffn + j]);
  ref_gemm_bf16(wd, xn, B, d, ffn, y);
  for (int64_t i = 0; i < (int64_t)B * d; ++i) h[i] += y[i];
  const double t1 = now_s();
  if (lm_seconds) {
    uint16_t* lm = gen_alloc(seed, T_LMHEAD, (int64_t)c->V * d, 1.0 / sqrt((double)d), 0.0);
    uint16_t* nf = gen_alloc(seed, T_NORMF, d, 0.1, 1.0);
    float* lg = (float*)malloc((size_t)B * c->V * sizeof(float));
    const double t2 = now_s();
    ref_rmsnorm(h, nf, B, d, c->eps, xn);
    ref_gemm_bf16(lm, xn, B, c->V, d, lg);
    volatile int sink = 0;
    for (int b = 0; b < B; ++b) {
      int best = 0;
      for (int v = 1; v < c->V; ++v)
        if (lg[(int64_t)b * c->V + v] > lg[(int64_t)b * c->V + best]) best = v;
      sink += best;
    }
    *lm_seconds = now_s() - t2;
    free(lm); free(nf); free(lg);
  }
  free(n1); free(n2); free(wqkv); free(wo); free(wgu); free(wd); free(kc); free(vc); free(h);
  free(embed_row); free(xn); free(y); free(att); free(cs); free(sn);
  return t1 - t0;
}
