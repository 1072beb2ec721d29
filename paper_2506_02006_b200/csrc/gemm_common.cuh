// gemm_common.cuh -- pieces of the tcgen05 GEMM kernels (gemm.cu): packed-chunk
// sizes, the weight chunk cursor over a variant image's page table, the
// stream-K / whole-tile segment walker, and the int4 -> bf16 magic.
#pragma once
#include <cstdint>

#include "kernels.h"
#include "ptx.cuh"

namespace ms {


__device__ __forceinline__ const uint8_t* chunk_ptr(const GemmWeights& w, int64_t ci, int chunk_bytes) {
  const int64_t c = w.first_chunk + ci;
  const int64_t page = c / w.chunks_per_page;
  const int64_t off = (c - page * w.chunks_per_page) * chunk_bytes;
  return reinterpret_cast<const uint8_t*>(w.pages[page]) + off;
}

// Walks consecutive chunks of one weight image: one division per segment,
// one page-table load per page crossing (the producer thread must stay far
// ahead of the MMAs, so no per-chunk 64-bit division or dependent load).
struct ChunkCursor {
  const GemmWeights* w;
  int64_t cpp, page, in_page;
  const uint8_t* base;
  int chunk_bytes;
  __device__ ChunkCursor(const GemmWeights& w_, int cb)
      : w(&w_), cpp(w_.chunks_per_page), page(-1), in_page(0), base(nullptr), chunk_bytes(cb) {}
  __device__ const uint8_t* page_base(int64_t p) const {
    const int64_t i = p - w->inl_p0;
    return reinterpret_cast<const uint8_t*>(i >= 0 && i < w->n_inl ? w->inl[i] : w->pages[p]);
  }
  __device__ void seek(int64_t c) {
    const int64_t p = (c >> 31) == 0 && (cpp >> 31) == 0 ? (int64_t)((uint32_t)c / (uint32_t)cpp) : c / cpp;
    in_page = c - p * cpp;
    if (p != page) {
      page = p;
      base = page_base(p);
    }
  }
  __device__ const uint8_t* get() {
    if (in_page >= cpp) {  // crossed one or more page ends (advance() does not normalise)
      do {
        in_page -= cpp;
        ++page;
      } while (in_page >= cpp);
      base = page_base(page);
    }
    return base + in_page * chunk_bytes;
  }
  __device__ void advance() { ++in_page; }
};

// Segment walker shared by every role so they all see the same sequence.
// Stream-K plans: CTA c takes the contiguous k-step range [T c / C, T (c+1) / C).
// Whole-tile plans (long prefills): CTA c takes logical tiles c, c + C, ...,
// so the C tiles in flight at any time are C consecutive logical tiles, and
// logical tiles are rastered in groups of kRasterM token tiles (all weight
// tiles of a group before the next): the tiles in flight then share ~8 token
// tiles and ~C/8 weight tiles, whose k-slices stay in L2 (group size = the
// plan's `aligned` field, MS_GEMM_RASTER, default 8) (contiguous ranges
// per CTA had every CTA streaming its own A and B from DRAM: 6-8 GB per
// prefill GEMM instead of ~0.5 GB).
struct SegIter {
  int64_t g, g1;
  int nk;
  int u, tiles, C, n_tiles, m_tiles, rm;
  bool al;
  __device__ SegIter(const GemmPlanDev& p, int c) : nk(p.nk), al(p.aligned != 0) {
    if (al) {
      rm = p.aligned;  // raster group: token tiles per group
      u = c;
      tiles = p.tiles;
      C = p.C;
      n_tiles = p.n_tiles;
      m_tiles = p.tiles / p.n_tiles;
      g = g1 = 0;
    } else {
      // stream-K plans satisfy (T + 1) * C < 2^31 (gemm_plan): 32-bit division
      g = (int64_t)((uint32_t)p.T * (uint32_t)c / (uint32_t)p.C);
      g1 = (int64_t)((uint32_t)p.T * (uint32_t)(c + 1) / (uint32_t)p.C);
    }
  }
  __device__ int raster(int v) const {
    const int grp = v / (rm * n_tiles);
    const int r = v - grp * rm * n_tiles;
    const int gm = min(rm, m_tiles - grp * rm);
    const int nt = r / gm;
    return (grp * rm + (r - nt * gm)) * n_tiles + nt;
  }
  // next segment: tile t, k-steps [k0, k1)
  __device__ bool next(int& t, int& k0, int& k1) {
    if (al) {
      if (u >= tiles) return false;
      t = raster(u);
      k0 = 0;
      k1 = nk;
      u += C;
      return true;
    }
    if (g >= g1) return false;
    t = (int)((uint32_t)g / (uint32_t)nk);
    k0 = (int)(g - (int64_t)t * nk);
    const int64_t end = min(g1, (int64_t)(t + 1) * nk);
    k1 = (int)(end - (int64_t)t * nk);
    g = end;
    return true;
  }
};

// bf16x2 (128 + nib_lo, 128 + nib_hi) from the nibbles at bits 0..3 / 16..19.
__device__ __forceinline__ uint32_t nib_magic(uint32_t w) {
  uint32_t x;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(w), "r"(0x000F000Fu), "r"(0x43004300u));
  return x;
}

}  // namespace ms
