// rac_pack.cu -- relation-tensor packer (N1) and device instance generator (N7).
//
// "Prepare Cons" (Fig. 1): the paper stores
// Cons ∈ {0,1}^{n×n×d×d} in fp32.  Here each support set c_xy|(x,a)
// (line 45) becomes one W-byte mask in column y at row (x,a) of the column-major
// tensor (rac_internal.cuh); both orientations are stored,
// the (y,x) one being the bit-transpose built with warp ballots.  Absent pairs
// and y == x keep the all-ones fill (cudaMemset 0xFF) and presence bit 0.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../synth/csp_synth.h"
#include "rac_internal.cuh"

namespace rac {

namespace {

__device__ __forceinline__ void put_w(uint8_t* p, int W, uint64_t m) {
  switch (W) {
    case 8: *reinterpret_cast<uint64_t*>(p) = m; break;
    case 4: *reinterpret_cast<uint32_t*>(p) = (uint32_t)m; break;
    case 2: *reinterpret_cast<uint16_t*>(p) = (uint16_t)m; break;
    default: *p = (uint8_t)m; break;
  }
}

// Mask c_xy|(x,a): column-major copy (column y, local row (x - x_lo)*dmax + a)
// and, when present, the row-major copy (that row, byte offset y*W).
__device__ __forceinline__ void store_mask(const PackGeom& g, int x, int a, int y, uint64_t m) {
  const size_t r = (size_t)(x - g.x_lo) * g.dmax + a;
  put_w(g.M + (size_t)y * g.col_stride + r * g.W, g.W, m);
  if (g.Mr) put_w(g.Mr + r * g.row_bytes + (size_t)y * g.W, g.W, m);
}

__device__ __forceinline__ void set_present(const PackGeom& g, int x, int y) {
  atomicOr(&g.P[(size_t)(x - g.x_lo) * g.pw + (y >> 5)], 1u << (y & 31));
}

// A warp holds rows a = lane and a = lane + 32 of rel(c_xy) (x < y or x > y),
// dx = dom[x], dy = dom[y].  Writes the forward masks M[x][a][y] and the
// transposed masks M[y][b][x] = { a : (a,b) ∈ rel(c_xy) } for whichever of x,
// y lies in the local block.
__device__ __forceinline__ void pack_pair_warp(const PackGeom& g, int x, int y, int dx, int dy, uint64_t row_lo,
                                               uint64_t row_hi) {
  const int lane = threadIdx.x & 31;
  const bool x_local = x >= g.x_lo && x < g.x_hi;
  const bool y_local = y >= g.x_lo && y < g.x_hi;
  if (x_local) {
    if (lane < dx) store_mask(g, x, lane, y, row_lo);
    if (lane + 32 < dx) store_mask(g, x, lane + 32, y, row_hi);
    if (lane == 0) set_present(g, x, y);
  }
  if (y_local) {
    uint64_t col_lo = 0, col_hi = 0;  // column b = lane and b = lane + 32
    for (int b = 0; b < dy; ++b) {
      const uint32_t lo = __ballot_sync(0xffffffffu, (row_lo >> b) & 1ull);  // rows a = 0..31
      const uint32_t hi = __ballot_sync(0xffffffffu, (row_hi >> b) & 1ull);  // rows a = 32..63
      const uint64_t col = (uint64_t)lo | ((uint64_t)hi << 32);
      if (b == lane) col_lo = col;
      if (b == lane + 32) col_hi = col;
    }
    if (lane < dy) store_mask(g, y, lane, x, col_lo);
    if (lane + 32 < dy) store_mask(g, y, lane + 32, x, col_hi);
    if (lane == 0) set_present(g, y, x);
  }
}

__global__ void pack_relations_kernel(PackGeom g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                                      int n_rel, int row_words) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = warp; r < n_rel; r += nwarps) {
    const int x = xs[r], y = ys[r];
    const bool touches = (x >= g.x_lo && x < g.x_hi) || (y >= g.x_lo && y < g.x_hi);
    if (!touches) continue;
    const int dx = g.dom[x], dy = g.dom[y];
    const uint64_t* rr = rows + (size_t)r * row_words;
    const uint64_t row_lo = lane < dx ? rr[lane] : 0ull;
    const uint64_t row_hi = lane + 32 < dx ? rr[lane + 32] : 0ull;
    pack_pair_warp(g, x, y, dx, dy, row_lo, row_hi);
  }
}

// Device generator: warp per unordered pair (x < y), same bits as
// synth/csp_synth.h (the host oracle regenerates them independently).
__global__ void generate_kernel(PackGeom g, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  const long n = g.n;
  // pairs touching the local block: x in block (any y > x) or y in block (x < y)
  const long total = n * n;
  const uint32_t q = (uint32_t)(d + 3) / 4u;
  for (long idx = warp; idx < total; idx += nwarps) {
    const int x = (int)(idx / n), y = (int)(idx - (long)x * n);
    if (y <= x) continue;
    const bool touches = (x >= g.x_lo && x < g.x_hi) || (y >= g.x_lo && y < g.x_hi);
    if (!touches) continue;
    if (!synth_present(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y, dens_q32)) continue;
    const uint64_t pk = synth_pair_key(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y);
    uint64_t rows2[2] = {0ull, 0ull};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int a = lane + 32 * h;
      if (a >= d) continue;
      uint64_t row = 0;
      for (uint32_t bq = 0; bq < q; ++bq) {
        const uint64_t w = synth_cell_word_pk(pk, (uint32_t)d, (uint32_t)a, bq);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t b = bq * 4u + j;
          if (b < (uint32_t)d && ((uint32_t)(w >> (16 * j)) & 0xFFFFu) >= t_q16) row |= 1ull << b;
        }
      }
      rows2[h] = row;
    }
    pack_pair_warp(g, x, y, d, d, rows2[0], rows2[1]);
  }
}

// Sparse arc-block packer (NEXT-3): warp per pair, rows a = lane, lane + 32 of
// rel(c_xy) from the host array or the generator; forward masks to block
// fwd[r] (row a at byte a*W), the ballot-transposed masks c_yx|(y,b) to block
// bwd[r].  Blocks were filled with 0xFF (rows a >= dom(x) are never live).
__global__ void pack_sparse_kernel(SparsePack g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                                   int row_words, const uint32_t* fwd, const uint32_t* bwd, long n_pairs, int d,
                                   uint32_t t_q16, uint64_t seed) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = warp; r < n_pairs; r += nwarps) {
    const int x = xs[r], y = ys[r];
    const int dx = g.dom[x], dy = g.dom[y];
    uint64_t row_lo = 0, row_hi = 0;
    if (rows) {
      const uint64_t* rr = rows + (size_t)r * row_words;
      row_lo = lane < dx ? rr[lane] : 0ull;
      row_hi = lane + 32 < dx ? rr[lane + 32] : 0ull;
    } else {
      const uint64_t pk = synth_pair_key(seed, (uint32_t)g.n, (uint32_t)x, (uint32_t)y);
      const uint32_t q = (uint32_t)(d + 3) / 4u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = lane + 32 * h;
        if (a >= d) continue;
        uint64_t row = 0;
        for (uint32_t bq = 0; bq < q; ++bq) {
          const uint64_t w = synth_cell_word_pk(pk, (uint32_t)d, (uint32_t)a, bq);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t b = bq * 4u + j;
            if (b < (uint32_t)d && ((uint32_t)(w >> (16 * j)) & 0xFFFFu) >= t_q16) row |= 1ull << b;
          }
        }
        if (h == 0) row_lo = row; else row_hi = row;
      }
    }
    if (fwd[r] != 0xffffffffu) {
      uint8_t* blk = g.S + (size_t)fwd[r] * g.bbytes;
      if (lane < dx) put_w(blk + lane * g.W, g.W, row_lo);
      if (lane + 32 < dx) put_w(blk + (lane + 32) * g.W, g.W, row_hi);
    }
    if (bwd[r] != 0xffffffffu) {
      uint64_t col_lo = 0, col_hi = 0;  // column b = lane and b = lane + 32
      for (int b = 0; b < dy; ++b) {
        const uint32_t lo = __ballot_sync(0xffffffffu, (row_lo >> b) & 1ull);
        const uint32_t hi = __ballot_sync(0xffffffffu, (row_hi >> b) & 1ull);
        const uint64_t col = (uint64_t)lo | ((uint64_t)hi << 32);
        if (b == lane) col_lo = col;
        if (b == lane + 32) col_hi = col;
      }
      uint8_t* blk = g.S + (size_t)bwd[r] * g.bbytes;
      if (lane < dy) put_w(blk + lane * g.W, g.W, col_lo);
      if (lane + 32 < dy) put_w(blk + (lane + 32) * g.W, g.W, col_hi);
    }
  }
}

int grid_for(long work_warps) {
  long blocks = (work_warps * 32 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return (int)blocks;
}

}  // namespace

cudaError_t launch_pack_relations(const PackGeom& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                                  int n_rel, int row_words, cudaStream_t s) {
  if (n_rel == 0) return cudaSuccess;
  pack_relations_kernel<<<grid_for(n_rel), 256, 0, s>>>(g, xs, ys, rows, n_rel, row_words);
  return cudaGetLastError();
}

cudaError_t launch_generate(const PackGeom& g, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                            cudaStream_t s) {
  generate_kernel<<<grid_for((long)g.n * g.n), 256, 0, s>>>(g, d, dens_q32, t_q16, seed);
  return cudaGetLastError();
}

cudaError_t launch_pack_sparse(const SparsePack& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                               int row_words, const uint32_t* fwd, const uint32_t* bwd, long n_pairs, int d,
                               uint32_t t_q16, uint64_t seed, cudaStream_t s) {
  if (n_pairs == 0) return cudaSuccess;
  pack_sparse_kernel<<<grid_for(n_pairs), 256, 0, s>>>(g, xs, ys, rows, row_words, fwd, bwd, n_pairs, d, t_q16, seed);
  return cudaGetLastError();
}

}  // namespace rac
