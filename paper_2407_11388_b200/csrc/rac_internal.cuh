// rac_internal.cuh -- internal declarations and device helpers of librac (sm_100a).
//
// Data layout in HBM:
//   W          bytes per support mask: 1, 2, 4 or 8 (smallest >= max dom bits).
//   nvec       ceil(n*W / 16): 16-byte vectors per (x,a) row.
//   row_stride nvec*16 bytes.
//   M          [local rows][row_stride] bytes; local row r = (x - x_lo)*dmax + a.
//              Bytes [y*W, y*W+W) of row (x,a) hold the support mask
//              c_xy|(x,a) as a d_y-bit set; absent pairs
//              and y == x hold all-ones; bytes beyond n*W hold 0xFF.
//   P          presence bitmap, [local x][pw = ceil(n/32)] u32; bit y of
//              variable x set iff c_xy is declared (C_x).
//   D (smem)   the alive bitvector D_t in the same W-byte layout as a row
//              (variable x at bytes [x*W, x*W+W)), padded with 0xFF to
//              row_stride bytes, so 16-byte vector v of a row lines up with
//              16-byte vector v of D.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace rac {

constexpr int kThreads = 512;  // CTA size of the support-pass kernels
constexpr int kUnroll = 4;     // 16-byte loads in flight per lane per batch

// ---------------------------------------------------------------------------- params
struct PassGeom {
  const uint8_t* M;       // first local row
  size_t row_stride;      // bytes
  int nvec;               // 16-byte vectors per row
  int n;                  // variables
  int dmax;               // rows per variable
  int x_lo, x_hi;         // rows of variables [x_lo, x_hi) are processed (M indexed from x_lo_alloc)
  int x_lo_alloc;         // first variable whose rows M points at
  const uint32_t* P;      // presence bits of variable x_lo_alloc onward
  int pw;                 // u32 words per presence row
  int seg_vecs;           // vectors per work item (a row is split into n_seg segments)
  int n_seg;
};

struct FusedParams {
  PassGeom g;
  const uint64_t* dommask;  // [n]
  const uint64_t* d_in;     // [n] device
  uint64_t* d_out;          // [n] device
  int32_t* iters;           // device scalar
  int32_t* status;          // device scalar
  int32_t* removed_at;      // nullable [n*64], pre-zeroed
  unsigned long long* R;    // [3][n] removal masks (rotating)
  unsigned* bar;            // grid barrier words [4]
  const int32_t* seeds;     // nullable device [n_seeds]: Alg. 1 initial @changed
  int n_seeds;
  uint32_t flags;
};

struct ShardState {
  uint64_t* Dcur;            // [n] current D_t (u64 per variable)
  uint64_t* Dg;              // [world*blk] gathered D_{t+1}
  uint8_t* Dw;               // [row_stride] D_t in the W-byte smem layout (TMA source)
  unsigned long long* R;     // [n] removal masks of the current pass
  int32_t* iters;            // device scalars
  int32_t* status;
  int32_t* done;
  int32_t* vcnt;             // length of vlist (vectors changed in the last pass)
  uint16_t* vlist;           // [nvec] Prop. 2 incremental vector list
};

struct PassParams {
  PassGeom g;
  ShardState s;
  int32_t* removed_at;
};

struct BatchParams {
  PassGeom g;
  const uint64_t* dommask;
  const uint64_t* d_in;   // [S][n]
  uint64_t* d_out;        // [S][n]
  int32_t* iters;         // [S]
  int32_t* status;        // [S]
  const int32_t* seed_var;  // nullable [S]: per-state seed variable (-1 = all)
  uint32_t flags;
};

struct BatchBSParams {
  const uint8_t* M;
  size_t row_stride;
  int n, dmax;
  const uint32_t* P;
  int pw;
  const uint64_t* dommask;
  const uint64_t* d_in;     // [.][n] caller's states
  uint64_t* d_out;
  int32_t* iters;
  int32_t* status;
  const int32_t* seed_var;  // nullable [.]
  int S;                    // states in this launch
  int s0;                   // index of the first state in the caller's arrays
  int NW;                   // words (32 states) in this launch
  int RB;                   // CTAs per word
  bool use_table;
  uint32_t* X2;             // [2][NW][n*dmax] exchange buffers
  unsigned* bar;            // [NW][4] per-word barrier words (zero between launches)
  uint32_t flags;
};

// Dynamic smem of rac_fused / rac_batch: D (nvec x 16 B), then the incremental
// vector list (u16[nvec]) and the per-vector "needed" flags (u8[nvec]).
__host__ __device__ constexpr size_t list_offset(int nvec) { return (size_t)nvec * 16; }
__host__ __device__ constexpr size_t need_offset(int nvec) {
  return (size_t)nvec * 16 + (((size_t)nvec * 2 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t fused_smem(int nvec) {
  return need_offset(nvec) + (((size_t)nvec + 15) & ~(size_t)15);
}

// ---------------------------------------------------------------------------- host launchers
// (defined in rac_kernels.cu / rac_pack.cu; return cudaError_t of the launch)
int choose_group(int nvec);  // lanes per row
cudaError_t launch_fused(int W, int G, const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool cooperative);
cudaError_t fused_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
cudaError_t launch_pass(int W, int G, const PassParams& p, int grid, size_t smem, cudaStream_t s);
cudaError_t pass_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
cudaError_t launch_shard_init(const ShardState& s, const uint64_t* d_in, const uint64_t* dommask, int n, int W,
                              size_t row_stride, int total_g, cudaStream_t st);
cudaError_t launch_shard_slice(const ShardState& s, int x_lo, int x_hi, int n, cudaStream_t st);
cudaError_t launch_shard_update(const ShardState& s, int n, int W, int nvec, uint32_t flags, cudaStream_t st);
cudaError_t launch_shard_finalize(const ShardState& s, int n, uint64_t* d_out, int32_t* iters, int32_t* status,
                                  cudaStream_t st);
cudaError_t launch_batch(int W, int G, const BatchParams& p, int n_states, size_t smem, cudaStream_t s);
cudaError_t batch_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
size_t batch_bs_smem(int n, int dmax, int W, bool use_table);
cudaError_t batch_bs_occupancy(int W, size_t smem, int* blocks_per_sm);
cudaError_t launch_batch_bs(int W, const BatchBSParams& p, int grid, size_t smem, cudaStream_t s);

struct PackGeom {
  uint8_t* M;             // local rows
  size_t row_stride;
  int W;
  int n, dmax;
  int x_lo, x_hi;         // local block
  uint32_t* P;
  int pw;
  const int32_t* dom;     // device [n]
};
cudaError_t launch_pack_relations(const PackGeom& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                                  int n_rel, int row_words, cudaStream_t s);
cudaError_t launch_generate(const PackGeom& g, int d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                            cudaStream_t s);

// ---------------------------------------------------------------------------- device helpers
#ifdef __CUDACC__

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Does any W-byte lane of t equal zero?  (t = mask & D, 16 bytes = 16/W masks)
template <int W>
__device__ __forceinline__ bool vec_any_zero(uint4 t) {
  if constexpr (W == 8) {
    return ((t.x | t.y) == 0u) | ((t.z | t.w) == 0u);
  } else if constexpr (W == 4) {
    return (t.x == 0u) | (t.y == 0u) | (t.z == 0u) | (t.w == 0u);
  } else if constexpr (W == 2) {
    return (__vcmpeq2(t.x, 0u) | __vcmpeq2(t.y, 0u) | __vcmpeq2(t.z, 0u) | __vcmpeq2(t.w, 0u)) != 0u;
  } else {
    return (__vcmpeq4(t.x, 0u) | __vcmpeq4(t.y, 0u) | __vcmpeq4(t.z, 0u) | __vcmpeq4(t.w, 0u)) != 0u;
  }
}

__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
  return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}

template <int W>
__device__ __forceinline__ uint64_t load_w(const uint8_t* p) {
  if constexpr (W == 8) return *reinterpret_cast<const uint64_t*>(p);
  else if constexpr (W == 4) return *reinterpret_cast<const uint32_t*>(p);
  else if constexpr (W == 2) return *reinterpret_cast<const uint16_t*>(p);
  else return *p;
}

template <int W>
__device__ __forceinline__ void store_w(uint8_t* p, uint64_t v) {
  if constexpr (W == 8) *reinterpret_cast<uint64_t*>(p) = v;
  else if constexpr (W == 4) *reinterpret_cast<uint32_t*>(p) = (uint32_t)v;
  else if constexpr (W == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
  else *p = (uint8_t)v;
}

__device__ __forceinline__ uint64_t extract_w(const uint4& v, int i, int W) {
  // i-th W-byte lane of a 16-byte vector
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if (W == 8) return (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  if (W == 4) return w[i];
  if (W == 2) return (w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
  return (w[i >> 2] >> (8 * (i & 3))) & 0xFFu;
}

// A 16-byte vector had some mask & D == 0.  Decide whether that is a real
// loss of support: mask_y & D(y) == 0 removes (x,a) iff c_xy is declared
// (reading R2) -- absent pairs store all-ones, so they only "fail" when D(y)
// is empty, and then P decides.  Padding lanes (y >= n) never fail.
template <int W>
__device__ __noinline__ bool vec_real_fail(uint4 m, uint4 d, int v, int n, const uint32_t* Prow) {
  constexpr int L = 16 / W;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    int y = v * L + i;
    if (y >= n) break;
    uint64_t mi = extract_w(m, i, W), di = extract_w(d, i, W);
    if ((mi & di) == 0) {
      if (di != 0) return true;
      if ((Prow[y >> 5] >> (y & 31)) & 1u) return true;
    }
  }
  return false;
}

template <int G>
__device__ __forceinline__ bool group_any(bool f, unsigned gmask) {
  if constexpr (G == 32) return __any_sync(0xffffffffu, f);
  else if constexpr (G == 1) return f;
  else return (__ballot_sync(gmask, f) & gmask) != 0u;
}

// Support test of one (x,a) row segment [vb, ve) against D in smem:
// returns true iff some declared c_xy has c_xy|(x,a) ∩ D(y) = ∅ for y in the
// segment (Eq. 1 condition, intersection form of line 59).
// G lanes cooperate; kUnroll 16-byte streaming loads per lane are in flight
// before the AND/test; the group exits early once a failure is seen.
template <int W, int G>
__device__ __forceinline__ bool row_fails(const uint4* __restrict__ row, const uint4* Ds, int vb, int ve, int gl,
                                          unsigned gmask, int n, const uint32_t* Prow) {
  bool fail = false;
  for (int v0 = vb; v0 < ve; v0 += G * kUnroll) {
    uint4 m[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int v = v0 + u * G + gl;
      if (v < ve) m[u] = ldg_stream(row + v);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int v = v0 + u * G + gl;
      if (v < ve) {
        uint4 d = Ds[v];
        if (vec_any_zero<W>(and4(m[u], d))) fail |= vec_real_fail<W>(m[u], d, v, n, Prow);
      }
    }
    if (group_any<G>(fail, gmask)) return true;
  }
  return false;
}

// As row_fails, but only over the 16-byte vectors listed in vl[lb, le)
// (Prop. 2: after pass 1 a row can only lose support
// on a constraint whose other variable changed in the previous pass, so only
// the vectors holding masks of changed variables are re-tested).
template <int W, int G>
__device__ __forceinline__ bool row_fails_list(const uint4* __restrict__ row, const uint4* Ds, const uint16_t* vl,
                                               int lb, int le, int gl, unsigned gmask, int n,
                                               const uint32_t* Prow) {
  bool fail = false;
  for (int i0 = lb; i0 < le; i0 += G * kUnroll) {
    uint4 m[kUnroll];
    int vv[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int i = i0 + u * G + gl;
      vv[u] = i < le ? (int)vl[i] : -1;
      if (vv[u] >= 0) m[u] = ldg_stream(row + vv[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (vv[u] >= 0) {
        uint4 d = Ds[vv[u]];
        if (vec_any_zero<W>(and4(m[u], d))) fail |= vec_real_fail<W>(m[u], d, vv[u], n, Prow);
      }
    }
    if (group_any<G>(fail, gmask)) return true;
  }
  return false;
}

// Block-wide compaction of the flags need[0, cnt) into the ascending index
// list out[]; clears need[].  Returns the list length (same in every thread).
__device__ __forceinline__ int block_compact(uint8_t* need, uint16_t* out, int cnt, int* scratch) {
  const int T = blockDim.x, t = threadIdx.x;
  const int chunk = (cnt + T - 1) / T;
  const int b = min(cnt, t * chunk), e = min(cnt, b + chunk);
  int c = 0;
  for (int i = b; i < e; ++i) c += need[i] != 0;
  // inclusive scan over threads: warp shuffles, then warp totals in scratch
  const int lane = t & 31, w = t >> 5;
  int v = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    int s = lane < (T >> 5) ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    if (lane < (T >> 5)) scratch[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  int pos = v - c + (w > 0 ? scratch[w - 1] : 0);
  for (int i = b; i < e; ++i) {
    if (need[i]) out[pos++] = (uint16_t)i;
    need[i] = 0;
  }
  const int total = scratch[(T >> 5) - 1];
  __syncthreads();
  return total;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Software grid barrier for a co-resident (cooperative) grid.  bar[0] counts
// arrivals over the whole launch, bar[1] is the released epoch.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned epoch) {
  __syncthreads();
  if (nblocks > 1 && threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&bar[0], 1u);
    if (prev + 1u == nblocks * epoch) {
      st_release_gpu(&bar[1], epoch);
    } else {
      while (ld_acquire_gpu(&bar[1]) < epoch) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

#endif  // __CUDACC__

}  // namespace rac
