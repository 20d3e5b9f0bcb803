// rac_batch.cu -- bit-sliced batched enforcement on sm_100a.
//
// Many domain states (search-tree nodes, Alg. 2) on one
// instance.  The states are transposed to state-major bit slices: for a word
// w of 32 states, X_w[(x,a)] is a u32 whose bit j says (x,a) ∈ D_{32w+j}.
// One pass of Eq. 1 for all 32 states at once is then
//   X_w'[(x,a)] = X_w[(x,a)] & AND_{y ∈ C_x} ( OR_{b ∈ c_xy|(x,a)} X_w[(y,b)] )
// i.e. the support test "c_xy|(x,a) ∩ D_s(y) ≠ ∅" evaluated for 32 states in
// one 32-bit OR; the OR over b uses per-pass nibble tables
//   T[y][q][v] = OR_{j : bit j of v} X_w[(y, 4q+j)]
// so one mask costs ceil(d/4) shared-memory lookups.  Per-state loop control
// (Alg. 1) runs on 32-bit masks: wipeout first, then "changed";
// a state that stops is frozen (its bits are no longer updated) and its own
// pass count is its iteration count.  Passes >= 2 (and pass 1 of seeded
// states) test only variables changed in the previous pass (union over the
// word's active states; Prop. 2, lines 130-143 -- testing extra columns is
// harmless for a state whose column did not change).
//
// Work split: CTA = (word w, block of 256 rows).  The RB CTAs of a word
// exchange their new rows through a global double buffer and synchronise
// with a per-word software barrier (co-resident cooperative grid).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

constexpr int kBT = 256;  // threads per CTA = rows per CTA
constexpr uint32_t kFullFlag = 1u;

__device__ __forceinline__ void word_sync(unsigned* bar, unsigned nblocks, unsigned epoch) {
  __syncthreads();
  if (nblocks > 1 && threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&bar[0], 1u);
    if (prev + 1u == nblocks * epoch) {
      st_release_gpu(&bar[1], epoch);
    } else {
      while (ld_relaxed_gpu(&bar[1]) < epoch) __nanosleep(128);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int W>
__device__ __forceinline__ uint32_t load_mask(const uint8_t* p) {
  // only the low d bits matter (d <= 32 here is not assumed: W == 8 keeps 64)
  if constexpr (W == 8) return 0u;  // unused: W == 8 goes through load_mask64
  else if constexpr (W == 4) return __ldg(reinterpret_cast<const uint32_t*>(p));
  else if constexpr (W == 2) return __ldg(reinterpret_cast<const uint16_t*>(p));
  else return __ldg(p);
}

__device__ __forceinline__ uint64_t load_mask64(const uint8_t* p) {
  return __ldg(reinterpret_cast<const unsigned long long*>(p));
}

}  // namespace

template <int W>
__global__ void __launch_bounds__(kBT, 3) rac_batch_bs(BatchBSParams p) {
  extern __shared__ uint32_t sm[];
  constexpr int NQ = 2 * W;  // nibbles per mask (d <= 8W)
  const int rows = p.n * p.dmax;
  const int rows4 = (rows + 3) & ~3;  // per-word stride of the exchange buffers (16-B aligned)
  const int w = blockIdx.x / p.RB;
  const int rb = blockIdx.x - w * p.RB;
  uint32_t* X = sm;                                                   // [rows]
  uint32_t* T = X + ((rows + 3) & ~3);                                // [n][NQ][16] (if p.use_table), 16-B aligned
  int* list = reinterpret_cast<int*>(T + (p.use_table ? (size_t)p.n * NQ * 16 : 0));  // [n]
  uint8_t* need = reinterpret_cast<uint8_t*>(list + p.n);             // [n]
  uint8_t* inlist = need + ((p.n + 15) & ~15);                         // [n] columns of this pass
  __shared__ int s_iters[32], s_status[32];
  __shared__ uint32_t s_or, s_and;
  __shared__ int s_cnt;
  unsigned* bar = p.bar + 4 * w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int sbase = p.s0 + 32 * w;  // first state of this word (caller's index)
  const int nst = min(32, p.S - 32 * w);
  const bool full = (p.flags & kFullFlag) != 0;

  // ---- transpose the word's states into bit slices (every CTA, redundantly)
  for (int x = warp; x < p.n; x += nwarps) {
    uint64_t v = lane < nst ? __ldg(p.d_in + (size_t)(sbase + lane) * p.n + x) & __ldg(p.dommask + x) : 0ull;
    for (int a = 0; a < p.dmax; ++a) {
      const uint32_t b = __ballot_sync(0xffffffffu, (v >> a) & 1ull);
      if (lane == 0) X[x * p.dmax + a] = b;
    }
  }
  for (int i = threadIdx.x; i < p.n; i += blockDim.x) need[i] = 0;
  if (threadIdx.x < 32) {
    s_iters[threadIdx.x] = 0;
    s_status[threadIdx.x] = 0;
  }
  __syncthreads();
  uint32_t active = nst >= 32 ? 0xffffffffu : ((1u << nst) - 1u);
  // ---- initial column list: union of the seeds (any unseeded state -> all)
  bool all_cols = p.seed_var == nullptr;
  if (!all_cols) {
    int any_all = 0;
    if (threadIdx.x < nst) {
      const int sv = p.seed_var[sbase + threadIdx.x];
      if (sv < 0 || sv >= p.n) any_all = 1;
      else need[sv] = 1;
    }
    all_cols = __syncthreads_or(any_all) != 0;
  }
  if (all_cols) {
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) need[i] = 1;
    __syncthreads();
  }

  const int row = rb * kBT + threadIdx.x;
  const int x = row < rows ? row / p.dmax : 0;
  const int a = row - x * p.dmax;
  const uint8_t* Mrow = p.M + (size_t)row * W;  // + y * col_stride: column-major masks
  const uint32_t* Prow = p.P + (size_t)x * p.pw;
  int t = 0;
  unsigned epoch = 0;
  unsigned long long* dbg = (p.dbg && threadIdx.x == 0) ? p.dbg + (size_t)blockIdx.x * 64 : nullptr;
  if (dbg) dbg[0] = globaltimer();
  for (;;) {
    ++t;
    // column list for this pass from need[] (ascending), need[] cleared
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
      inlist[i] = need[i];
      if (need[i]) {
        list[atomicAdd(&s_cnt, 1)] = i;
        need[i] = 0;
      }
    }
    __syncthreads();
    const int ncol = s_cnt;
    // nibble tables for the listed columns: one thread per (column, nibble q)
    // loads the 4 slices X[(y, 4q..4q+3)] and writes the 16 OR-combinations
    if (p.use_table) {
      for (int i = threadIdx.x; i < ncol * NQ; i += blockDim.x) {
        const int k = i / NQ, q = i - k * NQ;
        const int y = list[k];
        uint32_t xb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) xb[j] = (4 * q + j < p.dmax) ? X[y * p.dmax + 4 * q + j] : 0u;
        uint32_t tv[16];
        tv[0] = 0u;
#pragma unroll
        for (int v = 1; v < 16; ++v) tv[v] = tv[v & (v - 1)] | xb[__ffs(v) - 1];
        uint4* dst = reinterpret_cast<uint4*>(T + (y * NQ + q) * 16);
#pragma unroll
        for (int v = 0; v < 16; v += 4) dst[v >> 2] = make_uint4(tv[v], tv[v + 1], tv[v + 2], tv[v + 3]);
      }
      __syncthreads();
    }
    // ---- the support test of my row for the 32 states of the word
    uint32_t nb = 0;
    if (row < rows) {
      const uint32_t cur = X[row];
      const uint32_t live = cur & active;
      nb = cur;
      if (live) {
        uint32_t acc = 0xffffffffu;
        const int nvecr = p.row_bytes / 16;
        if (p.Mr != nullptr && ncol >= nvecr && W < 8) {
          // dense column list: stream the row-major copy of my row, 16 bytes =
          // 16/W masks per load, kRV loads in flight; listed columns only.
          constexpr int L = 16 / W, kRV = 8;
          const bool all_cols = ncol == p.n;
          const uint4* rowv = reinterpret_cast<const uint4*>(p.Mr + (size_t)row * p.row_bytes);
          for (int v0 = 0; v0 < nvecr && (acc & live) != 0; v0 += kRV) {
            uint4 mv[kRV];
#pragma unroll
            for (int u = 0; u < kRV; ++u)
              if (v0 + u < nvecr) mv[u] = __ldg(rowv + v0 + u);
#pragma unroll
            for (int u = 0; u < kRV; ++u) {
              if (v0 + u >= nvecr) continue;
              const uint32_t w4[4] = {mv[u].x, mv[u].y, mv[u].z, mv[u].w};
#pragma unroll
              for (int i = 0; i < L; ++i) {
                const int y = (v0 + u) * L + i;
                if (y >= p.n) break;
                if (!all_cols && !inlist[y]) continue;
                const uint32_t m = (w4[(i * W) >> 2] >> ((8 * W * i) & 31));
                uint32_t sup = 0;
                if (p.use_table) {
                  const uint32_t* Ty = T + y * (NQ * 16);
#pragma unroll
                  for (int q = 0; q < NQ; ++q) sup |= Ty[q * 16 + ((m >> (4 * q)) & 15u)];
                } else {
                  uint32_t mm = m & (p.dmax >= 32 ? ~0u : ((1u << p.dmax) - 1u));
                  while (mm) {
                    const int b = __ffs(mm) - 1;
                    sup |= X[y * p.dmax + b];
                    mm &= mm - 1;
                  }
                }
                if ((sup & live) != live) {
                  if (!((__ldg(Prow + (y >> 5)) >> (y & 31)) & 1u)) sup = 0xffffffffu;
                }
                acc &= sup;
              }
            }
          }
        } else
        // kBU mask loads in flight per thread, then the table lookups
        for (int k0 = 0, kBU = 8; k0 < ncol && (acc & live) != 0; k0 += kBU) {
          uint64_t mv[8];
          int yv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            yv[u] = k0 + u < ncol ? list[k0 + u] : -1;
            if (yv[u] >= 0) {
              if constexpr (W == 8) mv[u] = load_mask64(Mrow + (size_t)yv[u] * p.col_stride);
              else mv[u] = load_mask<W>(Mrow + (size_t)yv[u] * p.col_stride);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int y = yv[u];
            if (y < 0) continue;
            const uint64_t m = mv[u];
            uint32_t sup = 0;
            if (p.use_table) {
#pragma unroll
              for (int q = 0; q < NQ; ++q) sup |= T[(y * NQ + q) * 16 + (uint32_t)((m >> (4 * q)) & 15u)];
            } else {
              uint64_t mm = m & (p.dmax >= 64 ? ~0ull : ((1ull << p.dmax) - 1ull));
              while (mm) {
                const int b = __ffsll((long long)mm) - 1;
                sup |= X[y * p.dmax + b];
                mm &= mm - 1;
              }
            }
            if ((sup & live) != live) {
              // some live state lost support on column y: only a declared c_xy
              // removes (absent pairs and y == x store all-ones; reading R2)
              if (!((__ldg(Prow + (y >> 5)) >> (y & 31)) & 1u)) sup = 0xffffffffu;
            }
            acc &= sup;
          }
        }
        nb = cur & (acc | ~active);
      }
      p.X2[((size_t)(t & 1) * p.NW + w) * rows4 + row] = nb;
    }
    word_sync(bar, p.RB, ++epoch);
    // ---- gather the word's new rows; per-state flags (every CTA redundantly)
    if (threadIdx.x == 0) {
      s_or = 0u;
      s_and = 0xffffffffu;
    }
    __syncthreads();
    uint32_t diff = 0;
    const uint32_t* Xg = p.X2 + ((size_t)(t & 1) * p.NW + w) * rows4;
    {
      // 16-byte loads, all issued before use; the last partial group of 4
      // rows is read past `rows` (the stride is rows4) and ignored
      const uint4* Xg4 = reinterpret_cast<const uint4*>(Xg);
      const int r4 = rows4 >> 2;
      constexpr int U = 4;
      for (int i0 = threadIdx.x; i0 < r4; i0 += U * blockDim.x) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * blockDim.x;
          if (i < r4) v[u] = __ldcg(Xg4 + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * blockDim.x;
          if (i >= r4) continue;
          const uint32_t nw4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = 4 * i + k;
            if (r >= rows) break;
            const uint32_t o = X[r], nw = nw4[k];
            diff |= o ^ nw;
            if (o ^ nw) need[r / p.dmax] = 1;
            X[r] = nw;
          }
        }
      }
    }
    diff = __reduce_or_sync(0xffffffffu, diff);
    if (lane == 0 && diff) atomicOr(&s_or, diff);
    __syncthreads();
    uint32_t allne = 0xffffffffu;  // states in which every variable is nonempty
    for (int v = threadIdx.x; v < p.n; v += blockDim.x) {
      uint32_t ne = 0;
      for (int b = 0; b < p.dmax; ++b) ne |= X[v * p.dmax + b];
      allne &= ne;
    }
    allne = __reduce_and_sync(0xffffffffu, allne);
    if (lane == 0 && allne != 0xffffffffu) atomicAnd(&s_and, allne);
    __syncthreads();
    const uint32_t changed = s_or, wipe = ~s_and;
    const uint32_t stop_wipe = full ? 0u : (wipe & active);
    const uint32_t stop_conv = ~changed & active & ~stop_wipe;
    if (threadIdx.x < 32) {
      const uint32_t bit = 1u << threadIdx.x;
      if (active & bit) s_iters[threadIdx.x] = t;
      if (stop_wipe & bit) s_status[threadIdx.x] = 1;
      if (stop_conv & bit) s_status[threadIdx.x] = (wipe & bit) ? 1 : 0;
    }
    active &= ~(stop_wipe | stop_conv);
    if (dbg && t < 63) dbg[t] = globaltimer();
    __syncthreads();
    if (active == 0) break;
  }
  // ---- outputs: CTA 0 of the word transposes the slices back
  if (rb == 0) {
    for (int xx = warp; xx < p.n; xx += nwarps) {
      uint64_t v = 0;
      for (int b = 0; b < p.dmax; ++b) v |= (uint64_t)((X[xx * p.dmax + b] >> lane) & 1u) << b;
      if (lane < nst) p.d_out[(size_t)(sbase + lane) * p.n + xx] = v;
    }
    if (threadIdx.x < nst) {
      p.iters[sbase + threadIdx.x] = s_iters[threadIdx.x];
      p.status[sbase + threadIdx.x] = s_status[threadIdx.x];
    }
  }
  // the last CTA of the word out resets its barrier words
  if (threadIdx.x == 0 && p.RB > 1) {
    __threadfence();
    if (atomicAdd(&bar[2], 1u) + 1u == (unsigned)p.RB) {
      bar[0] = 0u;
      bar[1] = 0u;
      bar[2] = 0u;
      __threadfence();
    }
  }
}

size_t batch_bs_smem(int n, int dmax, int W, bool use_table) {
  const size_t rows = (size_t)n * dmax;
  return ((rows + 3) & ~(size_t)3) * 4 + (use_table ? (size_t)n * (2 * W) * 16 * 4 : 0) + (size_t)n * 4 +
         2 * (((size_t)n + 15) & ~(size_t)15);
}

cudaError_t batch_bs_occupancy(int W, size_t smem, int* out) {
  const void* k = nullptr;
  switch (W) {
    case 1: k = (const void*)rac_batch_bs<1>; break;
    case 2: k = (const void*)rac_batch_bs<2>; break;
    case 4: k = (const void*)rac_batch_bs<4>; break;
    case 8: k = (const void*)rac_batch_bs<8>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kBT, smem);
}

cudaError_t launch_batch_bs(int W, const BatchBSParams& p, int grid, size_t smem, cudaStream_t s) {
  const void* k = nullptr;
  switch (W) {
    case 1: k = (const void*)rac_batch_bs<1>; break;
    case 2: k = (const void*)rac_batch_bs<2>; break;
    case 4: k = (const void*)rac_batch_bs<4>; break;
    case 8: k = (const void*)rac_batch_bs<8>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  BatchBSParams pp = p;
  void* args[] = {&pp};
  return cudaLaunchCooperativeKernel(k, dim3(grid), dim3(kBT), args, smem, s);
}

}  // namespace rac
