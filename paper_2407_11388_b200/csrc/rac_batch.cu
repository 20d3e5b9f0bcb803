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
      while (ld_acquire_gpu(&bar[1]) < epoch) __nanosleep(32);
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
__global__ void __launch_bounds__(kBT) rac_batch_bs(BatchBSParams p) {
  extern __shared__ uint32_t sm[];
  constexpr int NQ = 2 * W;  // nibbles per mask (d <= 8W)
  const int rows = p.n * p.dmax;
  const int w = blockIdx.x / p.RB;
  const int rb = blockIdx.x - w * p.RB;
  uint32_t* X = sm;                                                   // [rows]
  uint32_t* T = X + rows;                                             // [n][NQ][16] (if p.use_table)
  int* list = reinterpret_cast<int*>(T + (p.use_table ? (size_t)p.n * NQ * 16 : 0));  // [n]
  uint8_t* need = reinterpret_cast<uint8_t*>(list + p.n);             // [n]
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
  for (;;) {
    ++t;
    // column list for this pass from need[] (ascending), need[] cleared
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) {
      if (need[i]) {
        list[atomicAdd(&s_cnt, 1)] = i;
        need[i] = 0;
      }
    }
    __syncthreads();
    const int ncol = s_cnt;
    // nibble tables for the listed columns
    if (p.use_table) {
      for (int i = threadIdx.x; i < ncol * NQ * 16; i += blockDim.x) {
        const int k = i / (NQ * 16), r = i - k * (NQ * 16), q = r >> 4, v = r & 15;
        const int y = list[k];
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int b = 4 * q + j;
          if (((v >> j) & 1) && b < p.dmax) o |= X[y * p.dmax + b];
        }
        T[((size_t)y * NQ + q) * 16 + v] = o;
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
        // kBU mask loads in flight per thread, then the table lookups
        constexpr int kBU = 8;
        for (int k0 = 0; k0 < ncol && (acc & live) != 0; k0 += kBU) {
          uint64_t mv[kBU];
          int yv[kBU];
#pragma unroll
          for (int u = 0; u < kBU; ++u) {
            yv[u] = k0 + u < ncol ? list[k0 + u] : -1;
            if (yv[u] >= 0) {
              if constexpr (W == 8) mv[u] = load_mask64(Mrow + (size_t)yv[u] * p.col_stride);
              else mv[u] = load_mask<W>(Mrow + (size_t)yv[u] * p.col_stride);
            }
          }
#pragma unroll
          for (int u = 0; u < kBU; ++u) {
            const int y = yv[u];
            if (y < 0) continue;
            const uint64_t m = mv[u];
            uint32_t sup = 0;
            if (p.use_table) {
#pragma unroll
              for (int q = 0; q < NQ; ++q) sup |= T[((size_t)y * NQ + q) * 16 + ((m >> (4 * q)) & 15u)];
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
      p.X2[((size_t)(t & 1) * p.NW + w) * rows + row] = nb;
    }
    word_sync(bar, p.RB, ++epoch);
    // ---- gather the word's new rows; per-state flags (every CTA redundantly)
    if (threadIdx.x == 0) {
      s_or = 0u;
      s_and = 0xffffffffu;
    }
    __syncthreads();
    uint32_t diff = 0;
    const uint32_t* Xg = p.X2 + ((size_t)(t & 1) * p.NW + w) * rows;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const uint32_t o = X[i], nw = __ldcg(Xg + i);
      diff |= o ^ nw;
      if (o ^ nw) need[i / p.dmax] = 1;
      X[i] = nw;
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
  return rows * 4 + (use_table ? (size_t)n * (2 * W) * 16 * 4 : 0) + (size_t)n * 4 + (((size_t)n + 15) & ~(size_t)15);
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
