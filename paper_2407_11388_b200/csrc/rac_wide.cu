// rac_wide.cu -- wide domains (65..256 values per variable).
//
// The same recurrence as rac_kernels.cu -- Eq. 1 with Alg. 1's loop
// control, Prop. 2's incremental passes -- on domains
// wider than one 64-bit word.  The paper fixes no domain-size limit (its Cons
// is a dense [n, d, n, d] fp32 tensor); only the mask width
// changes here.
//
// Layout (HBM).  Row-major masks: the WS-word mask c_xy|(x,a) of row
// (x,a) and column y at M[((x*dmax + a)*n + y)*WS], WS = 2 (d <= 128) or 4
// (d <= 256) words, i.e. one or two 16-byte vectors; d in 129..192 uses WS = 4
// with a zero pad word.  Absent pairs and the diagonal hold all-ones masks and
// presence bit 0 (P[x][y], n x n bits), exactly as the one-word layout.
//
// Kernel.  One persistent cooperative launch per enforcement (a5 on the
// device).  Per pass: every CTA stages D_{t-1} (n*WS words) in shared memory;
// warps take live rows (x,a) (static warp-stride), the 32 lanes stream the
// row's masks over the tested columns -- all y in pass 1, the variables changed
// by the previous pass afterwards (Alg. 1's Cons[:, @changed], Prop. 2) -- four
// 16-byte loads in flight per lane, AND with D(y) from smem; a zero result on
// a declared pair is a failure (warp vote, early exit) and sets the row's
// removal bit R[x][a] (a4).  A pass with at most kThreadRowCols tested
// columns (a seeded pass 1, a late pass) gives each thread a row instead, so
// rows are not serialised behind 31 idle lanes.  Grid barrier; one thread per variable applies
// D_t = D_{t-1} & ~R, appends changed variables to the next column list,
// records removal epochs, raises the wipeout flag (a5); grid barrier; every
// thread reads the same flags and takes the same stop decision.
#include <cooperative_groups.h>

#include "../../include/rac.h"
#include "rac_internal.cuh"
#include "../../synth/csp_synth.h"

namespace cg = cooperative_groups;

namespace rac {
namespace {

constexpr int kWideThreads = 512;
constexpr unsigned kThreadRowCols = 8;  // tested columns at or below which a thread takes a row

struct WideSlot {
  unsigned cnt;   // variables changed by the pass (length of the slot's column list)
  unsigned wipe;  // some domain empty after the pass
};

template <int WS>
struct Mask {
  ulonglong2 v[WS / 2];
};

template <int WS>
__device__ __forceinline__ Mask<WS> load_mask(const uint64_t* p) {
  Mask<WS> m;
#pragma unroll
  for (int i = 0; i < WS / 2; ++i) {
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p) + i;
    asm("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
                 : "=l"(m.v[i].x), "=l"(m.v[i].y)
                 : "l"(q));
  }
  return m;
}

template <int WS>
__device__ __forceinline__ bool meets(const Mask<WS>& m, const uint64_t* dy) {
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < WS / 2; ++i) acc |= (m.v[i].x & dy[2 * i]) | (m.v[i].y & dy[2 * i + 1]);
  return acc != 0;
}

__device__ __forceinline__ bool present(const uint32_t* P, int pw, int x, int y) {
  return (__ldg(P + (size_t)x * pw + (y >> 5)) >> (y & 31)) & 1u;
}

template <int WS>
__global__ void __launch_bounds__(kWideThreads) wide_fused(WideParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint64_t sD[];  // [n * WS]
  const int n = p.n, dmax = p.dmax, wq = p.wq;
  const int tid = threadIdx.x;
  const size_t gtid = (size_t)blockIdx.x * blockDim.x + tid;
  const size_t gthreads = (size_t)gridDim.x * blockDim.x;
  const int lane = tid & 31;
  const size_t gwarp = gtid >> 5;
  const size_t nwarps = gthreads >> 5;
  WideSlot* slots = reinterpret_cast<WideSlot*>(p.slots);

  // D_0 = d_in (bits beyond dom(x) dropped), boundary n x wq -> internal n x WS
  for (size_t i = gtid; i < (size_t)n * WS; i += gthreads) {
    const int x = (int)(i / WS), w = (int)(i % WS);
    uint64_t v = 0;
    if (w < wq) {
      const int bits = min(64, max(0, p.dom[x] - 64 * w));
      const uint64_t dm = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
      v = p.d_in[(size_t)x * wq + w] & dm;
    }
    p.D[i] = v;
    p.R[i] = 0;
  }
  if (p.removed_at)
    for (size_t i = gtid; i < (size_t)n * 64 * wq; i += gthreads) p.removed_at[i] = 0;
  if (gtid < 3) slots[gtid] = WideSlot{0u, 0u};
  grid.sync();

  int pass = 0;
  int status = RAC_OK;
  const uint32_t* cols = nullptr;  // nullptr: every column (pass 1)
  unsigned ncols = (unsigned)n;
  if (p.n_seeds >= 0) {  // seeded call: pass 1 tests Cons[:, seeds] (Alg. 1 @changed = seeds)
    cols = reinterpret_cast<const uint32_t*>(p.seeds);  // duplicates re-test a column: same result
    ncols = (unsigned)p.n_seeds;
  }
  if (p.n_seeds == 0) {  // empty @changed: no pass, status from D_in (include/rac.h)
    for (size_t x = gtid; x < (size_t)n; x += gthreads) {
      uint64_t v = 0;
#pragma unroll
      for (int w = 0; w < WS; ++w) v |= p.D[x * WS + w];
      if (!v) atomicOr(&slots[0].wipe, 1u);
    }
    grid.sync();
    status = *((volatile unsigned*)&slots[0].wipe) ? RAC_WIPEOUT : RAC_OK;
  }
  for (; p.n_seeds != 0;) {
    ++pass;
    const int s = pass % 3;
    for (int i = tid; i < n * WS; i += blockDim.x) sD[i] = __ldcg(p.D + i);  // L2: written by other SMs
    __syncthreads();

    // ---- a3/a4: support tests of the live rows against the tested columns
    const size_t rows = (size_t)n * dmax;
    // Few tested columns (a seeded pass 1, a late pass): a thread per row, so the
    // 31 idle lanes of the warp-per-row loop do not serialise the rows.
    if (ncols <= kThreadRowCols) {
      for (size_t r = gtid; r < rows; r += gthreads) {
        const int x = (int)(r / dmax), a = (int)(r % dmax);
        if (!((sD[(size_t)x * WS + (a >> 6)] >> (a & 63)) & 1ull)) continue;  // dead row
        const uint64_t* row = p.M + r * (size_t)n * WS;
        bool failed = false;
        for (unsigned i = 0; i < ncols && !failed; ++i) {
          const int y = cols ? (int)__ldcg(cols + i) : (int)i;
          if ((unsigned)y >= (unsigned)n) continue;  // a bad seed is skipped (as in rac_fused)
          const Mask<WS> m = load_mask<WS>(row + (size_t)y * WS);
          failed = !meets<WS>(m, sD + (size_t)y * WS) && present(p.P, p.pw, x, y);
        }
        if (failed) atomicOr(reinterpret_cast<unsigned long long*>(p.R) + (size_t)x * WS + (a >> 6),
                             1ull << (a & 63));
      }
    } else
    for (size_t r = gwarp; r < rows; r += nwarps) {
      const int x = (int)(r / dmax), a = (int)(r % dmax);
      if (!((sD[(size_t)x * WS + (a >> 6)] >> (a & 63)) & 1ull)) continue;  // dead row
      const uint64_t* row = p.M + r * (size_t)n * WS;
      bool failed = false;
      for (unsigned base = 0; base < ncols && !failed; base += 32u * 4u) {
        int ys[4];
        Mask<WS> m[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned i = base + (unsigned)u * 32u + (unsigned)lane;
          ys[u] = i < ncols ? (cols ? (int)__ldcg(cols + i) : (int)i) : -1;
          if ((unsigned)ys[u] >= (unsigned)n) ys[u] = -1;  // a bad seed is skipped (as in rac_fused)
          if (ys[u] >= 0) m[u] = load_mask<WS>(row + (size_t)ys[u] * WS);
        }
        bool f = false;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ys[u] >= 0 && !meets<WS>(m[u], sD + (size_t)ys[u] * WS) && present(p.P, p.pw, x, ys[u])) f = true;
        failed = __any_sync(0xffffffffu, f);
      }
      if (failed && lane == 0) atomicOr(reinterpret_cast<unsigned long long*>(p.R) + (size_t)x * WS + (a >> 6),
                                        1ull << (a & 63));
    }
    grid.sync();

    // ---- a5: D_t = D_{t-1} & ~R, change list, epochs, wipeout flag
    uint32_t* next_cols = p.clist + (size_t)s * n;
    for (size_t x = gtid; x < (size_t)n; x += gthreads) {
      bool chg = false, empty = true;
#pragma unroll
      for (int w = 0; w < WS; ++w) {
        const uint64_t rm = __ldcg(p.R + x * WS + w);
        uint64_t v = __ldcg(p.D + x * WS + w);
        if (rm) {
          chg = true;
          v &= ~rm;
          p.D[x * WS + w] = v;
          p.R[x * WS + w] = 0;
          if (p.removed_at) {
            uint64_t b = rm;
            while (b) {
              const int k = __ffsll((long long)b) - 1;
              b &= b - 1;
              p.removed_at[x * 64 * wq + 64 * w + k] = pass;
            }
          }
        }
        if (v) empty = false;
      }
      if (chg) next_cols[atomicAdd(&slots[s].cnt, 1u)] = (uint32_t)x;
      if (empty) atomicOr(&slots[s].wipe, 1u);
    }
    grid.sync();

    const unsigned cnt = *((volatile unsigned*)&slots[s].cnt);
    const unsigned wipe = *((volatile unsigned*)&slots[s].wipe);
    if (gtid == 0) slots[(pass + 1) % 3] = WideSlot{0u, 0u};
    if (wipe && !p.full) { status = RAC_WIPEOUT; break; }  // Alg. 1, checked first
    if (cnt == 0) { status = wipe ? RAC_WIPEOUT : RAC_OK; break; }
    cols = next_cols;
    ncols = cnt;
  }

  for (size_t i = gtid; i < (size_t)n * wq; i += gthreads) {
    const int x = (int)(i / wq), w = (int)(i % wq);
    p.d_out[i] = __ldcg(p.D + (size_t)x * WS + w);
  }
  if (gtid == 0) {
    *p.iters = pass;
    *p.status = status;
  }
}

// ---- a7 on wide domains: one thread block per domain state (batched mode,
// search-tree nodes, Alg. 2).  The block runs its
// state's whole enforcement -- Eq. 1 with Alg. 1's loop control, D / removal
// bits / tested-column list in shared memory, __syncthreads as the pass
// barrier -- so each state stops at its own pass; no cross-state barrier.
// Pass t: every live row (x,a) (thread-strided) is tested against the tested
// columns (the seed variable in pass 1 of a seeded state, all columns in pass 1
// of a root state, then the variables changed in pass t-1; Prop. 2), four
// masks in flight, early exit at the first declared c_xy with an empty
// support set.
template <int WS>
__global__ void __launch_bounds__(256) wide_state(WideStateParams p) {
  extern __shared__ uint64_t wsm[];
  __shared__ unsigned sc[256 / 32];
  const int n = p.n, dmax = p.dmax, wq = p.wq, tid = threadIdx.x, T = blockDim.x;
  const int s = p.s0 + blockIdx.x;
  uint64_t* D = wsm;                                          // [n*WS]
  unsigned long long* R = reinterpret_cast<unsigned long long*>(D + (size_t)n * WS);  // [n*WS]
  uint32_t* list = reinterpret_cast<uint32_t*>(R + (size_t)n * WS);                  // [n]
  uint32_t* nlist = list + n;                                                          // [n]
  const uint64_t* din = p.d_in + (size_t)s * n * wq;
  for (int i = tid; i < n * WS; i += T) {
    const int x = i / WS, w = i % WS;
    uint64_t v = 0;
    if (w < wq) {
      const int bits = min(64, max(0, p.dom[x] - 64 * w));
      v = din[(size_t)x * wq + w] & (bits >= 64 ? ~0ull : ((1ull << bits) - 1ull));
    }
    D[i] = v;
    R[i] = 0ull;
  }
  const int sv = p.seed_var ? p.seed_var[s] : -1;
  bool all_cols = !(sv >= 0 && sv < n);
  int cnt = all_cols ? n : 1;
  if (!all_cols && tid == 0) list[0] = (uint32_t)sv;
  __syncthreads();
  int has_empty = 0;
  for (int x = tid; x < n; x += T) {
    uint64_t v = 0;
#pragma unroll
    for (int w = 0; w < WS; ++w) v |= D[x * WS + w];
    has_empty |= v == 0ull;
  }
  has_empty = __syncthreads_or(has_empty);
  const int rows = n * dmax;
  int t = 0, status = RAC_OK;
  for (;;) {
    ++t;
    // a3/a4: live rows against the tested columns
    int any = 0;
    for (int r = tid; r < rows; r += T) {
      const int x = r / dmax, a = r - x * dmax;
      if (!((D[x * WS + (a >> 6)] >> (a & 63)) & 1ull)) continue;  // dead row
      const uint64_t* row = p.M + (size_t)r * n * WS;
      bool failed = false;
      for (int c0 = 0; c0 < cnt && !failed; c0 += 4) {
        Mask<WS> m[4];
        int yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          yv[u] = c0 + u < cnt ? (all_cols ? c0 + u : (int)list[c0 + u]) : -1;
          if (yv[u] >= 0) m[u] = load_mask<WS>(row + (size_t)yv[u] * WS);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (yv[u] >= 0 && !failed && !meets<WS>(m[u], D + (size_t)yv[u] * WS) && present(p.P, p.pw, x, yv[u]))
            failed = true;
      }
      if (failed) {
        // 32-bit shared atomic (native; a 64-bit one compiles to a CAS spin loop)
        atomicOr(reinterpret_cast<unsigned*>(&R[x * WS + (a >> 6)]) + ((a >> 5) & 1), 1u << (a & 31));
        any = 1;
      }
    }
    if (!__syncthreads_or(any)) {  // nothing removed: D_t = D_{t-1}
      status = has_empty ? RAC_WIPEOUT : RAC_OK;
      break;
    }
    // a5: D_t = D_{t-1} & ~R; changed variables (ascending) -> next columns
    const int per = (n + T - 1) / T, xb = min(n, tid * per), xe = min(n, xb + per);
    unsigned c = 0;
    for (int x = xb; x < xe; ++x) {
      unsigned long long rr = 0;
#pragma unroll
      for (int w = 0; w < WS; ++w) rr |= R[x * WS + w];
      c += rr != 0ull;
    }
    unsigned total = 0;
    {
      // block exclusive scan of c
      const int lane = tid & 31, wp = tid >> 5, nw = T >> 5;
      unsigned v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane == 31) sc[wp] = v;
      __syncthreads();
      unsigned base = 0;
      for (int k = 0; k < nw; ++k) {
        if (k < wp) base += sc[k];
        total += sc[k];
      }
      c = base + v - c;  // exclusive prefix
    }
    int wipe = has_empty;
    for (int x = xb; x < xe; ++x) {
      bool chx = false, empty = true;
#pragma unroll
      for (int w = 0; w < WS; ++w) {
        const unsigned long long rr = R[x * WS + w];
        if (rr) {
          chx = true;
          D[x * WS + w] &= ~rr;
          R[x * WS + w] = 0ull;
        }
        if (D[x * WS + w]) empty = false;
      }
      if (chx) {
        nlist[c++] = (uint32_t)x;
        wipe |= empty;
      }
    }
    wipe = __syncthreads_or(wipe);
    uint32_t* tmp = list;
    list = nlist;
    nlist = tmp;
    all_cols = false;
    cnt = (int)total;
    has_empty = wipe;
    if (wipe && !p.full) { status = RAC_WIPEOUT; break; }  // Alg. 1, checked first
    if (cnt == 0) { status = wipe ? RAC_WIPEOUT : RAC_OK; break; }
  }
  uint64_t* dout = p.d_out + (size_t)s * n * wq;
  for (int i = tid; i < n * wq; i += T) dout[i] = D[(size_t)(i / wq) * WS + (i % wq)];
  if (tid == 0) {
    p.iters[s] = t;
    p.status[s] = status;
  }
}

// ---- a1: packing.  One CTA per constrained pair: the d x d relation bit matrix
// in smem (rows a, words of b), its transpose, both orientations written.
template <bool GEN>
__global__ void __launch_bounds__(256) wide_pack(WidePack g, const int32_t* xs, const int32_t* ys,
                                                 const uint64_t* rows, int n_pairs, int d, uint32_t t_q16,
                                                 uint64_t seed) {
  __shared__ uint64_t F[256 * 4];  // F[a][w] = c_xy|(x,a)
  __shared__ uint64_t T[256 * 4];  // T[b][w] = c_yx|(y,b)
  const int WS = g.WS, n = g.n, dmax = g.dmax;
  for (long long pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
    int x, y;
    if (GEN) {
      // pair index -> (x < y) by rows of the upper triangle
      x = 0;
      long long rem = pr;
      while (rem >= n - 1 - x) { rem -= n - 1 - x; ++x; }
      y = x + 1 + (int)rem;
      if (!synth_present(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y, g.dens_q32)) continue;  // block-uniform
    } else {
      x = xs[pr];
      y = ys[pr];
    }
    const int dx = GEN ? d : g.dom[x], dy = GEN ? d : g.dom[y];
    for (int i = threadIdx.x; i < 256 * 4; i += blockDim.x) { F[i] = 0; T[i] = 0; }
    __syncthreads();
    if (GEN) {
      const uint64_t pk = synth_pair_key(seed, (uint32_t)n, (uint32_t)x, (uint32_t)y);
      const int q = (d + 3) / 4;
      for (int i = threadIdx.x; i < d * q; i += blockDim.x) {
        const int a = i / q, bq = i % q;
        const uint64_t h = synth_cell_word_pk(pk, (uint32_t)d, (uint32_t)a, (uint32_t)bq);
        uint64_t bits = 0;
        for (int j = 0; j < 4 && bq * 4 + j < d; ++j)
          if (((h >> (16 * j)) & 0xFFFFull) >= t_q16) bits |= 1ull << j;
        if (bits) {
          const int b0 = bq * 4;  // 4 | 64: the nibble never straddles a word
          atomicOr(reinterpret_cast<unsigned long long*>(&F[a * 4 + (b0 >> 6)]), bits << (b0 & 63));
        }
      }
    } else {
      for (int i = threadIdx.x; i < dx * g.wq; i += blockDim.x)
        F[(i / g.wq) * 4 + (i % g.wq)] = rows[((size_t)pr * dmax + i / g.wq) * g.wq + (i % g.wq)];
    }
    __syncthreads();
    // transpose: T[b] bit a = F[a] bit b
    for (int i = threadIdx.x; i < dy * 4; i += blockDim.x) {
      const int b = i >> 2, w = i & 3;
      uint64_t v = 0;
      for (int k = 0; k < 64; ++k) {
        const int a = 64 * w + k;
        if (a < dx && ((F[a * 4 + (b >> 6)] >> (b & 63)) & 1ull)) v |= 1ull << k;
      }
      T[b * 4 + w] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < dx * WS; i += blockDim.x)
      g.M[(((size_t)x * dmax + i / WS) * n + y) * WS + (i % WS)] = F[(i / WS) * 4 + (i % WS)];
    for (int i = threadIdx.x; i < dy * WS; i += blockDim.x)
      g.M[(((size_t)y * dmax + i / WS) * n + x) * WS + (i % WS)] = T[(i / WS) * 4 + (i % WS)];
    if (threadIdx.x == 0) {
      atomicOr(g.P + (size_t)x * g.pw + (y >> 5), 1u << (y & 31));
      atomicOr(g.P + (size_t)y * g.pw + (x >> 5), 1u << (x & 31));
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_wide_fused(const WideParams& p, int grid, size_t smem, cudaStream_t s) {
  void* args[] = {const_cast<WideParams*>(&p)};
  if (p.WS == 2)
    return cudaLaunchCooperativeKernel((const void*)wide_fused<2>, grid, kWideThreads, args, smem, s);
  return cudaLaunchCooperativeKernel((const void*)wide_fused<4>, grid, kWideThreads, args, smem, s);
}

cudaError_t wide_fused_grid(int WS, size_t smem, int sm_count, int* grid) {
  const void* fn = WS == 2 ? (const void*)wide_fused<2> : (const void*)wide_fused<4>;
  // the attribute is per function: set the largest size any context may use
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWideThreads, smem);
  if (e != cudaSuccess) return e;
  *grid = per_sm * sm_count;
  return *grid > 0 ? cudaSuccess : cudaErrorInvalidConfiguration;
}

size_t wide_state_smem(int n, int WS) { return (size_t)n * WS * 16 + (size_t)n * 8; }

cudaError_t launch_wide_state(const WideStateParams& p, int n_states, cudaStream_t s) {
  const size_t smem = wide_state_smem(p.n, p.WS);
  const void* k = p.WS == 2 ? (const void*)wide_state<2> : (const void*)wide_state<4>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p.WS == 2) wide_state<2><<<n_states, 256, smem, s>>>(p);
  else wide_state<4><<<n_states, 256, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_wide_pack(const WidePack& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                             int n_rel, cudaStream_t s) {
  if (n_rel <= 0) return cudaSuccess;
  wide_pack<false><<<std::min(n_rel, 148 * 16), 256, 0, s>>>(g, xs, ys, rows, n_rel, 0, 0u, 0ull);
  return cudaGetLastError();
}

cudaError_t launch_wide_generate(const WidePack& g, int d, uint32_t t_q16, uint64_t seed, cudaStream_t s) {
  const long long pairs = (long long)g.n * (g.n - 1) / 2;
  if (pairs <= 0) return cudaSuccess;
  const int grid = (int)std::min<long long>(pairs, 148LL * 16);
  wide_pack<true><<<grid, 256, 0, s>>>(g, nullptr, nullptr, nullptr, (int)pairs, d, t_q16, seed);
  return cudaGetLastError();
}

}  // namespace rac
