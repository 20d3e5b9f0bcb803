// rac_state.cu -- one thread block per domain state: the batched mode (SURVEY
// §8(a7), many search-tree nodes, Alg. 2) and the
// single-CTA enforcement of small instances (C1-sized, latency-bound).
//
// Each block runs the whole RAC enforcement of ITS state on its own: Eq. 1
// (intersection form of line 59) with Alg. 1's loop
// control (lines 198-210), D_t / the removal bits / the tested-column list in
// shared memory, __syncthreads as the pass barrier, so a state stops at its
// own pass (freeze-on-stop is free) and no block ever waits for another.
// States are independent: the grid is simply one block per state and the
// hardware keeps as many resident as fit (no grid-wide barrier, no exchange).
//
// Support test (a3/a4): pass t tests the live rows (x,a) against the columns
// of the variables changed in pass t-1 (all columns in pass 1 of a root call,
// the seed variables in pass 1 of a seeded call -- Alg. 1's Cons[:, @changed],
// line 215, Prop. 2).  Work item = one 16-byte vector of a
// tested column of the column-major mask tensor (16/W rows (x, a..a+16/W-1)),
// loaded with ld.global.nc (the relation of a batched instance is shared by
// every block and stays L2-resident) only when one of its rows is live in
// D_{t-1} and c_xy is declared (presence bitmap staged in shared memory):
// dead rows, absent pairs and the diagonal cost no load.  mask & D(y) == 0 on
// a live row is a removal (atomicOr into R[x] in shared memory).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

constexpr uint32_t kFullS = 1u;  // RAC_FULL_FIXPOINT
constexpr int kOKs = 0, kWIPEOUTs = 1;
constexpr int kUs = 8;  // vector loads in flight per thread

// Block-wide exclusive scan of one int per thread; returns the prefix, *total
// gets the sum.  `sc` holds blockDim/32 ints.
__device__ __forceinline__ int scan_excl(int v, int* total, int* sc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (nw == 1) {
    *total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  }
  __syncthreads();
  if (lane == 31) sc[w] = x;
  __syncthreads();
  int base = 0, tot = 0;
  for (int k = 0; k < nw; ++k) {
    const int s = sc[k];
    if (k < w) base += s;
    tot += s;
  }
  *total = tot;
  return base + x - v;
}

// live rows of vector v (L = 16/W rows r0 = v*L ..) as an L-bit mask
template <int W>
__device__ __forceinline__ uint32_t vec_live(const uint8_t* Db, int v, int n, int dmax, bool aligned) {
  constexpr int L = 16 / W;
  constexpr uint32_t LM = L == 32 ? 0xffffffffu : ((1u << L) - 1u);
  const int r0 = v * L;
  if (aligned) {  // dmax % L == 0: the L rows are values a0.. of one variable
    const int x = r0 / dmax;
    if (x >= n) return 0u;
    const int a0 = r0 - x * dmax;
    return (uint32_t)(load_w<W>(Db + x * W) >> a0) & LM;
  }
  uint32_t m = 0;
  for (int i = 0; i < L; ++i) {
    const int r = r0 + i, x = r / dmax;
    if (x >= n) break;
    const int a = r - x * dmax;
    m |= (uint32_t)((load_w<W>(Db + x * W) >> a) & 1u) << i;
  }
  return m;
}

template <int W, int T>
__global__ void __launch_bounds__(T) rac_state(StateParams p) {
  constexpr int L = 16 / W;
  extern __shared__ uint4 smem4[];
  __shared__ int sc[T / 32 > 0 ? T / 32 : 1];
  const int n = p.n, dmax = p.dmax, tid = threadIdx.x;
  const int s = blockIdx.x;
  // phase stamps (tooling, RAC_DEBUG_TIMELINE): thread 0 of block 0
  int nd = 0;
  const bool dbg = p.dbg != nullptr && blockIdx.x == 0 && tid == 0;
#define RAC_SMARK() do { if (dbg && nd < 255) p.dbg[1 + nd++] = globaltimer(); } while (0)
  RAC_SMARK();
  const int nvec = p.nvec;  // 16-byte vectors per column
  const bool aligned = (dmax % L) == 0;
  // shared memory: D | R (u64 per variable) | live[nvec] (u32) | vx[nvec] (u16) | list | nlist | P (optional)
  uint8_t* Db = reinterpret_cast<uint8_t*>(smem4);
  unsigned long long* R = reinterpret_cast<unsigned long long*>(Db + p.off_R);
  uint32_t* live = reinterpret_cast<uint32_t*>(Db + p.off_live);
  uint16_t* vx = reinterpret_cast<uint16_t*>(Db + p.off_vx);
  uint16_t* list = reinterpret_cast<uint16_t*>(Db + p.off_list);
  uint16_t* nlist = reinterpret_cast<uint16_t*>(Db + p.off_nlist);
  const uint32_t* Ps = p.off_P ? reinterpret_cast<const uint32_t*>(Db + p.off_P) : nullptr;
  // a tiny relation (C1: 10 KB) is staged in shared memory once, so no pass
  // waits on L2: the passes of a latency-bound enforcement run from smem
  const uint4* Ms = p.off_M ? reinterpret_cast<const uint4*>(Db + p.off_M) : nullptr;
  const size_t cs16 = p.col_stride / 16;

  // ---- stage D_0 = d_in (bits beyond dom dropped), P, per-vector variable
  const uint64_t* din = p.d_in + (size_t)(p.s0 + s) * n;
  for (int x = tid; x < n; x += T) {
    store_w<W>(Db + x * W, __ldg(din + x) & __ldg(p.dommask + x));
    R[x] = 0ull;
  }
  if (Ps)
    for (int i = tid; i < n * p.pw; i += T) const_cast<uint32_t*>(Ps)[i] = __ldg(p.P + i);
  __shared__ alignas(8) uint64_t mbar;
  if (Ms) bulk_stage_start(const_cast<uint4*>(Ms), p.M, (uint32_t)((size_t)n * p.col_stride), &mbar);
  for (int v = tid; v < nvec; v += T) {
    const int r0 = v * L, x0 = r0 / dmax, x1 = (r0 + L - 1) / dmax;
    // one variable per vector (absent-pair skip allowed) -> x0, else 0xffff
    vx[v] = (x0 == x1 && x0 < n) ? (uint16_t)x0 : (uint16_t)0xffffu;
  }
  // ---- initial tested columns: the seeds (seeded call) or every column
  int cnt = n;
  bool all_cols = true;
  {
    const int sv = p.seed_var ? p.seed_var[p.s0 + s] : -1;
    if (p.n_seeds >= 0 || (sv >= 0 && sv < n)) {
      all_cols = false;
      // flags in nlist (as u16), then compact into list
      for (int i = tid; i < n; i += T) nlist[i] = 0;
      __syncthreads();
      if (p.n_seeds >= 0) {
        for (int i = tid; i < p.n_seeds; i += T) {
          const int y = p.seeds[i];
          if (y >= 0 && y < n) nlist[y] = 1;
        }
      } else if (tid == 0) {
        nlist[sv] = 1;
      }
      __syncthreads();
      int c = 0, total = 0;
      const int per = (n + T - 1) / T, b = min(n, tid * per), e = min(n, b + per);
      for (int i = b; i < e; ++i) c += nlist[i] != 0;
      int pos = scan_excl(c, &total, sc);
      for (int i = b; i < e; ++i)
        if (nlist[i]) list[pos++] = (uint16_t)i;
      cnt = total;
    }
  }
  if (Ms) bulk_stage_wait(&mbar);
  __syncthreads();
  RAC_SMARK();
  int has_empty = 0;
  for (int x = tid; x < n; x += T) has_empty |= load_w<W>(Db + x * W) == 0;
  has_empty = __syncthreads_or(has_empty);
  for (int v = tid; v < nvec; v += T) live[v] = vec_live<W>(Db, v, n, dmax, aligned);
  __syncthreads();

  const bool full = (p.flags & kFullS) != 0;
  int t = 0, status = kOKs;
  if (cnt == 0) {  // empty @changed: no pass, status from D_in
    status = has_empty ? kWIPEOUTs : kOKs;
  } else {
    RAC_SMARK();
    for (;;) {
      ++t;
      // ---- a3/a4: sweep (items = tested column c x vector v)
      int c = tid / nvec, v = tid - c * nvec;
      bool any_rm = false;
      while (c < cnt) {
        uint4 m[kUs];
        int yy[kUs], vv[kUs];
        uint32_t lv[kUs];
#pragma unroll
        for (int u = 0; u < kUs; ++u) {
          lv[u] = 0u;
          if (c < cnt) {
            const int y = all_cols ? c : (int)list[c];
            const uint32_t l = live[v];
            const int xv = vx[v];
            // skip: no live row; or the vector's variable has no declared c_xy
            // (absent pair / diagonal: all-ones masks never fail a non-empty D(y))
            bool need = l != 0u;
            if (need && xv != 0xffff && (xv == y || (Ps && !((Ps[xv * p.pw + (y >> 5)] >> (y & 31)) & 1u))))
              need = false;
            if (need) {
              lv[u] = l;
              yy[u] = y;
              vv[u] = v;
              m[u] = Ms ? Ms[(size_t)y * cs16 + v]
                        : ldg_stream(reinterpret_cast<const uint4*>(p.M + (size_t)y * p.col_stride) + v);
            }
            v += T;
            while (v >= nvec) { v -= nvec; ++c; }
          }
        }
#pragma unroll
        for (int u = 0; u < kUs; ++u) {
          if (!lv[u]) continue;
          const int y = yy[u];
          const uint64_t dv = load_w<W>(Db + y * W);
          const uint32_t z = zero_lanes<W>(and4(m[u], rep16<W>(dv))) & lv[u];
          if (!z) continue;
          for (uint32_t zz = z; zz; zz &= zz - 1u) {
            const int r = vv[u] * L + __ffs(zz) - 1;
            const int x = r / dmax, a = r - x * dmax;
            // R2: an all-ones absent pair only "fails" on an empty D(y); then P decides
            if (dv == 0ull && !((__ldg(p.P + (size_t)x * p.pw + (y >> 5)) >> (y & 31)) & 1u)) continue;
            // 32-bit shared atomic (native; a 64-bit one compiles to a CAS spin loop)
            atomicOr(reinterpret_cast<unsigned*>(&R[x]) + (a >> 5), 1u << (a & 31));
            any_rm = true;
            if (p.removed_at) p.removed_at[(size_t)x * 64 + a] = t;
          }
        }
      }
      const int removed_any = __syncthreads_or(any_rm);
      RAC_SMARK();
      // ---- a5: D_t = D_{t-1} & ~R; the changed variables (R[x] != 0: marks are
      // made on live rows only) become the next pass's tested columns
      int changed = 0, wipe = has_empty;
      if (removed_any) {
        const int per = (n + T - 1) / T, b = min(n, tid * per), e = min(n, b + per);
        int cx = 0;
        for (int x = b; x < e; ++x) cx += R[x] != 0ull;
        int total = 0;
        int pos = scan_excl(cx, &total, sc);
        for (int x = b; x < e; ++x) {
          const unsigned long long r = R[x];
          if (!r) continue;
          const uint64_t nd = load_w<W>(Db + x * W) & ~r;
          store_w<W>(Db + x * W, nd);
          R[x] = 0ull;
          wipe |= nd == 0ull;
          nlist[pos++] = (uint16_t)x;
        }
        changed = total;
        wipe = __syncthreads_or(wipe);
        uint16_t* tmp = list;
        list = nlist;
        nlist = tmp;
        all_cols = false;
        cnt = total;
      }
      has_empty = wipe;
      if (wipe && !full) { status = kWIPEOUTs; break; }          // Alg. 1
      if (!changed) { status = wipe ? kWIPEOUTs : kOKs; break; }  // Prop. 1 end condition
      RAC_SMARK();
      for (int v2 = tid; v2 < nvec; v2 += T) live[v2] = vec_live<W>(Db, v2, n, dmax, aligned);
      __syncthreads();
      RAC_SMARK();
    }
  }
  RAC_SMARK();
  uint64_t* dout = p.d_out + (size_t)(p.s0 + s) * n;
  for (int x = tid; x < n; x += T) dout[x] = load_w<W>(Db + x * W);
  if (tid == 0) {
    p.iters[p.s0 + s] = t;
    p.status[p.s0 + s] = status;
  }
  RAC_SMARK();
  if (dbg) p.dbg[0] = nd;
#undef RAC_SMARK
}

// ---------------------------------------------------------------------------- rac_tiny
// One small BLOCK (kTinyT threads) runs the whole enforcement of a tiny
// instance (n <= 64 variables; the mask tensor staged in shared memory by one
// bulk copy): thread per row (x,a), the row's tested-and-declared columns as a
// 64-bit set (reading R2: an absent pair never removes) taken four at a time so
// the shared-memory loads overlap, early exit on the first empty support set;
// __syncthreads as the pass barrier, block-wide OR reductions for Alg. 1's loop
// control (lines 198-210: wipeout checked first, then "changed").  C1 (n = 20,
// d = 8: 160 rows) is one row per thread.
constexpr int kTinyT = 256;

template <int W>
__global__ void __launch_bounds__(kTinyT) rac_tiny(StateParams p) {
  extern __shared__ uint4 tsm4[];
  __shared__ alignas(8) uint64_t mbar;
  __shared__ unsigned s_or[2];  // the pass's changed variables (low / high word)
  const int n = p.n, dmax = p.dmax, tid = threadIdx.x;
  uint8_t* Ms = reinterpret_cast<uint8_t*>(tsm4);  // n * col_stride bytes
  unsigned long long* D = reinterpret_cast<unsigned long long*>(Ms + (((size_t)n * p.col_stride + 15) & ~(size_t)15));
  unsigned long long* R = D + 64;
  unsigned long long* Pm = R + 64;  // Pm[x]: bit y set iff c_xy is declared
  const int s = p.s0 + blockIdx.x;
  int nd = 0;  // phase stamps (tooling, RAC_DEBUG_TIMELINE): thread 0 of block 0
  const bool dbg = p.dbg != nullptr && blockIdx.x == 0 && tid == 0;
#define RAC_TMARK() do { if (dbg && nd < 255) p.dbg[1 + nd++] = globaltimer(); } while (0)
  RAC_TMARK();
  // the whole mask tensor in one bulk copy (TMA engine) while D and P load
  bulk_stage_start(Ms, p.M, (uint32_t)((size_t)n * p.col_stride), &mbar);
  if (tid < 64) {
    const int x = tid;
    D[x] = x < n ? __ldg(p.d_in + (size_t)s * n + x) & __ldg(p.dommask + x) : ~0ull;
    R[x] = 0ull;
    unsigned long long pm = 0;
    if (x < n) {
      pm = __ldg(p.P + (size_t)x * p.pw);
      if (p.pw > 1) pm |= (unsigned long long)__ldg(p.P + (size_t)x * p.pw + 1) << 32;
    }
    Pm[x] = pm;
  }
  if (tid < 2) s_or[tid] = 0u;
  // tested columns of pass 1: the seeds (seeded call), else every column
  unsigned long long T = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
  const int sv = p.seed_var ? p.seed_var[s] : -1;
  if (p.n_seeds >= 0) {
    unsigned long long m = 0;
    for (int i = tid & 31; i < p.n_seeds; i += 32) {  // every warp computes the same set
      const int y = p.seeds[i];
      if (y >= 0 && y < n) m |= 1ull << y;
    }
    for (int o = 16; o; o >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
    T = m;
  } else if (sv >= 0 && sv < n) {
    T = 1ull << sv;
  }
  bulk_stage_wait(&mbar);  // includes a __syncthreads: D, P visible
  RAC_TMARK();
  int has_empty = __syncthreads_or(tid < n && D[tid] == 0ull);
  const bool full = (p.flags & 1u) != 0;
  const int rows = n * dmax;
  int t = 0, status = 0;
  if (T == 0ull) {
    status = has_empty ? 1 : 0;  // empty @changed: no pass
  } else {
    for (;;) {
      ++t;
      bool any = false;
      for (int r = tid; r < rows; r += kTinyT) {
        const int x = r / dmax, a = r - x * dmax;
        if (!((D[x] >> a) & 1ull)) continue;  // dead row
        const uint8_t* mrow = Ms + (size_t)r * W;
        bool failed = false;
        for (unsigned long long cols = T & Pm[x]; cols && !failed;) {
          int yv[4];
          uint64_t mv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            yv[u] = cols ? __ffsll((long long)cols) - 1 : -1;
            cols &= cols - 1ull;
            if (yv[u] >= 0) mv[u] = load_w<W>(mrow + (size_t)yv[u] * p.col_stride);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (yv[u] >= 0 && (mv[u] & D[yv[u]]) == 0ull) failed = true;
        }
        if (failed) {
          // 32-bit shared atomic (native; a 64-bit one compiles to a CAS spin loop)
          atomicOr(reinterpret_cast<unsigned*>(&R[x]) + (a >> 5), 1u << (a & 31));
          if (p.removed_at) p.removed_at[(size_t)x * 64 + a] = t;
          any = true;
        }
      }
      if (!__syncthreads_or(any)) {  // nothing removed: D_t = D_{t-1}
        RAC_TMARK();
        status = has_empty ? 1 : 0;
        break;
      }
      RAC_TMARK();
      int wl = 0;
      if (tid < n) {
        const int x = tid;
        const unsigned long long rr = R[x];
        if (rr) {
          const unsigned long long nd2 = D[x] & ~rr;
          D[x] = nd2;
          R[x] = 0ull;
          atomicOr(&s_or[x >> 5], 1u << (x & 31));
          wl = nd2 == 0ull;
        }
      }
      const int wipe = has_empty | __syncthreads_or(wl);
      const unsigned long long C = ((unsigned long long)s_or[1] << 32) | s_or[0];
      __syncthreads();
      if (tid < 2) s_or[tid] = 0u;  // ordered before the next pass's atomics by its barrier
      has_empty = wipe;
      if (wipe && !full) { status = 1; break; }   // Alg. 1
      if (C == 0ull) { status = wipe ? 1 : 0; break; }
      T = C;  // the changed variables are the next pass's columns (Prop. 2)
      RAC_TMARK();
    }
  }
  if (tid < n) p.d_out[(size_t)s * n + tid] = D[tid];
  if (tid == 0) {
    p.iters[s] = t;
    p.status[s] = status;
  }
  RAC_TMARK();
  if (dbg) p.dbg[0] = nd;
#undef RAC_TMARK
}

template <int W, int T>
struct LaunchS {
  static cudaError_t go(const StateParams& p, int n_states, size_t smem, cudaStream_t st) {
    auto k = rac_state<W, T>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k<<<n_states, T, smem, st>>>(p);
    return cudaGetLastError();
  }
};

}  // namespace

size_t tiny_smem(int n, size_t col_stride) { return (((size_t)n * col_stride + 15) & ~(size_t)15) + 3 * 64 * 8; }

// One block; 16-byte loads of pinned host memory, all in flight at once (the
// staging is 16-byte aligned and padded: d_in words then the seeds).
__global__ void __launch_bounds__(512) stage_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                         uint32_t n16, const uint32_t* __restrict__ tsrc,
                                                         uint32_t* __restrict__ tdst, uint32_t ntail) {
  for (uint32_t i0 = threadIdx.x; i0 < n16; i0 += 4 * blockDim.x) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * blockDim.x < n16) v[k] = src[i0 + k * blockDim.x];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * blockDim.x < n16) dst[i0 + k * blockDim.x] = v[k];
  }
  if (threadIdx.x < ntail) tdst[threadIdx.x] = tsrc[threadIdx.x];
}

cudaError_t launch_stage_copy(const void* host_src, void* dev_dst, size_t bytes, cudaStream_t s) {
  if (((uintptr_t)host_src | (uintptr_t)dev_dst) & 15) return cudaErrorInvalidValue;
  const uint32_t n16 = (uint32_t)(bytes / 16), ntail = (uint32_t)((bytes - (size_t)n16 * 16) / 4);
  stage_copy_kernel<<<1, 512, 0, s>>>(reinterpret_cast<const uint4*>(host_src), reinterpret_cast<uint4*>(dev_dst),
                                      n16, reinterpret_cast<const uint32_t*>(host_src) + n16 * 4,
                                      reinterpret_cast<uint32_t*>(dev_dst) + n16 * 4, ntail);
  return cudaGetLastError();
}

cudaError_t launch_tiny(int W, const StateParams& p, int n_states, size_t smem, cudaStream_t st) {
  const void* k = W == 1 ? (const void*)rac_tiny<1> : W == 2 ? (const void*)rac_tiny<2> : W == 4 ? (const void*)rac_tiny<4>
                                                                                                  : (const void*)rac_tiny<8>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  StateParams pp = p;
  void* args[] = {&pp};
  return cudaLaunchKernel(k, dim3(n_states), dim3(kTinyT), args, smem, st);
}

// Shared-memory layout of rac_state for an instance (offsets into the dynamic
// buffer); returns the total bytes.  P is staged only if it fits in `p_cap`.
size_t state_layout(StateParams& p, int n, int dmax, int W, int rows_pad, int pw, size_t p_cap, size_t m_cap) {
  const int L = 16 / W;
  p.nvec = (rows_pad + L - 1) / L;
  size_t off = (((size_t)n * W) + 15) & ~(size_t)15;  // D
  p.off_R = (uint32_t)off;
  off += (size_t)n * 8;
  p.off_live = (uint32_t)off;
  off += ((size_t)p.nvec * 4 + 15) & ~(size_t)15;
  p.off_vx = (uint32_t)off;
  off += ((size_t)p.nvec * 2 + 15) & ~(size_t)15;
  p.off_list = (uint32_t)off;
  off += ((size_t)n * 2 + 15) & ~(size_t)15;
  p.off_nlist = (uint32_t)off;
  off += ((size_t)n * 2 + 15) & ~(size_t)15;
  const size_t pb = (size_t)n * pw * 4;
  if (pb <= p_cap) {
    p.off_P = (uint32_t)off;
    off += (pb + 15) & ~(size_t)15;
  } else {
    p.off_P = 0;
  }
  const size_t mb = (size_t)n * rows_pad * W;  // the whole column-major mask tensor
  if (mb <= m_cap) {
    off = (off + 15) & ~(size_t)15;
    p.off_M = (uint32_t)off;
    off += mb;
  } else {
    p.off_M = 0;
  }
  return off;
}

cudaError_t launch_state(int W, int T, const StateParams& p, int n_states, size_t smem, cudaStream_t st) {
#define RAC_T_SWITCH(WW)                                        \
  switch (T) {                                                  \
    case 32: return LaunchS<WW, 32>::go(p, n_states, smem, st);   \
    case 128: return LaunchS<WW, 128>::go(p, n_states, smem, st); \
    case 256: return LaunchS<WW, 256>::go(p, n_states, smem, st); \
    default: return cudaErrorInvalidValue;                      \
  }
  switch (W) {
    case 1: RAC_T_SWITCH(1)
    case 2: RAC_T_SWITCH(2)
    case 4: RAC_T_SWITCH(4)
    case 8: RAC_T_SWITCH(8)
    default: return cudaErrorInvalidValue;
  }
#undef RAC_T_SWITCH
}

}  // namespace rac
