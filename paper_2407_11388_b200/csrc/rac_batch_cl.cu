// rac_batch_cl.cu -- batched enforcement: 32 domain states
// per bit-sliced word, each word owned by ONE thread-block cluster.
//
// Many search-tree nodes (Alg. 2) on one instance.
// As in rac_batch.cu the states are bit-sliced: for a word of 32 states,
// X[(x,a)] is a u32 whose bit j says (x,a) ∈ D_j, and one pass of Eq. 1
// (lines 89-99) for all 32 states is
//   X'[(x,a)] = X[(x,a)] & AND_{y ∈ C_x} ( OR_{b ∈ c_xy|(x,a)} X[(y,b)] )
// with the OR over b read from per-pass nibble tables
//   T[y][q][v] = OR_{j : bit j of v} X[(y, 4q+j)]     (ceil(d/4) lookups per mask).
// Per-state loop control (Alg. 1): wipeout first, then
// "changed", each state frozen at its own pass.  The tested columns of a pass
// are the union over the word's active states of the variables that changed
// for them in the previous pass (the seed variable of a seeded state in pass 1;
// Prop. 2, lines 130-143 -- testing a column that did not change for a state
// re-passes, so the union is exact).
//
// What is different from rac_batch.cu (the r01 design measured at 0.68 ms per
// C5 batch: 13 CTAs per word meeting at a global atomic barrier and exchanging
// their rows through a global double buffer):
//   * the word's CTAs form ONE cluster (C <= 8 CTAs, rows split between them);
//     passes are separated by cluster barriers (barrier.cluster) and the new
//     rows are exchanged through distributed shared memory -- no global
//     barrier, no global exchange buffer;
//   * every CTA keeps the whole word's slices in its shared memory and copies
//     from the other CTAs only the rows of variables that changed;
//   * a row takes one 16/W-byte... (column-major mask loads, 8 in flight per
//     thread) and stops as soon as none of its live states is supported.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace cg = cooperative_groups;

namespace rac {

namespace {

constexpr uint32_t kFullCL = 1u;  // RAC_FULL_FIXPOINT
constexpr int kMaxT = 1024;

template <int W>
__device__ __forceinline__ uint32_t mask_at(const uint8_t* p) {
  if constexpr (W == 4) return __ldg(reinterpret_cast<const uint32_t*>(p));
  else if constexpr (W == 2) return __ldg(reinterpret_cast<const uint16_t*>(p));
  else return __ldg(p);
}

// The support test of my rows against the pass's tested columns.  ci[c] =
// {byte offset of column c's masks, word offset of its nibble tables}; the
// list is padded to a multiple of 8 with copies of its last column (a column
// tested twice gives the same answer), so the 8-wide inner loop has no bounds
// checks.  CP: some active state has an empty domain (pass 1 of an input with
// an empty row, or full mode), so an all-ones mask of an absent pair could
// "fail" and the presence bit must decide (reading R2); otherwise no absent
// pair can fail and the presence test is skipped.
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

template <int W, bool CP>
__device__ __forceinline__ uint32_t sweep_rows(const uint8_t* __restrict__ M, const uint32_t* __restrict__ P, int pw,
                                               uint32_t* X, const uint32_t* Tb, const uint2* ci, int cnt8, int r0,
                                               int r1, int dmax, uint32_t active, uint32_t* chgn) {
  constexpr int NQ = 2 * W;
  // nibble tables addressed with 32-bit shared-memory addresses: ci[c].y is the
  // byte offset of column c's tables, the nibble q of the mask selects the
  // word (v << 2) of its 16-entry table at byte q * 64
  const uint32_t tb0 = (uint32_t)__cvta_generic_to_shared(Tb);
  uint32_t my_or = 0u;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    const uint32_t cur = X[r];
    const uint32_t live = cur & active;
    if (!live) continue;
    const uint8_t* Mrow = M + (size_t)r * W;
    const int x = r / dmax;
    uint32_t acc = 0xffffffffu;
    for (int c0 = 0; c0 < cnt8 && (acc & live) != 0u; c0 += 8) {
      uint32_t mv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mv[u] = mask_at<W>(Mrow + ci[c0 + u].x);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t ty = tb0 + ci[c0 + u].y;
        const uint32_t m = mv[u];
        uint32_t sup = lds32(ty + ((m << 2) & 0x3Cu));
#pragma unroll
        for (int q = 1; q < NQ; ++q) sup |= lds32(ty + 64u * q + ((m >> (4 * q - 2)) & 0x3Cu));
        if constexpr (CP) {
          if ((sup & live) != live) {
            const int y = (int)(ci[c0 + u].y / (NQ * 64));
            if (!((__ldg(P + (size_t)x * pw + (y >> 5)) >> (y & 31)) & 1u)) sup = 0xffffffffu;
          }
        }
        acc &= sup;
      }
    }
    const uint32_t nb = cur & (acc | ~active);
    if (nb != cur) {
      X[r] = nb;
      atomicOr(&chgn[x], cur ^ nb);
      my_or |= cur ^ nb;
    }
  }
  return my_or;
}

}  // namespace

// Shared memory (dynamic): X [rows4] u32 | T [n][NQ][16] u32 | chg [n] u32 |
// chgn [n] u32 | list [n] u16.  Cluster rank k owns rows [k*RPC, (k+1)*RPC),
// RPC a multiple of dmax, so every variable's rows live in one CTA.
template <int W>
__global__ void __launch_bounds__(kMaxT, 1) rac_batch_cl(BatchCLParams p) {
  constexpr int NQ = 2 * W;  // nibbles per mask (d <= 8W <= 32)
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t s_part[2];   // this CTA's [changed lanes OR, non-empty lanes AND]
  __shared__ int sc[kMaxT / 32];
  __shared__ int s_iters[32], s_status[32];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int k = (int)cluster.block_rank();
  const int g = blockIdx.x / C, G = gridDim.x / C;
  const int n = p.n, dmax = p.dmax, rows = n * dmax, rows4 = (rows + 3) & ~3;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = T >> 5;
  uint32_t* X = sm;
  uint32_t* Tb = X + rows4;
  uint32_t* chg = Tb + (size_t)n * NQ * 16;
  uint32_t* chgn = chg + n;
  uint16_t* list = reinterpret_cast<uint16_t*>(chgn + n);
  uint2* ci = reinterpret_cast<uint2*>(list + (((size_t)n + 7) & ~(size_t)7));  // [n + 8] column info
  const int r0 = k * p.RPC, r1 = min(rows, r0 + p.RPC);  // my rows
  const int x0 = r0 / dmax, x1 = (r1 + dmax - 1) / dmax;  // my variables
  const bool full = (p.flags & kFullCL) != 0;
  const int NW = (p.S + 31) / 32;
  // debug stamps: per word [start, staged, per pass: list, tables, sweep, A, B], end
  int nd = 0;
  const bool dbg = p.dbg != nullptr && k == 0 && tid == 0;
#define CL_MARK() do { if (dbg && nd < 255) p.dbg[(size_t)g * 256 + nd++] = globaltimer(); } while (0)

  for (int w = g; w < NW; w += G) {
    const int s0 = 32 * w, nst = min(32, p.S - s0);
    CL_MARK();
    // ---- the word's states -> bit slices (every CTA, all rows); seeds -> chg
    for (int x = warp; x < n; x += nwarps) {
      const uint64_t v = lane < nst ? __ldg(p.d_in + (size_t)(s0 + lane) * n + x) & __ldg(p.dommask + x) : 0ull;
      for (int a = 0; a < dmax; ++a) {
        const uint32_t b = __ballot_sync(0xffffffffu, (v >> a) & 1ull);
        if (lane == 0) X[x * dmax + a] = b;
      }
    }
    for (int x = tid; x < n; x += T) {
      chg[x] = 0u;
      chgn[x] = 0u;
    }
    if (tid < 32) {
      s_iters[tid] = 0;
      s_status[tid] = 0;
    }
    uint32_t active = nst >= 32 ? 0xffffffffu : ((1u << nst) - 1u);
    __syncthreads();
    {
      // a root state (no seed) tests every column in pass 1
      uint32_t rootl = 0;
      if (tid < nst) {
        const int sv = p.seed_var ? p.seed_var[s0 + tid] : -1;
        if (sv >= 0 && sv < n) atomicOr(&chg[sv], 1u << tid);
        else rootl = 1u << tid;
      }
      rootl = __reduce_or_sync(0xffffffffu, rootl);  // lanes 0..31 are warp 0
      if (warp == 0) sc[0] = (int)rootl;
      __syncthreads();
      const uint32_t roots = (uint32_t)sc[0];
      if (roots)
        for (int x = tid; x < n; x += T) chg[x] |= roots;
      __syncthreads();
    }
    // lanes whose every domain is non-empty at the start of the pass (an empty
    // one can only come from the input or, in full mode, from a wipeout)
    uint32_t allne0;
    {
      uint32_t ne_all = 0xffffffffu;
      for (int x = tid; x < n; x += T) {
        uint32_t ne = 0u;
        for (int a = 0; a < dmax; ++a) ne |= X[x * dmax + a];
        ne_all &= ne;
      }
      ne_all = __reduce_and_sync(0xffffffffu, ne_all);
      if (lane == 0) sc[warp] = (int)ne_all;
      __syncthreads();
      allne0 = 0xffffffffu;
      for (int w2 = 0; w2 < nwarps; ++w2) allne0 &= (uint32_t)sc[w2];
      __syncthreads();
    }
    int t = 0;
    CL_MARK();
    for (;;) {
      ++t;
      // ---- tested columns U = { y : chg[y] & active } (ascending, block scan)
      int cnt;
      {
        const int per = (n + T - 1) / T, b = min(n, tid * per), e = min(n, b + per);
        uint32_t c = 0;
        for (int i = b; i < e; ++i) c += (chg[i] & active) != 0u;
        uint32_t total;
        uint32_t pos = block_scan_u32(c, &total, sc);
        for (int i = b; i < e; ++i)
          if (chg[i] & active) list[pos++] = (uint16_t)i;
        cnt = (int)total;
      }
      __syncthreads();
      CL_MARK();
      // ---- per-column offsets (the list padded to a multiple of 8) and nibble tables
      const int cnt8 = (cnt + 7) & ~7;
      for (int c = tid; c < cnt8; c += T) {
        const int y = list[min(c, cnt - 1)];
        ci[c] = make_uint2((uint32_t)((size_t)y * p.col_stride), (uint32_t)(y * NQ * 64));  // {mask bytes, table bytes}
      }
      for (int i = tid; i < cnt * NQ; i += T) {
        const int c = i / NQ, q = i - c * NQ;
        const int y = list[c];
        uint32_t xb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) xb[j] = (4 * q + j < dmax) ? X[y * dmax + 4 * q + j] : 0u;
        uint32_t tv[16];
        tv[0] = 0u;
#pragma unroll
        for (int v = 1; v < 16; ++v) tv[v] = tv[v & (v - 1)] | xb[__ffs(v) - 1];
        uint4* dst = reinterpret_cast<uint4*>(Tb + ((size_t)y * NQ + q) * 16);
#pragma unroll
        for (int v = 0; v < 16; v += 4) dst[v >> 2] = make_uint4(tv[v], tv[v + 1], tv[v + 2], tv[v + 3]);
      }
      __syncthreads();
      CL_MARK();
      // ---- a3/a4: my rows against the tested columns, 32 states at a time
      uint32_t my_or = (~allne0 & active)
                                 ? sweep_rows<W, true>(p.M, p.P, p.pw, X, Tb, ci, cnt8, r0, r1, dmax, active, chgn)
                                 : sweep_rows<W, false>(p.M, p.P, p.pw, X, Tb, ci, cnt8, r0, r1, dmax, active, chgn);
      CL_MARK();
      // this CTA's partials: lanes that changed; lanes with every variable non-empty
      uint32_t my_ne = 0xffffffffu;
      __syncthreads();
      for (int x = x0 + tid; x < x1; x += T) {
        uint32_t ne = 0u;
        for (int a = 0; a < dmax; ++a) ne |= X[x * dmax + a];
        my_ne &= ne;
      }
      my_or = __reduce_or_sync(0xffffffffu, my_or);
      my_ne = __reduce_and_sync(0xffffffffu, my_ne);
      if (tid == 0) {
        s_part[0] = 0u;
        s_part[1] = 0xffffffffu;
      }
      __syncthreads();
      if (lane == 0) {
        if (my_or) atomicOr(&s_part[0], my_or);
        if (my_ne != 0xffffffffu) atomicAnd(&s_part[1], my_ne);
      }
      cluster.sync();  // [A] every CTA's rows, change masks and partials are final
      CL_MARK();
      // ---- exchange: change masks of every variable from its owner, the rows of
      // the variables that changed, and the partials
      uint32_t changed = 0u, allne = 0xffffffffu;
      for (int q = 0; q < C; ++q) {
        const uint32_t* rp = cluster.map_shared_rank(s_part, q);
        changed |= rp[0];
        allne &= rp[1];
      }
      for (int x = tid; x < n; x += T) {
        const int owner = min(C - 1, (x * dmax) / p.RPC);
        chg[x] = owner == k ? chgn[x] : *cluster.map_shared_rank(chgn + x, owner);
      }
      __syncthreads();
      for (int i = tid; i < n * dmax; i += T) {
        const int x = i / dmax;
        if (!chg[x]) continue;
        const int owner = min(C - 1, i / p.RPC);
        if (owner != k) X[i] = *cluster.map_shared_rank(X + i, owner);
      }
      cluster.sync();  // [B] nobody rewrites its rows / chgn before the others read them
      CL_MARK();
      for (int x = x0 + tid; x < x1; x += T) chgn[x] = 0u;
      // ---- per-state loop control (Alg. 1): wipeout first, then "changed"
      const uint32_t wipe = ~allne;
      const uint32_t stop_wipe = full ? 0u : (wipe & active);
      const uint32_t stop_conv = ~changed & active & ~stop_wipe;
      if (tid < 32) {
        const uint32_t bit = 1u << tid;
        if (active & bit) s_iters[tid] = t;
        if (stop_wipe & bit) s_status[tid] = 1;
        if (stop_conv & bit) s_status[tid] = (wipe & bit) ? 1 : 0;
      }
      active &= ~(stop_wipe | stop_conv);
      allne0 = allne;
      __syncthreads();
      if (active == 0u) break;
    }
    // ---- outputs: each CTA writes its own variables; rank 0 the counters
    for (int x = x0 + warp; x < x1; x += nwarps) {
      uint64_t v = 0;
      for (int a = 0; a < dmax; ++a) v |= (uint64_t)((X[x * dmax + a] >> lane) & 1u) << a;
      if (lane < nst) p.d_out[(size_t)(s0 + lane) * n + x] = v;
    }
    if (k == 0 && tid < nst) {
      p.iters[s0 + tid] = s_iters[tid];
      p.status[s0 + tid] = s_status[tid];
    }
    cluster.sync();  // the next word reuses every CTA's shared memory
    CL_MARK();
  }
#undef CL_MARK
}

size_t batch_cl_smem(int n, int dmax, int W) {
  const size_t rows4 = (((size_t)n * dmax) + 3) & ~(size_t)3;
  return rows4 * 4 + (size_t)n * (2 * W) * 16 * 4 + (size_t)n * 8 + (((size_t)n + 7) & ~(size_t)7) * 2 +
         ((size_t)n + 8) * 8;
}

cudaError_t launch_batch_cl(int W, const BatchCLParams& p, int clusters, int C, int threads, size_t smem,
                            cudaStream_t s) {
  const void* k = nullptr;
  switch (W) {
    case 1: k = (const void*)rac_batch_cl<1>; break;
    case 2: k = (const void*)rac_batch_cl<2>; break;
    case 4: k = (const void*)rac_batch_cl<4>; break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BatchCLParams pp = p;
  void* args[] = {&pp};
  return cudaLaunchKernelExC(&cfg, k, args);
}

// Largest number of co-resident clusters of C CTAs with `threads` threads.
cudaError_t batch_cl_max_clusters(int W, int C, int threads, size_t smem, int* out) {
  const void* k = W == 1 ? (const void*)rac_batch_cl<1> : W == 2 ? (const void*)rac_batch_cl<2>
                                                                   : (const void*)rac_batch_cl<4>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, k, &cfg);
}

}  // namespace rac
