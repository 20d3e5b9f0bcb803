// rac_kernels.cu -- the RAC support pass on sm_100a.
//
// One pass of the recurrence, Eq. 1, read in the
// intersection form of line 59:
//   D_t(x,a) = D_{t-1}(x,a) ∧ ∧_{c_xy ∈ C_x} [ c_xy|(x,a) ∩ D_{t-1}(y) ≠ ∅ ]
// For each live row (x,a) the kernel streams the packed masks M[x][a][·]
// (coalesced 128-bit loads), ANDs them with D_{t-1} held in shared memory and
// reduces "some mask & D == 0" across the lanes of the row with warp votes
// (early exit on the first failure).  Removed values are OR-ed into a removal
// bitvector R; D_t = D_{t-1} & ~R.  Loop control (Alg. 1 tensorAC, lines
// 198-210): wipeout checked first, then "nothing changed".
//
// Kernels:
//   rac_fused  -- whole enforcement in one cooperative launch: every CTA keeps
//                 D in smem across passes; a software grid barrier separates
//                 passes; every CTA derives the same stop decision from R.
//                 (single GPU; the host is not in the per-iteration path)
//   rac_pass   -- one pass over a row block; D_{t-1} staged into smem with a
//                 TMA bulk copy (cp.async.bulk + mbarrier).  Used by the
//                 row-sharded multi-GPU path (and virtual shards on one GPU)
//                 together with rac_shard_{init,slice,update,finalize}.
//   rac_batch  -- one CTA per domain state (batched mode).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

constexpr uint32_t kFull = 1u;  // RAC_FULL_FIXPOINT
constexpr int kOK = 0, kWIPEOUT = 1;

struct GroupIds {
  int gl;          // lane within the group
  unsigned gmask;  // lanes of this group within the warp
  long gidx;       // global group index
  long ngroups;    // total groups in the grid
};

template <int G>
__device__ __forceinline__ GroupIds group_ids() {
  GroupIds r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = lane / G;
  r.gl = lane % G;
  r.gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  const long per_cta = (long)(blockDim.x / 32) * (32 / G);
  r.gidx = (long)blockIdx.x * per_cta + warp * (32 / G) + gw;
  r.ngroups = (long)gridDim.x * per_cta;
  return r;
}

// Test the rows of variables [g.x_lo, g.x_hi) assigned to this group (static
// round-robin over (row, segment) items) and record removals into R.
// vl == nullptr: stream every vector of the row; else only the listed
// vectors (vl[0, vcnt), Prop. 2 incremental pass).
template <int W, int G>
__device__ __forceinline__ void support_sweep(const PassGeom& g, const uint4* Ds, unsigned long long* R,
                                              int32_t* removed_at, int t, long item0, long istep,
                                              const GroupIds& id, const uint16_t* vl, int vcnt) {
  const uint8_t* Db = reinterpret_cast<const uint8_t*>(Ds);
  const long rows = (long)(g.x_hi - g.x_lo) * g.dmax;
  const int n_seg = vl ? 1 : g.n_seg;
  const long n_items = rows * n_seg;
  const long row0 = (long)(g.x_lo - g.x_lo_alloc) * g.dmax;
  for (long it = item0; it < n_items; it += istep) {
    long r, s;
    if (n_seg == 1) { r = it; s = 0; } else { r = it / n_seg; s = it - r * n_seg; }
    const int xl = (int)(r / g.dmax);
    const int a = (int)(r - (long)xl * g.dmax);
    const int x = g.x_lo + xl;
    if (!((Db[x * W + (a >> 3)] >> (a & 7)) & 1u)) continue;  // dead row: (x,a) ∉ D_{t-1}
    const uint4* row = reinterpret_cast<const uint4*>(g.M + (size_t)(row0 + r) * g.row_stride);
    const uint32_t* Prow = g.P + (size_t)(x - g.x_lo_alloc) * g.pw;
    bool f;
    if (vl) {
      f = row_fails_list<W, G>(row, Ds, vl, 0, vcnt, id.gl, id.gmask, g.n, Prow);
    } else {
      const int vb = (int)s * g.seg_vecs;
      const int ve = min(vb + g.seg_vecs, g.nvec);
      f = row_fails<W, G>(row, Ds, vb, ve, id.gl, id.gmask, g.n, Prow);
    }
    if (f && id.gl == 0) {
      atomicOr(&R[x], 1ull << a);
      if (removed_at) removed_at[(size_t)x * 64 + a] = t;
    }
  }
}

template <int W>
__device__ __forceinline__ void stage_from_u64(uint4* Ds, const uint64_t* src, const uint64_t* dommask, int n,
                                               int nvec) {
  uint32_t* w = reinterpret_cast<uint32_t*>(Ds);
  for (int i = threadIdx.x; i < nvec * 4; i += blockDim.x) w[i] = 0xffffffffu;
  __syncthreads();
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  // 4 independent loads per thread in flight (the whole of D for n <= 2048)
  for (int x0 = threadIdx.x; x0 < n; x0 += 4 * blockDim.x) {
    uint64_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int x = x0 + k * blockDim.x;
      v[k] = x < n ? __ldg(src + x) & __ldg(dommask + x) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int x = x0 + k * blockDim.x;
      if (x < n) store_w<W>(Db + x * W, v[k]);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------- fused
template <int W, int G>
__global__ void __launch_bounds__(kThreads, 2) rac_fused(FusedParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ int scratch[kThreads / 32];
  const PassGeom& g = p.g;
  uint16_t* vlist = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(Ds) + list_offset(g.nvec));
  uint8_t* vneed = reinterpret_cast<uint8_t*>(Ds) + need_offset(g.nvec);
  for (int i = threadIdx.x; i < g.nvec; i += blockDim.x) vneed[i] = 0;
  stage_from_u64<W>(Ds, p.d_in, p.dommask, g.n, g.nvec);
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  const GroupIds id = group_ids<G>();
  const bool full = (p.flags & kFull) != 0;
  int t = 0, status = kOK, vcnt = g.nvec;
  unsigned epoch = 0;
  // Seeded call (Alg. 1 with @changed = seeds): pass 1 only re-tests the
  // vectors holding the seed variables.
  bool seeded = p.seeds != nullptr;
  if (seeded) {
    for (int i = threadIdx.x; i < p.n_seeds; i += blockDim.x) {
      const int y = p.seeds[i];
      if (y >= 0 && y < g.n) vneed[(y * W) >> 4] = 1;
    }
    __syncthreads();
    vcnt = block_compact(vneed, vlist, g.nvec, scratch);
  }
  if (seeded && vcnt == 0) {  // empty @changed: no pass (status from D_in)
    int wipe = 0;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) wipe |= load_w<W>(Db + x * W) == 0;
    wipe = __syncthreads_or(wipe);
    status = wipe ? kWIPEOUT : kOK;
  } else for (;;) {
    ++t;
    unsigned long long* Rc = p.R + (size_t)(t % 3) * g.n;
    unsigned long long* Rn = p.R + (size_t)((t + 1) % 3) * g.n;
    // R of pass t+1 was last read before the previous barrier: clear it now.
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) Rn[i] = 0ull;
    // pass 1 (and any pass where many variables changed) streams whole rows;
    // otherwise only the vectors of variables changed in the previous pass.
    const bool use_list = (t > 1 || seeded) && 2 * vcnt <= g.nvec && g.nvec <= 65535;
    support_sweep<W, G>(g, Ds, Rc, p.removed_at, t, id.gidx, id.ngroups, id, use_list ? vlist : nullptr, vcnt);
    grid_sync(p.bar, gridDim.x, ++epoch);
    // D_t = D_{t-1} & ~R (every CTA, redundantly); flags for Alg. 1's checks.
    int changed = 0, wipe = 0;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) {
      const uint64_t r = __ldcg(&Rc[x]);
      const uint64_t dv = load_w<W>(Db + x * W);
      const uint64_t nd = dv & ~r;
      store_w<W>(Db + x * W, nd);
      const bool chx = (dv & r) != 0;
      changed |= chx;
      wipe |= nd == 0;
      if (chx) vneed[(x * W) >> 4] = 1;
    }
    changed = __syncthreads_or(changed);
    wipe = __syncthreads_or(wipe);
    vcnt = block_compact(vneed, vlist, g.nvec, scratch);
    if (wipe && !full) { status = kWIPEOUT; break; }          // Alg. 1
    if (!changed) { status = wipe ? kWIPEOUT : kOK; break; }  // Prop. 1 end condition
  }
  if (blockIdx.x == 0) {
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) p.d_out[x] = load_w<W>(Db + x * W);
    if (threadIdx.x == 0) { *p.iters = t; *p.status = status; }
  }
  // The last CTA out resets the barrier words and clears R[1] (the removal
  // buffer pass 1 of the next launch writes): every other CTA has finished
  // reading by the time it counts itself out.
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = gridDim.x == 1 ? 1 : (atomicAdd(&p.bar[2], 1u) + 1u == gridDim.x);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) p.R[(size_t)g.n + x] = 0ull;
    if (threadIdx.x == 0 && gridDim.x > 1) {
      p.bar[0] = 0u;
      p.bar[1] = 0u;
      p.bar[2] = 0u;
    }
    __threadfence();
  }
}

// ---------------------------------------------------------------------------- per-pass (sharded)
__device__ __forceinline__ void tma_stage(uint4* dst, const uint8_t* src, uint32_t bytes, uint64_t* mbar) {
  // One elected thread arms the mbarrier with the byte count and issues bulk
  // copies (<= 32 KB each); every thread waits on phase 0.
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      uint32_t sz = min(32768u, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d0 + off),
          "l"(src + off), "r"(sz), "r"(mb)
          : "memory");
    }
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb)
        : "memory");
  }
}

template <int W, int G>
__global__ void __launch_bounds__(kThreads, 2) rac_pass(PassParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ alignas(8) uint64_t mbar;
  if (*reinterpret_cast<volatile int32_t*>(p.s.done)) return;  // converged: speculative pass is a no-op
  tma_stage(Ds, p.s.Dw, (uint32_t)p.g.row_stride, &mbar);
  const int t = *p.s.iters + 1;
  const int vcnt = *p.s.vcnt;
  const bool use_list = t > 1 && 2 * vcnt <= p.g.nvec && p.g.nvec <= 65535;
  uint16_t* vlist = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(Ds) + list_offset(p.g.nvec));
  if (use_list) {
    for (int i = threadIdx.x; i < vcnt; i += blockDim.x) vlist[i] = p.s.vlist[i];
    __syncthreads();
  }
  const GroupIds id = group_ids<G>();
  support_sweep<W, G>(p.g, Ds, p.s.R, p.removed_at, t, id.gidx, id.ngroups, id, use_list ? vlist : nullptr, vcnt);
}

__global__ void rac_shard_init(ShardState s, const uint64_t* d_in, const uint64_t* dommask, int n, int W,
                               int row_stride, int total_g) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total_g; i += gridDim.x * blockDim.x) {
    if (i < n) {
      const uint64_t v = d_in[i] & dommask[i];
      s.Dcur[i] = v;
      s.R[i] = 0ull;
      for (int k = 0; k < W; ++k) s.Dw[(size_t)i * W + k] = (uint8_t)(v >> (8 * k));
    }
    s.Dg[i] = 0ull;
  }
  for (int b = n * W + blockIdx.x * blockDim.x + threadIdx.x; b < row_stride; b += gridDim.x * blockDim.x)
    s.Dw[b] = 0xffu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *s.iters = 0;
    *s.status = -1;
    *s.done = 0;
    *s.vcnt = 0;
  }
}

// D_{t}[x] = D_{t-1}[x] & ~R[x] for the local block, written into the
// all-gather buffer; R is cleared for the next pass.
__global__ void rac_shard_slice(ShardState s, int x_lo, int x_hi, int n) {
  if (*reinterpret_cast<volatile int32_t*>(s.done)) return;
  for (int x = x_lo + blockIdx.x * blockDim.x + threadIdx.x; x < x_hi; x += gridDim.x * blockDim.x) {
    if (x < n) {
      s.Dg[x] = s.Dcur[x] & ~s.R[x];
      s.R[x] = 0ull;
    } else {
      s.Dg[x] = 0ull;
    }
  }
}

// After the exchange: every rank derives the same flags from the gathered
// vector (changed = D_t != D_{t-1}, wipe = some D_t(x) empty), the list of
// vectors holding changed variables (Prop. 2 incremental next pass), and
// advances.  One CTA; dynamic smem = nvec flag bytes.
__global__ void __launch_bounds__(1024) rac_shard_update(ShardState s, int n, int W, int nvec, uint32_t flags) {
  extern __shared__ uint8_t need[];
  __shared__ int scratch[32];
  if (*reinterpret_cast<volatile int32_t*>(s.done)) return;
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) need[i] = 0;
  __syncthreads();
  int changed = 0, wipe = 0;
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    const uint64_t nv = s.Dg[x];
    const bool chx = nv != s.Dcur[x];
    changed |= chx;
    wipe |= nv == 0;
    if (chx) need[(x * W) >> 4] = 1;
    s.Dcur[x] = nv;
    for (int k = 0; k < W; ++k) s.Dw[(size_t)x * W + k] = (uint8_t)(nv >> (8 * k));
  }
  changed = __syncthreads_or(changed);
  wipe = __syncthreads_or(wipe);
  const int cnt = nvec <= 65535 ? block_compact(need, s.vlist, nvec, scratch) : nvec;
  if (threadIdx.x == 0) {
    *s.vcnt = cnt;
    *s.iters += 1;
    if (wipe && !(flags & kFull)) {
      *s.status = kWIPEOUT;
      *s.done = 1;
    } else if (!changed) {
      *s.status = wipe ? kWIPEOUT : kOK;
      *s.done = 1;
    }
  }
}

__global__ void rac_shard_finalize(ShardState s, int n, uint64_t* d_out, int32_t* iters, int32_t* status) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) d_out[x] = s.Dcur[x];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *iters = *s.iters;
    *status = *s.status;
  }
}

// ---------------------------------------------------------------------------- batched
// One CTA per state: D and R live in smem, __syncthreads is the pass barrier,
// each state stops at its own pass (freeze-on-stop).  The relation rows are
// shared by all states and stay L2-resident.
template <int W, int G>
__global__ void __launch_bounds__(kThreads, 2) rac_batch(BatchParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ int scratch[kThreads / 32];
  const PassGeom& g = p.g;
  const int s = blockIdx.x;
  uint16_t* vlist = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(Ds) + list_offset(g.nvec));
  uint8_t* vneed = reinterpret_cast<uint8_t*>(Ds) + need_offset(g.nvec);
  unsigned long long* R = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(Ds) + fused_smem(g.nvec));
  for (int i = threadIdx.x; i < g.nvec; i += blockDim.x) vneed[i] = 0;
  stage_from_u64<W>(Ds, p.d_in + (size_t)s * g.n, p.dommask, g.n, g.nvec);
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gw = lane / G;
  GroupIds id;
  id.gl = lane % G;
  id.gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
  id.gidx = warp * (32 / G) + gw;
  id.ngroups = (long)(blockDim.x / 32) * (32 / G);
  const bool full = (p.flags & kFull) != 0;
  int t = 0, status = kOK, vcnt = g.nvec;
  const int seed = p.seed_var ? p.seed_var[s] : -1;
  const bool seeded = seed >= 0 && seed < g.n;
  if (seeded) {
    if (threadIdx.x == 0) vneed[(seed * W) >> 4] = 1;
    __syncthreads();
    vcnt = block_compact(vneed, vlist, g.nvec, scratch);
  }
  for (;;) {
    ++t;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) R[x] = 0ull;
    __syncthreads();
    const bool use_list = (t > 1 || seeded) && 2 * vcnt <= g.nvec && g.nvec <= 65535;
    {
      const long rows = (long)g.n * g.dmax;
      for (long r = id.gidx; r < rows; r += id.ngroups) {
        const int x = (int)(r / g.dmax), a = (int)(r - (long)x * g.dmax);
        if (!((Db[x * W + (a >> 3)] >> (a & 7)) & 1u)) continue;
        const uint4* row = reinterpret_cast<const uint4*>(g.M + (size_t)r * g.row_stride);
        const uint32_t* Prow = g.P + (size_t)x * g.pw;
        const bool f = use_list ? row_fails_list<W, G>(row, Ds, vlist, 0, vcnt, id.gl, id.gmask, g.n, Prow)
                                : row_fails<W, G>(row, Ds, 0, g.nvec, id.gl, id.gmask, g.n, Prow);
        if (f && id.gl == 0) atomicOr(&R[x], 1ull << a);  // shared-memory u64 atomic
      }
    }
    __syncthreads();
    int changed = 0, wipe = 0;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) {
      const uint64_t r = R[x];
      const uint64_t dv = load_w<W>(Db + x * W);
      const uint64_t nd = dv & ~r;
      store_w<W>(Db + x * W, nd);
      const bool chx = (dv & r) != 0;
      changed |= chx;
      wipe |= nd == 0;
      if (chx) vneed[(x * W) >> 4] = 1;
    }
    changed = __syncthreads_or(changed);
    wipe = __syncthreads_or(wipe);
    vcnt = block_compact(vneed, vlist, g.nvec, scratch);
    if (wipe && !full) { status = kWIPEOUT; break; }
    if (!changed) { status = wipe ? kWIPEOUT : kOK; break; }
  }
  for (int x = threadIdx.x; x < g.n; x += blockDim.x) p.d_out[(size_t)s * g.n + x] = load_w<W>(Db + x * W);
  if (threadIdx.x == 0) {
    p.iters[s] = t;
    p.status[s] = status;
  }
}

template <template <int, int> class F, typename... A>
cudaError_t dispatch(int W, int G, A&&... a) {
#define RAC_CASE_G(WW)                                        \
  switch (G) {                                                \
    case 1: return F<WW, 1>::run(a...);                       \
    case 2: return F<WW, 2>::run(a...);                       \
    case 4: return F<WW, 4>::run(a...);                       \
    case 8: return F<WW, 8>::run(a...);                       \
    case 16: return F<WW, 16>::run(a...);                     \
    case 32: return F<WW, 32>::run(a...);                     \
    default: return cudaErrorInvalidValue;                    \
  }
  switch (W) {
    case 1: RAC_CASE_G(1)
    case 2: RAC_CASE_G(2)
    case 4: RAC_CASE_G(4)
    case 8: RAC_CASE_G(8)
    default: return cudaErrorInvalidValue;
  }
#undef RAC_CASE_G
}

template <int W, int G>
struct FusedLaunch {
  static cudaError_t run(const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool coop) {
    auto k = rac_fused<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (coop) {
      FusedParams pp = p;
      void* args[] = {&pp};
      return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kThreads), args, smem, s);
    }
    k<<<grid, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
};

template <int W, int G>
struct FusedOcc {
  static cudaError_t run(size_t smem, int* out) {
    auto k = rac_fused<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kThreads, smem);
  }
};

template <int W, int G>
struct PassLaunch {
  static cudaError_t run(const PassParams& p, int grid, size_t smem, cudaStream_t s) {
    auto k = rac_pass<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
};

template <int W, int G>
struct PassOcc {
  static cudaError_t run(size_t smem, int* out) {
    auto k = rac_pass<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kThreads, smem);
  }
};

template <int W, int G>
struct BatchLaunch {
  static cudaError_t run(const BatchParams& p, int n_states, size_t smem, cudaStream_t s) {
    auto k = rac_batch<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<n_states, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
};

template <int W, int G>
struct BatchOcc {
  static cudaError_t run(size_t smem, int* out) {
    auto k = rac_batch<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kThreads, smem);
  }
};

}  // namespace

int choose_group(int nvec) {
  // smallest power of two G with G * kUnroll >= nvec, capped at a warp
  int G = 1;
  while (G < 32 && G * kUnroll < nvec) G *= 2;
  return G;
}

cudaError_t launch_fused(int W, int G, const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool coop) {
  return dispatch<FusedLaunch>(W, G, p, grid, smem, s, coop);
}
cudaError_t fused_occupancy(int W, int G, size_t smem, int* out) { return dispatch<FusedOcc>(W, G, smem, out); }
cudaError_t launch_pass(int W, int G, const PassParams& p, int grid, size_t smem, cudaStream_t s) {
  return dispatch<PassLaunch>(W, G, p, grid, smem, s);
}
cudaError_t pass_occupancy(int W, int G, size_t smem, int* out) { return dispatch<PassOcc>(W, G, smem, out); }
cudaError_t launch_batch(int W, int G, const BatchParams& p, int n_states, size_t smem, cudaStream_t s) {
  return dispatch<BatchLaunch>(W, G, p, n_states, smem, s);
}
cudaError_t batch_occupancy(int W, int G, size_t smem, int* out) { return dispatch<BatchOcc>(W, G, smem, out); }

cudaError_t launch_shard_init(const ShardState& s, const uint64_t* d_in, const uint64_t* dommask, int n, int W,
                              size_t row_stride, int total_g, cudaStream_t st) {
  int work = total_g > (int)row_stride ? total_g : (int)row_stride;
  int grid = (work + 255) / 256;
  if (grid > 1024) grid = 1024;
  rac_shard_init<<<grid, 256, 0, st>>>(s, d_in, dommask, n, W, (int)row_stride, total_g);
  return cudaGetLastError();
}
cudaError_t launch_shard_slice(const ShardState& s, int x_lo, int x_hi, int n, cudaStream_t st) {
  int cnt = x_hi - x_lo;
  int grid = (cnt + 255) / 256;
  if (grid < 1) grid = 1;
  rac_shard_slice<<<grid, 256, 0, st>>>(s, x_lo, x_hi, n);
  return cudaGetLastError();
}
cudaError_t launch_shard_update(const ShardState& s, int n, int W, int nvec, uint32_t flags, cudaStream_t st) {
  if (nvec > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rac_shard_update, cudaFuncAttributeMaxDynamicSharedMemorySize, nvec);
    if (e != cudaSuccess) return e;
  }
  rac_shard_update<<<1, 1024, nvec, st>>>(s, n, W, nvec, flags);
  return cudaGetLastError();
}
cudaError_t launch_shard_finalize(const ShardState& s, int n, uint64_t* d_out, int32_t* iters, int32_t* status,
                                  cudaStream_t st) {
  int grid = (n + 255) / 256;
  if (grid > 256) grid = 256;
  rac_shard_finalize<<<grid, 256, 0, st>>>(s, n, d_out, iters, status);
  return cudaGetLastError();
}

}  // namespace rac
