// rac_kernels.cu -- the RAC support pass on sm_100a.
//
// One pass of the recurrence, Eq. 1, read in the
// intersection form of line 59:
//   D_t(x,a) = D_{t-1}(x,a) ∧ ∧_{c_xy ∈ C_x} [ c_xy|(x,a) ∩ D_{t-1}(y) ≠ ∅ ]
// evaluated column by column: for every tested column y (all y in a full
// pass; the variables changed in the previous pass otherwise -- Alg. 1's
// Cons[:, @changed], justified by Prop. 2)
// a warp streams 512 contiguous bytes of column y (16 bytes = 16/W masks per
// lane, 128-bit loads, kUnroll columns in flight per lane), ANDs each mask
// with D_{t-1}(y) held in shared memory and ORs "mask & D == 0" into a
// per-lane failure set; a lane stops as soon as all its live rows failed;
// dead rows are skipped.  Failing rows are OR-ed into a removal bitvector R
// (the only atomics; rare), and D_t = D_{t-1} & ~R.  Loop control (Alg. 1
// tensorAC, lines 198-210): wipeout checked first, then "nothing changed".
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
//   rac_batch  -- one CTA per domain state, removal bits in smem and
//                 __syncthreads as the pass barrier: the single-CTA enforcement
//                 of small instances (one state) and the per-state batched
//                 design kept for comparison (the default batched path is the
//                 bit-sliced rac_batch_bs).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

constexpr uint32_t kFull = 1u;  // RAC_FULL_FIXPOINT
constexpr int kOK = 0, kWIPEOUT = 1;
constexpr int kPeerTimeout = -7;  // RAC_EPEER

// OR removal bits into R[x]; with a change list `cl` ([0] = count, then the
// variables), the first removal of x in the pass appends x -- after the grid
// barrier only the listed words need to be read (and they are the next pass's
// tested columns, Alg. 1's @changed).
__device__ __forceinline__ void mark_removed(unsigned long long* R, int x, unsigned long long bits, uint32_t* cl) {
  if (cl == nullptr) {
    atomicOr(&R[x], bits);  // fire-and-forget reduction
    return;
  }
  const unsigned long long old = atomicOr(&R[x], bits);
  if (old == 0ull) cl[1 + atomicAdd(cl, 1u)] = (uint32_t)x;
}

// Work-item iterator of a warp: the first ~7/8 of the items are assigned
// round robin, the rest are claimed one at a time from a per-pass counter
// (the next claim in flight while the current item streams), so SMs that
// drain HBM faster take more of the tail.  Without a counter: plain round
// robin.  (Measured on the 4 KB items of the column and sparse sweeps: one
// same-address atomic per item costs more than the imbalance it removes --
// C3 W-stream 88.7 -> 92.1 us -- so those sweeps run round robin.  Claims of
// 4..16 items per atomic were no better (profiles/r02f/ab_claim.log, c3-prop
// 288 -> 344..575 us), and the generalised iterator alone slowed the static
// column sweep 88 -> 112 us on the same box (profiles/r02g): removed.)
#ifndef RAC_CLAIM_DIV
#define RAC_CLAIM_DIV 8
#endif
constexpr uint32_t kClaimDiv = RAC_CLAIM_DIV;  // 1/kClaimDiv of the items are claimed dynamically
#ifndef RAC_ROW_CLAIM_DIV
#define RAC_ROW_CLAIM_DIV 4  // r02av: C3 W-seed 124.0 (1/8) -> 119.3 us (1/4); 1/2 and 1/16: 129 us
#endif
constexpr int kRowClaimDiv = RAC_ROW_CLAIM_DIV;  // row sweep: 1/kRowClaimDiv of the rows are claimed
#ifndef RAC_COL_CLAIM
#define RAC_COL_CLAIM 0
#endif
struct ItemIter {
  uint32_t items, nw, per, S, k, pending;
  unsigned* wctr;
  int lane;
  uint32_t warp0;
  __device__ __forceinline__ ItemIter(uint32_t items_, long warp0_, long nwarps_, unsigned* wctr_)
      : items(items_), nw((uint32_t)nwarps_), k(0), pending(0), wctr(wctr_), lane(threadIdx.x & 31),
        warp0((uint32_t)warp0_) {
    per = wctr ? (items - items / kClaimDiv) / nw : (items + nw - 1) / nw;
    S = wctr ? per * nw : items;
    if (wctr && per == 0) pending = claim();
  }
  __device__ __forceinline__ uint32_t claim() {
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(wctr, 1u);
    return S + __shfl_sync(0xffffffffu, b, 0);
  }
  // next item of this warp (warp-uniform); false when done
  __device__ __forceinline__ bool next(uint32_t& it) {
    for (;;) {
      if (k < per) {
        it = warp0 + k * nw;
        if (++k == per && wctr) pending = claim();
        if (it < items) return true;
      } else if (wctr) {
        it = pending;
        if (it >= items) return false;
        pending = claim();
        return true;
      } else {
        return false;
      }
    }
  }
};

// (Measured, profiles/r02ag, same box: C3 W-stream 110.4 -> 107.5-108.4 us, but
// C2 14.3 -> 16.1 us, C3 W-prop 275 -> 280 us and C4 W-stream 5.7 -> 6.7 ms: off.)
// Partitioned tail claims (RAC_COL_CLAIM == 2, A/B): the last 1/kClaimDiv of a
// pass's items is split into kClaimParts contiguous partitions, each with its
// own counter on its own 128-byte line (ctr[j * 32]); a warp claims only from
// partition warp0 % kClaimParts (every partition has ~nwarps/kClaimParts warps,
// so each is drained by its own warps; walking the other partitions to detect
// the end cost one atomic round trip per partition -- c2 14 -> 30 us,
// profiles/r02af).  One same-address counter for every warp serialised the
// tail (profiles/r02f).  Lane 0 claims; returns the item or ~0u.
#ifndef RAC_CLAIM_PARTS
#define RAC_CLAIM_PARTS 32
#endif
constexpr uint32_t kClaimParts = RAC_CLAIM_PARTS;
#if RAC_COL_CLAIM == 2
struct TailClaim {
  uint32_t b, e;
  unsigned* ctr;
  __device__ __forceinline__ TailClaim(uint32_t S, uint32_t items, uint32_t warp0, unsigned* ctr_) {
    const uint32_t L = (items - S + kClaimParts - 1) / kClaimParts, j = warp0 % kClaimParts;
    b = S + j * L;
    e = min(items, b + L);
    ctr = ctr_ + j * 32;
  }
  __device__ __forceinline__ uint32_t claim() {
    uint32_t r = ~0u;
    if ((threadIdx.x & 31) == 0 && b < e) {
      const uint32_t i = atomicAdd(ctr, 1u);
      if (b + i < e) r = b + i;
    }
    return __shfl_sync(0xffffffffu, r, 0);
  }
};
#endif

// Column sweep: test the rows of variables [g.x_lo, g.x_hi) against the
// columns cols[0, ncol) (cols == nullptr: columns 0..ncol-1) and OR removals
// into R.  Work item = (tested column y, chunk of 32 x kUnrollC consecutive
// 16-byte vectors of column y's rows); the columns all have the same rows, so
// item -> (column, chunk) is one division.  Per item D(y) is read once; each
// lane streams kUnrollC vectors (16/W rows each) and tests them with a
// zero-lane check; only a vector with a zero lane (rare) works out which of
// its rows are live and declared-unsupported and ORs them into R.  Dead rows
// are not skipped here: the per-pass layout choice (pick_rows) sends passes
// with few live rows to the row-major sweep, which skips them.
template <int W>
__device__ __noinline__ void column_sweep(const PassGeom& g, const uint8_t* Db, unsigned long long* R,
                                          int32_t* removed_at, int t, long warp0, long nwarps,
                                          const uint16_t* cols, int ncol, unsigned* rflag = nullptr,
                                          unsigned* wctr = nullptr, uint32_t* cl = nullptr,
                                          const EpochMirror* em = nullptr, unsigned* cctr = nullptr) {
  constexpr int RPL = 16 / W, U = kUnroll;
  const int lane = threadIdx.x & 31;
  const int r_lo = (g.x_lo - g.x_lo_alloc) * g.dmax;
  const int r_hi = (g.x_hi - g.x_lo_alloc) * g.dmax;
  if (r_hi <= r_lo || ncol <= 0) return;
  const uint32_t v_lo = (uint32_t)r_lo / RPL, v_hi = ((uint32_t)r_hi + RPL - 1) / RPL;
  // vectors per lane per item: U, fewer when the pass is too small to give
  // every warp an item (latency-bound passes spread over more warps)
  const uint64_t tot = (uint64_t)(v_hi - v_lo) * (uint32_t)ncol;
  const uint64_t upl64 = tot / (32ull * (uint64_t)nwarps);
  const uint32_t upl = upl64 < 1ull ? 1u : (upl64 > (uint64_t)U ? (uint32_t)U : (uint32_t)upl64);
  const uint32_t ipc = (v_hi - v_lo + 32u * upl - 1u) / (32u * upl);  // items per column
  const uint32_t items = ipc * (uint32_t)ncol;
  bool flagged = false;  // this warp has raised the pass's removal flag
#if RAC_COL_CLAIM == 2
  // static round robin for the first items, then partitioned claims (cctr)
  const uint32_t per = cctr ? (items - items / kClaimDiv) / (uint32_t)nwarps
                            : (items + (uint32_t)nwarps - 1) / (uint32_t)nwarps;
  const uint32_t Sst = cctr ? per * (uint32_t)nwarps : items;
  TailClaim tc(Sst, items, (uint32_t)warp0, cctr);
  uint32_t kk = 0, pend = (cctr && per == 0) ? tc.claim() : ~0u;
  for (;;) {
    uint32_t it;
    if (kk < per) {
      it = (uint32_t)warp0 + kk * (uint32_t)nwarps;
      if (++kk == per && cctr) pend = tc.claim();
      if (it >= Sst) continue;
    } else if (cctr) {
      if (pend == ~0u) break;
      it = pend;
      pend = tc.claim();
    } else {
      break;
    }
#else
  ItemIter iter(items, warp0, nwarps, wctr);
  for (uint32_t it; iter.next(it);) {
#endif
    const uint32_t c = it / ipc, chunk = it - c * ipc;
    const int y = cols ? (int)cols[c] : (int)c;
    const uint4* col = reinterpret_cast<const uint4*>(g.M + (size_t)y * g.col_stride);
    const uint32_t v0 = v_lo + chunk * 32u * upl + (uint32_t)lane;
    const uint32_t ve = min(v_hi, v0 - (uint32_t)lane + 32u * upl);
    uint4 m[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 32u < ve) m[u] = ldg_stream(col + v0 + u * 32u);
    const uint64_t dv = load_w<W>(Db + y * W);
    const uint4 rd = rep16<W>(dv);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * 32u;
      // failing live rows of this lane's vector, as (variable, value bits): the
      // RPL rows of a vector span two variables at most when dmax >= RPL
      int x1 = -1, x2 = -1;
      unsigned long long b1 = 0ull, b2 = 0ull;
      if (v < ve) {
        const uint4 tv = and4(m[u], rd);
        if (vec_any_zero<W>(tv)) {  // rare: some row of this vector may lose its support
          const uint32_t z = zero_lanes<W>(tv);
          for (uint32_t zz = z; zz; zz &= zz - 1u) {
            const int r = (int)v * RPL + __ffs(zz) - 1;
            if (r < r_lo || r >= r_hi) continue;
            const int xl = r / g.dmax, a = r - xl * g.dmax;
            const int x = g.x_lo_alloc + xl;
            if (!((Db[x * W + (a >> 3)] >> (a & 7)) & 1u)) continue;  // (x,a) not live
            if (dv == 0ull && !((g.P[(size_t)xl * g.pw + (y >> 5)] >> (y & 31)) & 1u)) continue;  // R2
            if (x1 < 0 || x1 == x) { x1 = x; b1 |= 1ull << a; }
            else if (x2 < 0 || x2 == x) { x2 = x; b2 |= 1ull << a; }
            else mark_removed(R, x, 1ull << a, cl);  // a third variable (dmax < RPL): direct
            if (removed_at) put_epoch(removed_at, em, (size_t)x * 64 + a, t);
          }
        }
      }
      // one atomic per (lane, variable) instead of per row; the removal flag is
      // a plain store (same-address atomics from every failing lane serialised the
      // tail of removal-heavy passes, r02ar; a warp-wide merge of the atomics cost
      // more in the stream than it saved, r02as)
      if (x1 >= 0) {
        mark_removed(R, x1, b1, cl);
        if (x2 >= 0) mark_removed(R, x2, b2, cl);
        if (rflag && !flagged) {
          *reinterpret_cast<volatile unsigned*>(rflag) = 1u;
          flagged = true;
        }
      }
    }
  }
}

// Sparse arc-block sweep (NEXT-3).  Work item = (tested column y, chunk of
// 32 x kUnrollS consecutive 16-byte vectors of column y's blocks); ipref[i] =
// items before the i-th tested column (all columns in a full pass, the listed
// ones otherwise).  Per item: one binary search in shared memory, D(y) read
// once; each lane streams kUnrollS vectors and tests them against D(y) with a
// zero-lane check.  Only a vector with some zero lane (rare) looks up its arc
// (x, y) and the live rows of x, and ORs real failures into R[x].  Only
// declared arcs are stored, so no presence check is needed (reading R2).
template <int W>
__device__ __forceinline__ void sparse_sweep(const PassGeom& g, const uint8_t* Db, unsigned long long* R,
                                             int32_t* removed_at, int t, long warp0, long nwarps,
                                             const uint16_t* cols, int ncol, const uint32_t* ipref,
                                             uint32_t upl, unsigned* rflag, unsigned* wctr, uint32_t* cl) {
  constexpr int L = 16 / W, U = kUnrollS;
  constexpr uint32_t LM = (L == 32) ? 0xffffffffu : ((1u << L) - 1u);
  const int lane = threadIdx.x & 31;
  const uint32_t VB = (uint32_t)g.s_vb;
  const uint32_t items = ipref[ncol];
  const uint4* S4 = reinterpret_cast<const uint4*>(g.S);
  int ci = 0;
  bool flagged = false;
  ItemIter iter(items, warp0, nwarps, wctr);
  for (uint32_t it; iter.next(it);) {
    int hi = ncol - 1;  // last i with ipref[i] <= it (items increase: search from the previous ci)
    while (ci < hi) {
      const int mid = (ci + hi + 1) >> 1;
      if (ipref[mid] <= it) ci = mid; else hi = mid - 1;
    }
    const int y = cols ? (int)cols[ci] : ci;
    const uint32_t b0 = __ldg(g.s_off + y);
    const uint32_t nv = (__ldg(g.s_off + y + 1) - b0) * VB;
    const uint32_t v0 = (it - ipref[ci]) * 32u * upl + (uint32_t)lane;
    const uint32_t ve = min(nv, v0 - (uint32_t)lane + 32u * upl);
    const uint4* col = S4 + (size_t)b0 * VB;
    uint4 m[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * 32u < ve) m[u] = ldg_stream(col + v0 + u * 32u);
    const uint4 dy = rep16<W>(load_w<W>(Db + y * W));
    uint32_t any = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = v0 + u * 32u;
      if (v < ve) {
        const uint4 tv = and4(m[u], dy);
        if (vec_any_zero<W>(tv)) {  // rare: some row of this vector may lose its support
          const uint32_t k = v / VB, pp = v - k * VB;
          const int x = (int)(__ldg(g.s_arc + b0 + k) & 0xffffu);
          const int a0 = (int)pp * L;
          const uint32_t cand = (uint32_t)(load_w<W>(Db + x * W) >> a0) & LM;
          const uint32_t f = zero_lanes<W>(tv) & cand;
          if (f) {
            any = 1;
            mark_removed(R, x, (unsigned long long)f << a0, cl);
            if (removed_at)
              for (uint32_t ff = f; ff; ff &= ff - 1u) removed_at[(size_t)x * 64 + a0 + __ffs(ff) - 1] = t;
          }
        }
      }
    }
    // this pass removed something: a plain store, once per lane and sweep
    if (any && rflag && !flagged) {
      *reinterpret_cast<volatile unsigned*>(rflag) = 1u;
      flagged = true;
    }
  }
}

// Row-major sweep: every live row (x,a) of variables [g.x_lo, g.x_hi) is
// streamed whole (all n columns) by a group of G lanes, with early exit on
// the first failing column and dead-row skip.  Rows are split into n_seg
// segments so that every group gets several items.
template <int W, int G>
__device__ __noinline__ void row_sweep(const PassGeom& g, const uint4* Ds, unsigned long long* R,
                                          int32_t* removed_at, int t, long gidx, long ngroups,
                                          unsigned* wctr = nullptr, unsigned* rflag = nullptr,
                                          uint32_t* cl = nullptr, const EpochMirror* em = nullptr,
                                          unsigned long long* Rs = nullptr) {
  const uint8_t* Db = reinterpret_cast<const uint8_t*>(Ds);
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));
  const int nvec = g.dbytes / 16;
  const int rows = (g.x_hi - g.x_lo) * g.dmax;
  const int row0 = (g.x_lo - g.x_lo_alloc) * g.dmax;
  const int ng = (int)ngroups;
  int n_seg = 1;
  while ((long)rows * n_seg < 8L * ng && (nvec + 2 * n_seg - 1) / (2 * n_seg) >= G * kUnrollR) n_seg *= 2;
  const int seg = ((nvec + n_seg - 1) / n_seg + G * kUnrollR - 1) / (G * kUnrollR) * (G * kUnrollR);
  n_seg = (nvec + seg - 1) / seg;
  const int items = rows * n_seg;
  // Work items: static round robin; with wctr the first ~7/8 are static and the
  // rest are claimed one item per group (a warp claims for its groups, the next
  // claim in flight while the current item streams), so SMs that drain HBM
  // faster take more of the tail and the pass ends within about one row.
  const int gpw = 32 / G, gw = lane / G;
  bool flagged = false;
  auto process = [&](int it) {
    int r = it, sgi = 0;
    if (n_seg > 1) { r = it / n_seg; sgi = it - r * n_seg; }
    const int xl = r / g.dmax, a = r - xl * g.dmax;
    const int x = g.x_lo + xl;
    if (!((Db[x * W + (a >> 3)] >> (a & 7)) & 1u)) return;  // dead row: (x,a) ∉ D_{t-1}
    const uint4* row = reinterpret_cast<const uint4*>(g.Mr + (size_t)(row0 + r) * g.dbytes);
    const uint32_t* Prow = g.P + (size_t)(x - g.x_lo_alloc) * g.pw;
    const int vb = sgi * seg, ve = min(vb + seg, nvec);
    if (row_fails<W, G>(row, Ds, vb, ve, gl, gmask, g.n, Prow) && gl == 0) {
      if (Rs) atomicOr(reinterpret_cast<unsigned*>(&Rs[x]) + (a >> 5), 1u << (a & 31));  // shared (native)
      else mark_removed(R, x, 1ull << a, cl);
      if (rflag && !flagged) {  // this pass removed something: a plain store, once per group and sweep
        *reinterpret_cast<volatile unsigned*>(rflag) = 1u;
        flagged = true;
      }
      if (removed_at) put_epoch(removed_at, em, (size_t)x * 64 + a, t);
    }
  };
  const int per = wctr ? (items - items / kRowClaimDiv) / ng : (items + ng - 1) / ng;
  const int S = wctr ? per * ng : items;
  auto claim = [&]() {
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(wctr, (unsigned)gpw);
    return S + (int)__shfl_sync(0xffffffffu, b, 0) + gw;
  };
  int k = 0, pending = (wctr && per == 0) ? claim() : 0;
  for (;;) {  // one loop body (one copy of the row test): static items, then claims
    int it;
    if (k < per) {
      it = (int)gidx + k * ng;
      if (++k == per && wctr) pending = claim();  // first claim in flight during the last static item
    } else if (wctr) {
      it = pending;
      if (__all_sync(0xffffffffu, it >= items)) break;  // warp-uniform exit
      pending = claim();
    } else {
      break;
    }
    if (it < items) process(it);
  }
  if (Rs) {
    // one atomic per (CTA, variable): the rows of a variable sit in neighbouring
    // groups, so per-row atomics made chains of ~dmax on one R word (r02aw)
    __syncthreads();
    for (int x = g.x_lo + (int)threadIdx.x; x < g.x_hi; x += (int)blockDim.x) {
      const unsigned long long v = Rs[x];
      if (v) {
        Rs[x] = 0ull;
        mark_removed(R, x, v, cl);
      }
    }
  }
}

// Which layout reads fewer bytes this pass?  rows: every live row in full
// (live x n masks); columns: every row of the tested columns (rows x ncol).
__device__ __forceinline__ bool pick_rows(const PassGeom& g, long long live, int ncol) {
  if (g.Mr == nullptr || g.force == 2) return false;
  if (g.force == 1) return true;
  const long long rows = (long long)(g.x_hi - g.x_lo) * g.dmax;
  // tiny tensors are latency-bound: whole rows are fewer, simpler work items
  if (rows * (long long)g.dbytes <= (256ll << 10)) return true;
  // bytes of each layout; a tie (a full pass over live rows: C3 / C4 W-stream,
  // pass 1 of a root call) goes to the row sweep: on some pool boxes the column
  // sweep streams ~20 % slower (C3 W-stream 110 vs 90 us, C4 5.75 vs 4.99 ms on
  // one box, profiles/r02an) while the row sweep runs ~90 us on every box
  // measured.  L2-resident tensors keep the column sweep for ties (C2: 14.4 vs
  // 16.3 us); force == 3 (RAC_FORCE_LAYOUT=tiecols) keeps it for every tie.
  const bool hbm = rows * (long long)g.dbytes > (64ll << 20);
  if (g.force == 3 || !hbm) return live * (long long)g.n < rows * (long long)ncol;
  return live * (long long)g.n <= rows * (long long)ncol;
}

// Live rows (x,a) of variables [x_lo, x_hi) in D (every thread of the CTA gets it).
template <int W>
__device__ __forceinline__ long long count_live(const uint8_t* Db, int x_lo, int x_hi, int* scratch) {
  int c = 0;
  for (int x = x_lo + threadIdx.x; x < x_hi; x += blockDim.x) c += __popcll(load_w<W>(Db + x * W));
  c = __reduce_add_sync(0xffffffffu, c);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = c;
  __syncthreads();
  long long tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += scratch[w];
  __syncthreads();
  return tot;
}

template <int W>
__device__ __forceinline__ void stage_from_u64(uint8_t* Db, const uint64_t* src, const uint64_t* dommask, int n,
                                               int dbytes) {
  uint32_t* w = reinterpret_cast<uint32_t*>(Db);
  for (int i = threadIdx.x; i < dbytes / 4; i += blockDim.x) w[i] = 0xffffffffu;
  __syncthreads();
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
__global__ void __launch_bounds__(kThreads, kMinBlocks) rac_fused(const __grid_constant__ FusedParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ int scratch[kThreads / 32];
  __shared__ int s_last;
  __shared__ int s_red[2][2];  // per-pass-parity block reductions: [flags, removed live values]
  const PassGeom& g = p.g;
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  uint16_t* vlist = reinterpret_cast<uint16_t*>(Db + list_offset(g.dbytes));
  uint8_t* vneed = Db + need_offset(g.dbytes, g.n);
  // phase timestamps (debug): thread 0 of CTA 0 records %globaltimer
  int nd = 0;
  const bool dbg = p.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
#define RAC_MARK() do { if (dbg && nd < 255) p.dbg[1 + nd++] = globaltimer(); } while (0)
  // per-CTA stamps (debug): [256 + 3*cta] start, first barrier arrival, end
  const bool dbg_cta = p.dbg != nullptr && threadIdx.x == 0 && blockIdx.x < 1000;
  if (dbg_cta) p.dbg[256 + 3 * blockIdx.x] = globaltimer();
  RAC_MARK();
  for (int i = threadIdx.x; i < g.n; i += blockDim.x) vneed[i] = 0;
  unsigned long long* Rs = (G > 0 && p.row_agg) ? reinterpret_cast<unsigned long long*>(Db + fused_smem(g.dbytes, g.n))
                                                : nullptr;  // per-CTA removal bits of the row sweep
  if (Rs)
    for (int i = threadIdx.x; i < g.n; i += blockDim.x) Rs[i] = 0ull;
  stage_from_u64<W>(Db, p.d_in, p.dommask, g.n, g.dbytes);
  RAC_MARK();
  const long warp0 = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const long nwarps = (long)gridDim.x * (blockDim.x / 32);
  constexpr int GG = G == 0 ? 1 : G;  // G == 0: the sparse arc-block variant
  const long gidx = warp0 * (32 / GG) + (threadIdx.x & 31) / GG, ngroups = nwarps * (32 / GG);
  const bool full = (p.flags & kFull) != 0;
  int t = 0, status = kOK, vcnt = g.n;
  unsigned epoch = 0;
  long long live = count_live<W>(Db, g.x_lo, g.x_hi, scratch);  // this rank's rows
  if (threadIdx.x < 4) s_red[threadIdx.x >> 1][threadIdx.x & 1] = 0;  // (ordered by later barriers)
  // Rotating buffers and the cross-rank sequence follow the global pass
  // number base + t, which continues across launches: pass k clears the
  // buffers of pass k+1, so no launch needs a cleanup phase and a peer that
  // is already in the next launch only writes buffers this rank has cleared.
  const unsigned long long base = *reinterpret_cast<volatile unsigned long long*>(p.seq);
  const bool mg = p.mir.world > 1;
  // Removal epochs: written straight to p.removed_at on one rank; with peers,
  // into this call's epoch array E[calls % 2] of every rank (put_epoch), the
  // other array cleared for the next such call, and copied out at the end.
  int32_t* ep = p.removed_at;
  EpochMirror em{};
  const EpochMirror* emp = nullptr;
  unsigned long long calls0 = 0;
  if (mg && p.removed_at) {
    calls0 = *reinterpret_cast<volatile unsigned long long*>(p.calls);
    const size_t ne = (size_t)g.n * 64, par = (size_t)(calls0 & 1ull);
    ep = p.E + par * ne;
    int32_t* enext = p.E + (par ^ 1) * ne;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += (size_t)gridDim.x * blockDim.x)
      enext[i] = 0;
    em.world = p.mir.world;
    em.rank = p.mir.rank;
    for (int q = 0; q < p.mir.world && q < kMaxRanks; ++q) em.E[q] = q == p.mir.rank ? nullptr : p.Epeer[q] + par * ne;
    emp = &em;
  }
  // sparse layout, single rank: removals also go to a per-pass change list, so
  // the tail of a pass reads only the changed variables' R words and needs no
  // compaction.  (Measured on the dense layout it is a wash -- C3 W-prop
  // 239 -> 235 us but W-seed 132 -> 143 us -- so dense passes keep the
  // full-R apply; sparse W-prop 319 -> 304 us.)
  const bool use_list = G == 0 && p.clist != nullptr && !mg;
  // dense layout: small late passes (few tested columns, so few removals) keep the
  // change list too -- its atomics are cheap there, and the pass tail then
  // reads only the listed R words and needs no compaction; large passes keep
  // the full-R apply (the list's atomics cost more than they save there)
  const bool list_ok = G > 0 && p.clist != nullptr && !mg;
  int b = (int)(base % 3ull);  // buffer of global pass base + t, advanced each pass
  int has_empty = 0;  // some D(x) empty (block-uniform)
  for (int x = threadIdx.x; x < g.n; x += blockDim.x) has_empty |= load_w<W>(Db + x * W) == 0;
  has_empty = __syncthreads_or(has_empty);
  // Seeded call (Alg. 1 with @changed = seeds): pass 1 tests only the seed
  // columns.  n_seeds < 0: root call (every column); n_seeds == 0: empty
  // @changed, no pass (the seeds pointer is not read).
  const bool seeded = p.n_seeds >= 0;
  if (seeded) {
    for (int i = threadIdx.x; i < p.n_seeds; i += blockDim.x) {
      const int y = p.seeds[i];
      if (y >= 0 && y < g.n) vneed[y] = 1;
    }
    __syncthreads();
    vcnt = block_compact(vneed, vlist, g.n, scratch);
  }
  if (seeded && vcnt == 0) {  // empty @changed: no pass (status from D_in)
    int wipe = 0;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) wipe |= load_w<W>(Db + x * W) == 0;
    wipe = __syncthreads_or(wipe);
    status = wipe ? kWIPEOUT : kOK;
  } else {
    for (;;) {
      ++t;
      b = b == 2 ? 0 : b + 1;                   // (base + t) % 3
      const int bn = b == 2 ? 0 : b + 1;        // (base + t + 1) % 3
      unsigned long long* Rc = p.R + (size_t)b * g.n;
      unsigned long long* Rn = p.R + (size_t)bn * g.n;
      // R (and the row counter) of pass t+1 were last used before the
      // previous barrier: clear them now.
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x) Rn[i] = 0ull;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (p.wctr) p.wctr[bn] = 0u;
        p.rflag[bn] = 0u;
        if (use_list || list_ok) p.clist[(size_t)bn * (g.n + 1)] = 0u;
      }
      if (p.cctr && blockIdx.x == 0 && threadIdx.x < kClaimParts) p.cctr[((size_t)bn * kClaimParts + threadIdx.x) * 32] = 0u;
      const bool lst = seeded || t > 1;  // pass 1 of a root call tests every column
      // (not pass 1: one seed column can still remove values of most variables)
      const bool lp = use_list || (list_ok && t > 1 && vcnt <= p.list_max);  // this pass keeps a change list
      uint32_t* clc = lp ? p.clist + (size_t)b * (g.n + 1) : nullptr;  // this pass's change list
      RAC_MARK();
      if constexpr (G == 0) {
        uint32_t* ipref = reinterpret_cast<uint32_t*>(Db + pref_offset(g.dbytes, g.n));
        uint32_t upl = kUnrollS;
        if (lst) {
          upl = block_prefix_items(vlist, vcnt, g.s_off, (uint32_t)g.s_vb, kUnrollS, nwarps, ipref, scratch);
        } else {  // every column: the item prefix precomputed at create
          for (int i = threadIdx.x; i <= g.n; i += blockDim.x) ipref[i] = __ldg(g.s_ipref + i);
          __syncthreads();
        }
        sparse_sweep<W>(g, Db, Rc, ep, t, warp0, nwarps, lst ? vlist : nullptr, lst ? vcnt : g.n, ipref,
                        upl, p.rflag + b, (RAC_COL_CLAIM && p.wctr) ? p.wctr + b : nullptr, clc);
      } else {
        if (pick_rows(g, live, lst ? vcnt : g.n))
          row_sweep<W, G>(g, Ds, Rc, ep, t, gidx, ngroups, p.wctr ? p.wctr + b : nullptr, p.rflag + b,
                          clc, emp, Rs);
        else
          column_sweep<W>(g, Db, Rc, ep, t, warp0, nwarps, lst ? vlist : nullptr, lst ? vcnt : g.n,
                          p.rflag + b, (RAC_COL_CLAIM == 1 && p.wctr) ? p.wctr + b : nullptr, clc, emp,
                          p.cctr ? p.cctr + (size_t)b * kClaimParts * 32 : nullptr);
      }
      RAC_MARK();
      if (p.dbg != nullptr && t == 1) {  // block-uniform condition: the barrier is safe
        __syncthreads();
        if (dbg_cta) p.dbg[256 + 3 * blockIdx.x + 1] = globaltimer();
      }
      grid_sync(p.bar, gridDim.x, ++epoch, (int)(p.ab & 1u));
      if (mg) {
        // Row-sharded exchange: R of this rank's rows is complete; copy its
        // non-zero words into every peer's R (a peer's words for these rows are
        // zero until then: cleared in its previous pass, written only here),
        // raise the peers' removal flags, then the cross-rank barrier.
        if (__ldcg(p.rflag + b) != 0u) {
          for (int x = g.x_lo + blockIdx.x * blockDim.x + threadIdx.x; x < g.x_hi; x += gridDim.x * blockDim.x) {
            const unsigned long long v = __ldcg(&Rc[x]);
            if (v)
              for (int q = 0; q < p.mir.world; ++q)
                if (q != p.mir.rank) p.mir.R[q][(size_t)b * g.n + x] = v;
          }
          if (blockIdx.x == 0 && threadIdx.x == 0)
            for (int q = 0; q < p.mir.world; ++q)
              if (q != p.mir.rank) atomicOr_system(p.mir.flag[q] + b, 1u);
        }
        grid_sync_peer(p.bar, gridDim.x, ++epoch, p, base + (unsigned long long)t);
      }
      RAC_MARK();
      // D_t = D_{t-1} & ~R (every CTA, redundantly); flags for Alg. 1's checks;
      // the changed variables are the next pass's columns.  A pass that
      // removed nothing (the per-pass flag is still 0) leaves D as it was:
      // changed = 0, wipe = "D already had an empty row", no R read.
      int changed = 0, wipe = 0;
      bool listed = false;  // vlist/vcnt already hold the next pass's columns
      if (lp) {
        const int cnt = (int)__ldcg(clc);
        if (cnt == 0) {
          wipe = has_empty;
        } else {
          // every listed x lost a live value (marks are made for live rows only)
          int wp = 0, nrm = 0;
          const int par = t & 1;
          if (threadIdx.x == 0) s_red[par ^ 1][0] = 0, s_red[par ^ 1][1] = 0;  // next pass's slots
          for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int x = (int)__ldcg(clc + 1 + i);
            const uint64_t rv = __ldcg(&Rc[x]);
            const uint64_t dv = load_w<W>(Db + x * W);
            const uint64_t nd = dv & ~rv;
            store_w<W>(Db + x * W, nd);
            wp |= nd == 0;
            if (x >= g.x_lo && x < g.x_hi) nrm += __popcll(dv & rv);
            vlist[i] = (uint16_t)x;
          }
          wp = __reduce_or_sync(0xffffffffu, wp);
          nrm = __reduce_add_sync(0xffffffffu, nrm);
          if ((threadIdx.x & 31) == 0) {
            if (wp) atomicOr_block(&s_red[par][0], 2);
            if (nrm) atomicAdd_block(&s_red[par][1], nrm);
          }
          __syncthreads();
          changed = 1;
          wipe = has_empty | ((s_red[par][0] >> 1) & 1);
          live -= s_red[par][1];
          vcnt = cnt;
          listed = true;
        }
      } else if (!(p.ab & 4u) && __ldcg(p.rflag + b) == 0u) {  // ab bit 2: read R unconditionally
        wipe = has_empty;
      } else if (p.ab & 2u) {
        // A/B variant (RAC_FUSED_AB bit 1; measured slightly slower than the
        // separate compaction below, profiles/r02c/ab_fused.log): D_t = D_{t-1} &
        // ~R with the next pass's column list built in the same sweep: thread i
        // owns the contiguous variables [i*chunk, (i+1)*chunk), so a block scan of
        // the per-thread change counts gives every CTA the same ascending list
        // (the item -> column mapping must agree across CTAs).
        const int T = blockDim.x, chunk = (g.n + T - 1) / T;  // <= 128 (n <= 65535)
        const int xb = min(g.n, (int)threadIdx.x * chunk), xe = min(g.n, xb + chunk);
        const int par = t & 1;
        if (threadIdx.x == 0) s_red[par ^ 1][1] = 0;  // next pass's slot
        uint32_t cm[4] = {0u, 0u, 0u, 0u};
        int nrm = 0, wl = 0, cnt = 0;
        for (int x0 = xb; x0 < xe; x0 += 4) {
          uint64_t rv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) rv[k] = x0 + k < xe ? __ldcg(&Rc[x0 + k]) : 0ull;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + k;
            if (x >= xe) break;
            const uint64_t dv = load_w<W>(Db + x * W);
            const uint64_t nd = dv & ~rv[k];
            if ((dv & rv[k]) != 0) {
              store_w<W>(Db + x * W, nd);
              cm[(x - xb) >> 5] |= 1u << ((x - xb) & 31);
              ++cnt;
              wl |= nd == 0;
              if (x >= g.x_lo && x < g.x_hi) nrm += __popcll(dv & rv[k]);
            }
          }
        }
        nrm = __reduce_add_sync(0xffffffffu, nrm);
        if ((threadIdx.x & 31) == 0 && nrm) atomicAdd_block(&s_red[par][1], nrm);
        uint32_t total = 0;
        uint32_t pos = block_scan_u32((uint32_t)cnt, &total, scratch);  // barriers inside
        for (int w = 0; w < 4; ++w)
          for (uint32_t m = cm[w]; m; m &= m - 1u) vlist[pos++] = (uint16_t)(xb + 32 * w + __ffs(m) - 1);
        wipe = has_empty | __syncthreads_or(wl);  // also publishes vlist
        changed = total > 0;
        live -= s_red[par][1];
        vcnt = (int)total;
        listed = true;
      } else {
        // one block barrier for the three reductions: flags (changed | wipe)
        // and the live values of the local rows this pass removed
        int nrm = 0;
        const int par = t & 1;
        if (threadIdx.x == 0) { s_red[par ^ 1][0] = 0; s_red[par ^ 1][1] = 0; }  // next pass's slots
        for (int x0 = threadIdx.x; x0 < g.n; x0 += 4 * blockDim.x) {
          uint64_t rv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + k * blockDim.x;
            rv[k] = x < g.n ? __ldcg(&Rc[x]) : 0ull;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int x = x0 + k * blockDim.x;
            if (x >= g.n) break;
            const uint64_t dv = load_w<W>(Db + x * W);
            const uint64_t nd = dv & ~rv[k];
            store_w<W>(Db + x * W, nd);
            const bool chx = (dv & rv[k]) != 0;
            changed |= chx;
            wipe |= nd == 0;
            if (chx) vneed[x] = 1;
            if (x >= g.x_lo && x < g.x_hi) nrm += __popcll(dv & rv[k]);
          }
        }
        const int fl = __reduce_or_sync(0xffffffffu, changed | (wipe << 1));
        nrm = __reduce_add_sync(0xffffffffu, nrm);
        if ((threadIdx.x & 31) == 0) {
          if (fl) atomicOr_block(&s_red[par][0], fl);
          if (nrm) atomicAdd_block(&s_red[par][1], nrm);
        }
        __syncthreads();
        changed = s_red[par][0] & 1;
        wipe = (s_red[par][0] >> 1) & 1;
        live -= s_red[par][1];
      }
      has_empty = wipe;
      RAC_MARK();
      if (wipe && !full) { status = kWIPEOUT; break; }          // Alg. 1
      if (!changed) { status = wipe ? kWIPEOUT : kOK; break; }  // Prop. 1 end condition
      if (!listed) vcnt = block_compact(vneed, vlist, g.n, scratch);  // next pass's columns
      RAC_MARK();
    }
  }
  if (emp && t > 0) {
    // every rank's epochs arrived before the last cross-rank barrier
    const size_t ne = (size_t)g.n * 64;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += (size_t)gridDim.x * blockDim.x)
      p.removed_at[i] = __ldcv(ep + i);
  }
  if (blockIdx.x == 0) {
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) p.d_out[x] = load_w<W>(Db + x * W);
    if (threadIdx.x == 0) {
      if (emp && t > 0) *p.calls = calls0 + 1ull;  // every CTA read *calls before the first barrier
      *p.iters = t;
      *p.status = (mg && *reinterpret_cast<volatile int32_t*>(p.xerr)) ? kPeerTimeout : status;
      // every CTA read *p.seq before the first barrier
      if (t > 0) *p.seq = base + (unsigned long long)t;
    }
  }
  RAC_MARK();
  if (dbg) p.dbg[0] = nd;
  if (dbg_cta) p.dbg[256 + 3 * blockIdx.x + 2] = globaltimer();
#undef RAC_MARK
  // The last CTA out resets the barrier words: every other CTA has passed its
  // last barrier by the time it counts itself out.
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = gridDim.x == 1 ? 1 : (atomicAdd(&p.bar[2], 1u) + 1u == gridDim.x);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0 && gridDim.x > 1) {
      p.bar[0] = 0u;
      p.bar[1] = 0u;
      p.bar[2] = 0u;
    }
    __threadfence();
  }
}

// ---------------------------------------------------------------------------- per-pass (sharded)
__device__ __forceinline__ void tma_stage(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* mbar) {
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
__global__ void __launch_bounds__(kThreads, kMinBlocks) rac_pass(PassParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ alignas(8) uint64_t mbar;
  if (*reinterpret_cast<volatile int32_t*>(p.s.done)) return;  // converged: speculative pass is a no-op
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  tma_stage(Db, p.s.Dw, (uint32_t)p.g.dbytes, &mbar);
  const int t = *p.s.iters + 1;
  const int vcnt = *p.s.vcnt;
  const bool lst = t > 1 || *p.s.seeded;
  uint16_t* vlist = reinterpret_cast<uint16_t*>(Db + list_offset(p.g.dbytes));
  if (lst) {
    for (int i = threadIdx.x; i < vcnt; i += blockDim.x) vlist[i] = p.s.vlist[i];
    __syncthreads();
  }
  const long warp0 = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const long nwarps = (long)gridDim.x * (blockDim.x / 32);
  __shared__ int scratch[kThreads / 32];
  const long long live = count_live<W>(Db, p.g.x_lo, p.g.x_hi, scratch);
  if (pick_rows(p.g, live, lst ? vcnt : p.g.n))
    row_sweep<W, G>(p.g, Ds, p.s.R, p.removed_at, t, warp0 * (32 / G) + (threadIdx.x & 31) / G, nwarps * (32 / G));
  else
    column_sweep<W>(p.g, Db, p.s.R, p.removed_at, t, warp0, nwarps, lst ? vlist : nullptr, lst ? vcnt : p.g.n);
}

__global__ void rac_shard_init(ShardState s, const uint64_t* d_in, const uint64_t* dommask, int n, int W, int dbytes,
                               int total_g) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total_g; i += gridDim.x * blockDim.x) {
    if (i < n) {
      const uint64_t v = d_in[i] & dommask[i];
      s.Dcur[i] = v;
      s.R[i] = 0ull;
      for (int k = 0; k < W; ++k) s.Dw[(size_t)i * W + k] = (uint8_t)(v >> (8 * k));
    }
    s.Dg[i] = 0ull;
  }
  for (int b = n * W + blockIdx.x * blockDim.x + threadIdx.x; b < dbytes; b += gridDim.x * blockDim.x)
    s.Dw[b] = 0xffu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *s.iters = 0;
    *s.status = -1;
    *s.done = 0;
    *s.vcnt = 0;
    *s.seeded = 0;
  }
}

// Seeded call (Alg. 1 tensorAC(Vars, @changed = seeds)): pass 1 tests
// the columns of the listed variables (out-of-range entries skipped,
// duplicates once).  An empty list means no pass: done, iterations 0, status
// from D_in.  One CTA; dynamic smem = n flag bytes.
__global__ void __launch_bounds__(1024) rac_shard_seed(ShardState s, const int32_t* seeds, int n_seeds, int n) {
  extern __shared__ uint8_t need[];
  __shared__ int scratch[32];
  for (int i = threadIdx.x; i < n; i += blockDim.x) need[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n_seeds; i += blockDim.x) {
    const int y = seeds[i];
    if (y >= 0 && y < n) need[y] = 1;
  }
  __syncthreads();
  const int cnt = block_compact(need, s.vlist, n, scratch);
  int wipe = 0;
  for (int x = threadIdx.x; x < n; x += blockDim.x) wipe |= s.Dcur[x] == 0ull;
  wipe = __syncthreads_or(wipe);
  if (threadIdx.x == 0) {
    *s.vcnt = cnt;
    *s.seeded = 1;
    if (cnt == 0) {
      *s.status = wipe ? kWIPEOUT : kOK;
      *s.done = 1;
    }
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
// changed variables (the next pass's columns, Prop. 2), and advances.
// One CTA; dynamic smem = n flag bytes.
__global__ void __launch_bounds__(1024) rac_shard_update(ShardState s, int n, int W, uint32_t flags) {
  extern __shared__ uint8_t need[];
  __shared__ int scratch[32];
  if (*reinterpret_cast<volatile int32_t*>(s.done)) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) need[i] = 0;
  __syncthreads();
  int changed = 0, wipe = 0;
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    const uint64_t nv = s.Dg[x];
    const bool chx = nv != s.Dcur[x];
    changed |= chx;
    wipe |= nv == 0;
    if (chx) need[x] = 1;
    s.Dcur[x] = nv;
    for (int k = 0; k < W; ++k) s.Dw[(size_t)x * W + k] = (uint8_t)(nv >> (8 * k));
  }
  changed = __syncthreads_or(changed);
  wipe = __syncthreads_or(wipe);
  const int cnt = block_compact(need, s.vlist, n, scratch);
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

// ---------------------------------------------------------------------------- batched (per state)
// One CTA per state: D, the column list and R live in smem, __syncthreads is
// the pass barrier, each state stops at its own pass (freeze-on-stop).  The
// relation is shared by all states and stays L2-resident.
template <int W, int G>
__global__ void __launch_bounds__(kThreads, kMinBlocks) rac_batch(BatchParams p) {
  extern __shared__ uint4 Ds[];
  __shared__ int scratch[kThreads / 32];
  const PassGeom& g = p.g;
  const int s = blockIdx.x;
  uint8_t* Db = reinterpret_cast<uint8_t*>(Ds);
  uint16_t* vlist = reinterpret_cast<uint16_t*>(Db + list_offset(g.dbytes));
  uint8_t* vneed = Db + need_offset(g.dbytes, g.n);
  unsigned long long* R = reinterpret_cast<unsigned long long*>(Db + fused_smem(g.dbytes, g.n));
  for (int i = threadIdx.x; i < g.n; i += blockDim.x) vneed[i] = 0;
  stage_from_u64<W>(Db, p.d_in + (size_t)s * g.n, p.dommask, g.n, g.dbytes);
  const long warp0 = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const long gidx = warp0 * (32 / G) + (threadIdx.x & 31) / G, ngroups = nwarps * (32 / G);
  const bool full = (p.flags & kFull) != 0;
  int t = 0, status = kOK, vcnt = g.n;
  long long live = count_live<W>(Db, 0, g.n, scratch);
  const int seed = p.seed_var ? p.seed_var[s] : -1;
  const bool seeded = seed >= 0 && seed < g.n;
  if (seeded) {
    if (threadIdx.x == 0) vneed[seed] = 1;
    __syncthreads();
    vcnt = block_compact(vneed, vlist, g.n, scratch);
  }
  for (;;) {
    ++t;
    for (int x = threadIdx.x; x < g.n; x += blockDim.x) R[x] = 0ull;
    __syncthreads();
    const bool lst = seeded || t > 1;
    if (pick_rows(g, live, lst ? vcnt : g.n))
      row_sweep<W, G>(g, Ds, R, p.removed_at, t, gidx, ngroups);
    else
      column_sweep<W>(g, Db, R, p.removed_at, t, warp0, nwarps, lst ? vlist : nullptr, lst ? vcnt : g.n);
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
      if (chx) vneed[x] = 1;
    }
    changed = __syncthreads_or(changed);
    wipe = __syncthreads_or(wipe);
    vcnt = block_compact(vneed, vlist, g.n, scratch);
    live = count_live<W>(Db, 0, g.n, scratch);
    if (wipe && !full) { status = kWIPEOUT; break; }
    if (!changed) { status = wipe ? kWIPEOUT : kOK; break; }
  }
  for (int x = threadIdx.x; x < g.n; x += blockDim.x) p.d_out[(size_t)s * g.n + x] = load_w<W>(Db + x * W);
  if (threadIdx.x == 0) {
    p.iters[s] = t;
    p.status[s] = status;
  }
}

template <typename K>
cudaError_t set_smem(K k, size_t smem) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int W, int G>
struct LaunchF {
  static cudaError_t fused(const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool coop) {
    auto k = rac_fused<W, G>;
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    if (coop) {
      FusedParams pp = p;
      void* args[] = {&pp};
      return cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kThreads), args, smem, s);
    }
    k<<<grid, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t occ_fused(size_t smem, int* out) {
    const void* k = (const void*)rac_fused<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kThreads, smem);
  }
};

template <int W, int G>
struct Launch {
  static cudaError_t pass(const PassParams& p, int grid, size_t smem, cudaStream_t s) {
    auto k = rac_pass<W, G>;
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t batch(const BatchParams& p, int n_states, size_t smem, cudaStream_t s) {
    auto k = rac_batch<W, G>;
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    k<<<n_states, kThreads, smem, s>>>(p);
    return cudaGetLastError();
  }
  static cudaError_t occ(int which, size_t smem, int* out) {
    const void* k = which == 1 ? (const void*)rac_pass<W, G> : (const void*)rac_batch<W, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, kThreads, smem);
  }
};

}  // namespace

#define RAC_G_SWITCH(WW, G, CALL)                                  \
  switch (G) {                                                     \
    case 1: return Launch<WW, 1>::CALL;                            \
    case 2: return Launch<WW, 2>::CALL;                            \
    case 4: return Launch<WW, 4>::CALL;                            \
    case 8: return Launch<WW, 8>::CALL;                            \
    case 16: return Launch<WW, 16>::CALL;                          \
    case 32: return Launch<WW, 32>::CALL;                          \
    default: return cudaErrorInvalidValue;                         \
  }
// fused kernel only: G == 0 selects the sparse arc-block variant
#define RAC_G0_SWITCH(WW, G, CALL)                                 \
  switch (G) {                                                     \
    case 0: return LaunchF<WW, 0>::CALL;                           \
    case 1: return LaunchF<WW, 1>::CALL;                           \
    case 2: return LaunchF<WW, 2>::CALL;                           \
    case 4: return LaunchF<WW, 4>::CALL;                           \
    case 8: return LaunchF<WW, 8>::CALL;                           \
    case 16: return LaunchF<WW, 16>::CALL;                         \
    case 32: return LaunchF<WW, 32>::CALL;                         \
    default: return cudaErrorInvalidValue;                         \
  }
#define RAC_WG0_SWITCH(W, G, CALL)                                 \
  switch (W) {                                                     \
    case 1: RAC_G0_SWITCH(1, G, CALL)                              \
    case 2: RAC_G0_SWITCH(2, G, CALL)                              \
    case 4: RAC_G0_SWITCH(4, G, CALL)                              \
    case 8: RAC_G0_SWITCH(8, G, CALL)                              \
    default: return cudaErrorInvalidValue;                         \
  }
#define RAC_WG_SWITCH(W, G, CALL)                                  \
  switch (W) {                                                     \
    case 1: RAC_G_SWITCH(1, G, CALL)                               \
    case 2: RAC_G_SWITCH(2, G, CALL)                               \
    case 4: RAC_G_SWITCH(4, G, CALL)                               \
    case 8: RAC_G_SWITCH(8, G, CALL)                               \
    default: return cudaErrorInvalidValue;                         \
  }

int choose_group(int nvec) {
  // smallest power of two G with G * kUnrollR >= nvec, capped at a warp
  int G = 1;
  while (G < 32 && G * kUnrollR < nvec) G *= 2;
  return G;
}

cudaError_t launch_fused(int W, int G, const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool coop) {
  RAC_WG0_SWITCH(W, G, fused(p, grid, smem, s, coop))
}
cudaError_t fused_occupancy(int W, int G, size_t smem, int* out) { RAC_WG0_SWITCH(W, G, occ_fused(smem, out)) }
cudaError_t launch_pass(int W, int G, const PassParams& p, int grid, size_t smem, cudaStream_t s) {
  RAC_WG_SWITCH(W, G, pass(p, grid, smem, s))
}
cudaError_t pass_occupancy(int W, int G, size_t smem, int* out) { RAC_WG_SWITCH(W, G, occ(1, smem, out)) }
cudaError_t launch_batch(int W, int G, const BatchParams& p, int n_states, size_t smem, cudaStream_t s) {
  RAC_WG_SWITCH(W, G, batch(p, n_states, smem, s))
}
cudaError_t batch_occupancy(int W, int G, size_t smem, int* out) { RAC_WG_SWITCH(W, G, occ(2, smem, out)) }

cudaError_t launch_shard_init(const ShardState& s, const uint64_t* d_in, const uint64_t* dommask, int n, int W,
                              int dbytes, int total_g, cudaStream_t st) {
  int work = total_g > dbytes ? total_g : dbytes;
  int grid = (work + 255) / 256;
  if (grid > 1024) grid = 1024;
  rac_shard_init<<<grid, 256, 0, st>>>(s, d_in, dommask, n, W, dbytes, total_g);
  return cudaGetLastError();
}
cudaError_t launch_shard_seed(const ShardState& s, const int32_t* seeds, int n_seeds, int n, cudaStream_t st) {
  if (n > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rac_shard_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, n);
    if (e != cudaSuccess) return e;
  }
  rac_shard_seed<<<1, 1024, n, st>>>(s, seeds, n_seeds, n);
  return cudaGetLastError();
}
cudaError_t launch_shard_slice(const ShardState& s, int x_lo, int x_hi, int n, cudaStream_t st) {
  int cnt = x_hi - x_lo;
  int grid = (cnt + 255) / 256;
  if (grid < 1) grid = 1;
  rac_shard_slice<<<grid, 256, 0, st>>>(s, x_lo, x_hi, n);
  return cudaGetLastError();
}
cudaError_t launch_shard_update(const ShardState& s, int n, int W, uint32_t flags, cudaStream_t st) {
  if (n > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(rac_shard_update, cudaFuncAttributeMaxDynamicSharedMemorySize, n);
    if (e != cudaSuccess) return e;
  }
  rac_shard_update<<<1, 1024, n, st>>>(s, n, W, flags);
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
