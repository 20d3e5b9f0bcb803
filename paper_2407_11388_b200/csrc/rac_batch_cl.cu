// rac_batch_cl.cu -- batched enforcement: 32 domain states
// per bit-sliced word, each word owned by ONE thread-block cluster.
//
// Many search-tree nodes (Alg. 2) on one instance.
// The states are bit-sliced: for a word of 32 states, X[(x,a)] is a u32 whose
// bit j says (x,a) ∈ D_j, and one pass of Eq. 1 (lines 89-99) for all 32
// states is
//   X'[(x,a)] = X[(x,a)] & AND_{y tested} ( OR_{b ∈ c_xy|(x,a)} X[(y,b)]  |  ~tst[y] )
// where tst[y] = the active states for which y changed in the previous pass
// (the seed variable of a seeded state in pass 1, every variable of a root
// state): Alg. 1's Cons[:, @changed] (line 215) per state, so every state
// follows its own Alg. 1 trajectory exactly.  The OR over b comes from
// per-column chunk tables in shared memory,
//   T[y][q][v] = OR_{j : bit j of v} X[(y, shift_q + j)],
// one lookup per chunk of the mask (W=2: chunks of 6+5+5 bits, 3 lookups per
// mask; W=1: 2 nibbles; W=4: 8 nibbles).  A table is rebuilt only when its
// column's rows changed.  Per-state loop control (Alg. 1):
// wipeout first, then "changed", each state frozen at its own pass.
//
// Cluster organisation: the word's CTAs form ONE cluster, each owning a block
// of rows (whole variables) and keeping the whole word's slices X in shared
// memory.  Per pass:
//   prep   tst / the tested-column list (warp 0) and the tables of changed
//          columns (the other warps); then a split cluster barrier ARRIVE
//          ("I have read everybody's rows");
//   sweep  my rows against the tested-column list (column-major masks, one
//          2/4-byte load per tested column, 8 in flight); a row stops as soon
//          as none of its live states is supported.  (Testing every column
//          through the row-major copy, one 16-byte load per 16/W columns, was
//          measured slower: a warp's 16-byte row loads touch 32 lines.)
//   push   split barrier WAIT, then DSMEM stores of my changed rows, my change
//          masks and my [changed, emptied] lanes into every CTA of the cluster;
//   sync   one full cluster barrier; every CTA derives the same loop control.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>

#include "rac_internal.cuh"

namespace cg = cooperative_groups;

namespace rac {

namespace {

// build-time A/B variants (tools/session scripts build them with -D)
// (profiles/r02aa, same box: item tables 242 -> 234 us per C5 batch, global
// staging 242 -> 240, both 232; the alternatives stay selectable with -D...=0.
// Also measured, no gain: rotated conflict-free table stores (r02ab), a u32
// column list with 8 or 16 masks in flight per row (r02am: 232 / 236 us).)
#ifndef RAC_CL_ITEM_TABLES
#define RAC_CL_ITEM_TABLES 1  // 1: tables built one 16-entry block per thread; 0: one warp per column
#endif
#ifndef RAC_CL_STAGE_IF
#define RAC_CL_STAGE_IF 8  // variables whose 32 states a warp loads at once when staging a word (4 or 8: same, r02ba)
#endif
#ifndef RAC_CL_GLOBAL_STAGE
#define RAC_CL_GLOBAL_STAGE 1  // 1: the word's states transposed by ballots straight from global memory;
                               // 0: staged through shared memory by coalesced loads first
#endif

constexpr uint32_t kFullCL = 1u;  // RAC_FULL_FIXPOINT
constexpr int kMaxT = kBatchClThreads;
constexpr int kMaxC = 16;

// Chunk tables per mask width W: chunk q covers values [shift(q), shift(q) +
// bits(q)) of the mask; its table (2^bits(q) words) sits at byte off(q) of the
// column's TSB-byte table block.  TSB exceeds every chunk's largest byte
// offset, so (column base | entry offset) is an OR of disjoint bits.
template <int W>
struct Lut;
template <>
struct Lut<1> {
  static constexpr int NCH = 2, TSB = 128;
  __host__ __device__ static constexpr int bits(int) { return 4; }
  __host__ __device__ static constexpr int shift(int q) { return 4 * q; }
  __host__ __device__ static constexpr int off(int q) { return 64 * q; }
};
template <>
struct Lut<2> {
  static constexpr int NCH = 3, TSB = 512;
  __host__ __device__ static constexpr int bits(int q) { return q == 0 ? 6 : 5; }
  __host__ __device__ static constexpr int shift(int q) { return q == 0 ? 0 : (q == 1 ? 6 : 11); }
  __host__ __device__ static constexpr int off(int q) { return q == 0 ? 0 : (q == 1 ? 256 : 384); }
};
template <>
struct Lut<4> {
  static constexpr int NCH = 8, TSB = 512;
  __host__ __device__ static constexpr int bits(int) { return 4; }
  __host__ __device__ static constexpr int shift(int q) { return 4 * q; }
  __host__ __device__ static constexpr int off(int q) { return 64 * q; }
};

template <int IMM>
__device__ __forceinline__ uint32_t lds_imm(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(IMM));
  return v;
}

// Split cluster barrier.  The arrive is relaxed: what it announces ("I have
// read the peers' rows and my chg_in") needs no memory release -- those loads
// were consumed into shared-memory stores before the preceding __syncthreads --
// and a release arrive costs a MEMBAR.ALL.GPU per pass.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// DSMEM pushes: st.async stores into a peer CTA's shared memory that complete
// bytes on the peer's mbarrier (the peer's wait on its own mbarrier is the
// only synchronisation the data needs).
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(raddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               :: "r"(raddr), "r"(v), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t a, uint32_t b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
               :: "r"(raddr), "r"(a), "r"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}

// Bytes CTA k receives per pass: from every other rank q, its rows (16-byte
// stores, rounded up), its change masks and its two-word partial.
__device__ __forceinline__ uint32_t incoming_bytes(int k, int C, int RPC, int rows, int dmax) {
  uint32_t b = 0;
  for (int q = 0; q < C; ++q) {
    if (q == k) continue;
    const int a0 = q * RPC, a1 = min(rows, a0 + RPC);
    if (a1 <= a0) continue;
    b += 16u * (uint32_t)((a1 - a0 + 3) / 4) + 4u * (uint32_t)(a1 / dmax - a0 / dmax) + 8u;
  }
  return b;
}

// Byte offset of the table entry of chunk Q for the mask at bit SH of w.
template <int W, int Q, int SH>
__device__ __forceinline__ uint32_t lut_off(uint32_t w) {
  constexpr int S = Lut<W>::shift(Q) + SH;
  constexpr uint32_t MSK = ((1u << Lut<W>::bits(Q)) - 1u) << 2;
  if constexpr (S >= 2) return (w >> (S - 2)) & MSK;
  else return (w << (2 - S)) & MSK;
}

// OR over the mask's values of X[(y, b)]: one shared-memory lookup per chunk,
// address (cb | entry offset) + IMM + off(q): cb = the shared-memory address of
// a TSB-aligned table block, IMM = the column's block relative to cb.
template <int W, int SH, int IMM, int Q = 0>
__device__ __forceinline__ uint32_t sup_lookup(uint32_t w, uint32_t cb) {
  const uint32_t s = lds_imm<IMM + Lut<W>::off(Q)>(cb | lut_off<W, Q, SH>(w));
  if constexpr (Q + 1 < Lut<W>::NCH) return s | sup_lookup<W, SH, IMM, Q + 1>(w, cb);
  else return s;
}

// The chunk tables of column y, built by one warp: lane l computes the entries
// e = l, l + 32, ... of the column's TSB / 4 words (entry e of chunk q holds
// OR_{bit k of v} X[(y, shift(q) + k)], v = e - off(q) / 4).  The X words are
// read as broadcasts (every lane of a chunk reads the same address) and the
// stores are consecutive words (conflict-free).
template <int W>
__device__ __forceinline__ void build_column(uint8_t* Tb, const uint32_t* X, int y, int dmax, int lane) {
  const uint32_t* Xy = X + (size_t)y * dmax;
  uint32_t* Ty = reinterpret_cast<uint32_t*>(Tb + (size_t)y * Lut<W>::TSB);
#pragma unroll
  for (int e0 = 0; e0 < Lut<W>::TSB / 4; e0 += 32) {
    const int e = e0 + lane;
    int q = 0;
#pragma unroll
    for (int qq = 1; qq < Lut<W>::NCH; ++qq)
      if (e >= Lut<W>::off(qq) / 4) q = qq;
    const int v = e - Lut<W>::off(q) / 4, b0 = Lut<W>::shift(q), nb = Lut<W>::bits(q);
    uint32_t acc = 0u;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int b = b0 + k;
      if (k < nb && b < dmax && ((v >> k) & 1)) acc |= Xy[b];
    }
    Ty[e] = acc;
  }
}

#if RAC_CL_ITEM_TABLES
// A/B variant (build-time): one thread per 16-entry block (item i of column y:
// chunk q, block bi), the block built in registers and stored as 4 x 16 bytes.
template <int W>
__device__ __forceinline__ void build_item(uint8_t* Tb, const uint32_t* X, int y, int i, int dmax) {
  int q = 0, bi = i;
  while (bi >= (1 << (Lut<W>::bits(q) - 4))) {
    bi -= 1 << (Lut<W>::bits(q) - 4);
    ++q;
  }
  const int b0 = Lut<W>::shift(q), nb = Lut<W>::bits(q);
  const uint32_t* Xy = X + (size_t)y * dmax;
  uint32_t xb[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) xb[j] = b0 + j < dmax ? Xy[b0 + j] : 0u;
  uint32_t hi = 0u;
  for (int k = 0; k < nb - 4; ++k)
    if (((bi >> k) & 1) && b0 + 4 + k < dmax) hi |= Xy[b0 + 4 + k];
  uint32_t tv[16];
  tv[0] = hi;
#pragma unroll
  for (int v = 1; v < 16; ++v) {
    const int lb = (v & 1) ? 0 : (v & 2) ? 1 : (v & 4) ? 2 : 3;  // lowest set bit (folds; __ffs would not)
    tv[v] = tv[v & (v - 1)] | xb[lb];
  }
  uint4* dst = reinterpret_cast<uint4*>(Tb + (size_t)y * Lut<W>::TSB + Lut<W>::off(q) + bi * 64);
#pragma unroll
  for (int v = 0; v < 16; v += 4) dst[v >> 2] = make_uint4(tv[v], tv[v + 1], tv[v + 2], tv[v + 3]);
}
#endif

template <int W>
__device__ __forceinline__ uint32_t mask_at(const uint8_t* p) {
  if constexpr (W == 4) return __ldg(reinterpret_cast<const uint32_t*>(p));
  else if constexpr (W == 2) return __ldg(reinterpret_cast<const uint16_t*>(p));
  else return __ldg(p);
}

// Presence (R2): an absent pair's mask is all ones, so it can only "fail" for
// a state whose D(y) is empty; such a lane is kept by the presence bit.
__device__ __forceinline__ bool present(const uint32_t* P, int pw, int x, int y) {
  return (__ldg(P + (size_t)x * pw + (y >> 5)) >> (y & 31)) & 1u;
}

// One column's test: acc &= sup | ~t (t = lanes that test this column).
template <bool CP>
__device__ __forceinline__ void apply_col(uint32_t& acc, uint32_t s, uint32_t t, uint32_t live, const uint32_t* P,
                                          int pw, int x, int y) {
  if constexpr (CP) {
    if ((s & live & t) != (live & t) && !present(P, pw, x, y)) s = 0xffffffffu;
  }
  acc &= s | ~t;
}

// Listed columns: ci[c] = {byte offset of column c's masks, byte offset of its
// table block}, ctst[c] = the lanes that test it; the list is padded to a
// multiple of 8 with entries that test no lane.
template <int W, bool CP>
__device__ __forceinline__ uint32_t sweep_list(const uint8_t* __restrict__ M, const uint32_t* __restrict__ P, int pw,
                                               uint32_t* X, uint32_t tb0, const uint2* ci, const uint32_t* ctst,
                                               int cnt8, int r0, int r1, int dmax, uint32_t active, uint32_t* chgn) {
  uint32_t my_or = 0u;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    const uint32_t cur = X[r];
    const uint32_t live = cur & active;
    if (!live) continue;
    const uint8_t* Mrow = M + (size_t)r * W;
    const int x = r / dmax;
    uint32_t acc = 0xffffffffu;
    for (int c0 = 0; c0 < cnt8 && (acc & live) != 0u; c0 += 8) {
      uint2 cc[8];
      uint32_t mv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = ci[c0 + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) mv[u] = mask_at<W>(Mrow + cc[u].x);
      const uint4 ta = *reinterpret_cast<const uint4*>(ctst + c0);
      const uint4 tb = *reinterpret_cast<const uint4*>(ctst + c0 + 4);
      const uint32_t tz[8] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t s = sup_lookup<W, 0, 0>(mv[u], tb0 + cc[u].y);
        apply_col<CP>(acc, s, tz[u], live, P, pw, x, (int)(cc[u].y / Lut<W>::TSB));
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

// Per-state sweep (few active states): state s of slot k tests its own changed
// columns psl[k][0..psc[k]) against its own D_s(y) (psd[k][.], W-bit values
// extracted from the bit slices), one mask load and one AND per test instead
// of the word's union of columns through the chunk tables.  A failing test
// clears the row's lane s; an absent pair never fails (its mask is all ones,
// so m & D_s(y) == 0 only when D_s(y) is empty: then the presence bit decides).
constexpr int kPsMax = 8;  // per-state mode when at most this many states are active
template <int W, bool CP>
__device__ __forceinline__ uint32_t sweep_states(const uint8_t* __restrict__ M, size_t col_stride,
                                                 const uint32_t* __restrict__ P, int pw, uint32_t* X,
                                                 const uint16_t* psl, const uint32_t* psd, const int* psc,
                                                 const int* pslane, int nps, int stride, int r0, int r1, int dmax,
                                                 uint32_t active, uint32_t* chgn) {
  uint32_t my_or = 0u;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    const uint32_t cur = X[r];
    const uint32_t live = cur & active;
    if (!live) continue;
    const uint8_t* Mrow = M + (size_t)r * W;
    const int x = r / dmax;
    uint32_t fail = 0u;
    for (int k = 0; k < nps; ++k) {
      const int sl = pslane[k];
      if (!((live >> sl) & 1u)) continue;
      const uint16_t* L = psl + (size_t)k * stride;
      const uint32_t* Dv = psd + (size_t)k * stride;
      const int cntk = psc[k];
      bool f = false;
      for (int c0 = 0; c0 < cntk && !f; c0 += 8) {
        uint32_t mv[8];
        int yv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          yv[u] = c0 + u < cntk ? (int)L[c0 + u] : -1;
          mv[u] = yv[u] >= 0 ? mask_at<W>(Mrow + (size_t)yv[u] * col_stride) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (yv[u] < 0) continue;
          const uint32_t d = Dv[c0 + u];
          if ((mv[u] & d) == 0u) {
            if (d != 0u || !CP || present(P, pw, x, yv[u])) f = true;
          }
        }
      }
      if (f) fail |= 1u << sl;
    }
    const uint32_t nb = cur & ~fail;
    if (nb != cur) {
      X[r] = nb;
      atomicOr(&chgn[x], cur ^ nb);
      my_or |= cur ^ nb;
    }
  }
  return my_or;
}

// Listed column GROUPS (column-group layout Mg: one 8-byte load per row gives
// the masks of the 8/W columns g*8/W ..): cgrp[k] = the group, gtst[k*CPG + j]
// = the lanes that test its column j (0: the column is not tested -- a
// warp-uniform skip).  The list is padded to a multiple of 4 with groups that
// test nothing.
template <int W, bool CP, int J>
__device__ __forceinline__ void group_col(uint32_t& acc, uint2 mv, uint32_t t, uint32_t cb, uint32_t live,
                                          const uint32_t* P, int pw, int x, int y0) {
  if (!t) return;
  constexpr int MPW = 4 / W;  // masks per 32-bit word
  const uint32_t w = (J / MPW) == 0 ? mv.x : mv.y;
  const uint32_t s = sup_lookup<W, 8 * W * (J % MPW), J * Lut<W>::TSB>(w, cb);
  apply_col<CP>(acc, s, t, live, P, pw, x, y0 + J);
}
template <int W, bool CP, int... Js>
__device__ __forceinline__ void group_cols(std::integer_sequence<int, Js...>, uint32_t& acc, uint2 mv,
                                           const uint32_t* tq, uint32_t cb, uint32_t live, const uint32_t* P,
                                           int pw, int x, int y0) {
  (group_col<W, CP, Js>(acc, mv, tq[Js], cb, live, P, pw, x, y0), ...);
}

template <int W, bool CP>
__device__ __forceinline__ uint32_t sweep_groups(const uint8_t* __restrict__ Mg, size_t gstride,
                                                 const uint32_t* __restrict__ P, int pw, uint32_t* X, uint32_t tb0,
                                                 const uint32_t* cgrp, const uint32_t* gtst, int gcnt4, int r0,
                                                 int r1, int dmax, uint32_t active, uint32_t* chgn) {
  constexpr int CPG = 8 / W;
  uint32_t my_or = 0u;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    const uint32_t cur = X[r];
    const uint32_t live = cur & active;
    if (!live) continue;
    const uint8_t* Mrow = Mg + (size_t)r * 8;
    const int x = r / dmax;
    uint32_t acc = 0xffffffffu;
    for (int g0 = 0; g0 < gcnt4 && (acc & live) != 0u; g0 += 4) {
      const uint4 g4 = *reinterpret_cast<const uint4*>(cgrp + g0);
      const uint32_t gi[4] = {g4.x, g4.y, g4.z, g4.w};
      uint2 mv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) mv[u] = __ldg(reinterpret_cast<const uint2*>(Mrow + (size_t)gi[u] * gstride));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t tq[CPG];
#pragma unroll
        for (int j = 0; j < CPG; j += 2) {
          const uint2 t2 = *reinterpret_cast<const uint2*>(gtst + (g0 + u) * CPG + j);
          tq[j] = t2.x;
          tq[j + 1] = t2.y;
        }
        group_cols<W, CP>(std::make_integer_sequence<int, CPG>{}, acc, mv[u], tq,
                          tb0 + gi[u] * (uint32_t)(CPG * Lut<W>::TSB), live, P, pw, x, (int)gi[u] * CPG);
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

// Shared memory (dynamic), byte offsets from the TSB-aligned start:
//   Tb [npad][TSB] (or the staged d_in block) | X [rows4] u32 | chg [n4] | chgn [n4] |
//   chg_in [n4] | ctst [n + 8] u32 | ci [n + 8] uint2 | gtst [(ng + 4) * 8/W] u32 |
//   cgrp [ng + 4] u32  (ng = column groups).
// Cluster rank k owns rows [k*RPC, (k+1)*RPC), RPC a multiple of dmax, so
// every variable's rows live in one CTA.
extern __shared__ __align__(16) uint8_t cl_smem[];

template <int W>
__global__ void __launch_bounds__(kMaxT, 1) rac_batch_cl(BatchCLParams p) {
  using L = Lut<W>;
  constexpr int CPI = 32 / W;
  __shared__ uint32_t s_red[2][2];             // per pass parity: this CTA's [changed lanes, emptied lanes]
  __shared__ __align__(8) uint32_t s_part[2][kMaxC][2];  // per pass parity: every CTA's partial (pushed to all)
  __shared__ __align__(8) uint64_t s_mbar;     // incoming pushes of the current pass
  __shared__ int s_cnt;
  __shared__ int s_ps;                               // this pass runs the per-state sweep (nps slots)
  __shared__ int s_psc[kPsMax], s_pslane[kPsMax];    // per slot: column count, state lane
  __shared__ uint32_t s_empty0;
  __shared__ int s_iters[32], s_status[32];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int k = (int)cluster.block_rank();
  const int g = blockIdx.x / C, G = gridDim.x / C;
  const int n = p.n, dmax = p.dmax, rows = n * dmax, rows4 = (rows + 3) & ~3;
  const int npad = (n + CPI - 1) / CPI * CPI, n4 = (n + 3) & ~3;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = T >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(cl_smem);
  const uint32_t pad = (uint32_t)(L::TSB - (base & (L::TSB - 1))) & (L::TSB - 1);
  uint8_t* Tb = cl_smem + pad;
  const uint32_t tb0 = base + pad;  // shared-memory address, TSB-aligned
  const size_t tb_bytes = max((size_t)npad * L::TSB, (size_t)32 * (n + 1) * 8);  // tables / staged d_in
  uint32_t* X = reinterpret_cast<uint32_t*>(Tb + tb_bytes);
  uint32_t* chg = X + rows4;       // pass 1's tested lanes per column (seeds / roots)
  uint32_t* chgn2 = chg + n4;      // [2][n4] my variables' changed lanes, by pass parity
  uint32_t* chg_in = chgn2 + 2 * n4;
  uint32_t* ctst = chg_in + n4;
  uint2* ci = reinterpret_cast<uint2*>(ctst + ((n + 8 + 3) & ~3));
  constexpr int CPG = 8 / W;  // columns per 8-byte group
  const int ngr = (n + CPG - 1) / CPG;
  uint32_t* gtst = reinterpret_cast<uint32_t*>(ci + ((n + 8 + 1) & ~1));          // 16-byte aligned
  uint32_t* cgrp = gtst + (((size_t)(ngr + 4) * CPG + 3) & ~(size_t)3);          // 16-byte aligned
  const bool groups = p.Mg != nullptr;
  const int ps_stride = ((n + 8) + 7) & ~7;  // per-slot list stride (u16 / u32 entries)
  uint16_t* psl = reinterpret_cast<uint16_t*>(cgrp + ((ngr + 4 + 3) & ~3));          // [kPsMax][ps_stride]
  uint32_t* psd = reinterpret_cast<uint32_t*>(psl + (size_t)kPsMax * ps_stride);    // [kPsMax][ps_stride]
  const int r0 = k * p.RPC, r1 = min(rows, r0 + p.RPC);  // my rows
  const int x0 = r0 / dmax, x1 = (r1 + dmax - 1) / dmax;  // my variables
  const bool full = (p.flags & kFullCL) != 0;
  const int NW = (p.S + 31) / 32;
  // debug stamps: per word [start, staged, per pass: prep, sweep, push, sync, control], end
  int nd = 0;
  const bool dbg = p.dbg != nullptr && k == 0 && tid == 0;
#define CL_MARK() do { if (dbg && nd < 255) p.dbg[(size_t)g * 256 + nd++] = globaltimer(); } while (0)
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  const uint32_t in_bytes = incoming_bytes(k, C, p.RPC, rows, dmax);
  uint32_t ph = 0;  // parity of the mbarrier phase of the current pass
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (C > 1) mbar_expect_tx(mbar, in_bytes);  // pass 1 of the first word
  }
  cluster.sync();  // every peer's mbarrier is initialised before anybody pushes

  for (int w = g; w < NW; w += G) {
    const int s0 = 32 * w, nst = min(32, p.S - s0);
    CL_MARK();
    // ---- the word's states -> bit slices (every CTA, all rows); lanes with an
    // empty input domain; seeds -> chg
    if (tid == 0) s_empty0 = 0u;
    for (int x = tid; x < n4; x += T) {
      chg[x] = 0u;
      chgn2[x] = 0u;
      chgn2[n4 + x] = 0u;
    }
    if (tid < 32) {
      s_iters[tid] = 0;
      s_status[tid] = 0;
    }
#if RAC_CL_GLOBAL_STAGE
    // ballots straight from global memory, RAC_CL_STAGE_IF variables in flight per
    // warp (C5: 8 variables per warp = one load round trip per word)
    __syncthreads();
    {
      uint32_t emp = 0u;
      for (int xb = warp; xb < n; xb += RAC_CL_STAGE_IF * nwarps) {
        uint64_t v[RAC_CL_STAGE_IF];
#pragma unroll
        for (int j = 0; j < RAC_CL_STAGE_IF; ++j) {
          const int x = xb + j * nwarps;
          v[j] = (x < n && lane < nst) ? __ldg(p.d_in + (size_t)(s0 + lane) * n + x) & __ldg(p.dommask + x) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < RAC_CL_STAGE_IF; ++j) {
          const int x = xb + j * nwarps;
          if (x >= n) break;
          emp |= __ballot_sync(0xffffffffu, v[j] == 0ull);
          uint32_t mine = 0u;
          for (int a = 0; a < dmax; ++a) {
            const uint32_t b = __ballot_sync(0xffffffffu, (v[j] >> a) & 1ull);
            if (lane == a) mine = b;
          }
          if (lane < dmax) X[x * dmax + lane] = mine;
        }
      }
#else
    // the word's d_in block (nst x n contiguous words) -> shared memory with
    // coalesced loads, rows padded to n + 1 words (the transposing reads below
    // then hit distinct banks); it lives in the table area, built afterwards
    uint64_t* stg = reinterpret_cast<uint64_t*>(Tb);
    {
      const uint64_t* src = p.d_in + (size_t)s0 * n;
      const int tot = nst * n;
      for (int i0 = tid; i0 < tot; i0 += 8 * T) {
        uint64_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j * T;
          v[j] = i < tot ? __ldg(src + i) & __ldg(p.dommask + (i % n)) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j * T;
          if (i < tot) stg[i + i / n] = v[j];  // row s = i / n at s * (n + 1)
        }
      }
    }
    __syncthreads();
    {
      uint32_t emp = 0u;
      for (int x = warp; x < n; x += nwarps) {
        const uint64_t v = lane < nst ? stg[(size_t)lane * (n + 1) + x] : 0ull;
        emp |= __ballot_sync(0xffffffffu, v == 0ull);
        uint32_t mine = 0u;
        for (int a = 0; a < dmax; ++a) {
          const uint32_t b = __ballot_sync(0xffffffffu, (v >> a) & 1ull);
          if (lane == a) mine = b;
        }
        if (lane < dmax) X[x * dmax + lane] = mine;
      }
#endif
      if (lane == 0 && emp) atomicOr(&s_empty0, emp);
      uint32_t rootl = 0;
      if (tid < nst) {
        const int sv = p.seed_var ? p.seed_var[s0 + tid] : -1;
        if (sv >= 0 && sv < n) atomicOr(&chg[sv], 1u << tid);
        else rootl = 1u << tid;
      }
      if (warp == 0) {
        rootl = __reduce_or_sync(0xffffffffu, rootl);
        if (lane == 0) s_cnt = (int)rootl;
      }
      __syncthreads();
      const uint32_t roots = (uint32_t)s_cnt;
      if (roots)
        for (int x = tid; x < n; x += T) chg[x] |= roots;
    }
    uint32_t active = nst >= 32 ? 0xffffffffu : ((1u << nst) - 1u);
    uint32_t E = s_empty0;  // lanes with some empty domain (cumulative)
    int t = 0;
    __syncthreads();
    CL_MARK();
    for (;;) {
      ++t;
      const int par = t & 1;
      uint32_t* chgn = chgn2 + (size_t)par * n4;               // this pass's changed lanes (my variables)
      const uint32_t* chgp = chgn2 + (size_t)(par ^ 1) * n4;   // the previous pass's
      // lanes for which y changed in the previous pass (pass 1: the seeds / roots)
      auto chgof = [&](int y) -> uint32_t { return t == 1 ? chg[y] : (y >= x0 && y < x1 ? chgp[y] : chg_in[y]); };
      // ---- prep: tst / the column list (warp 0), tables of the changed columns
      // (every column in pass 1) by the other warps
      if (tid == 0) {
        s_red[par][0] = 0u;
        s_red[par][1] = 0u;
      }
      if (warp == 0 && groups) {
        // lane = one column group: listed when one of its columns is tested
        int cnt = 0;
        for (int gb = 0; gb < ngr; gb += 32) {
          const int g = gb + lane;
          uint32_t tj[CPG], any = 0u;
#pragma unroll
          for (int j = 0; j < CPG; ++j) {
            const int y = g * CPG + j;
            tj[j] = (g < ngr && y < n) ? chgof(y) & active : 0u;
            any |= tj[j];
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, any != 0u);
          if (any) {
            const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
            cgrp[pos] = (uint32_t)g;
#pragma unroll
            for (int j = 0; j < CPG; ++j) gtst[pos * CPG + j] = tj[j];
          }
          cnt += __popc(bal);
        }
        const int cnt4 = (cnt + 3) & ~3;
        if (cnt + lane < cnt4) {  // padding: tests nothing
          cgrp[cnt + lane] = 0u;
#pragma unroll
          for (int j = 0; j < CPG; ++j) gtst[(cnt + lane) * CPG + j] = 0u;
        }
        if (lane == 0) s_cnt = cnt;
      } else if (warp == 0) {
        int cnt = 0;
        for (int yb = 0; yb < n; yb += 32) {
          const int y = yb + lane;
          const uint32_t ty = y < n ? chgof(y) & active : 0u;
          const uint32_t bal = __ballot_sync(0xffffffffu, ty != 0u);
          if (ty) {
            const int pos = cnt + __popc(bal & ((1u << lane) - 1u));
            ci[pos] = make_uint2((uint32_t)((size_t)y * p.col_stride), (uint32_t)(y * L::TSB));
            ctst[pos] = ty;
          }
          cnt += __popc(bal);
        }
        const int cnt8 = (cnt + 7) & ~7;
        if (cnt + lane < cnt8) {  // padding: tests no lane
          ci[cnt + lane] = make_uint2(0u, 0u);
          ctst[cnt + lane] = 0u;
        }
        // few active states: each one's own changed columns, and the choice of sweep
        // (per-state tests cost ~1/3 of a union-column test through the tables)
        int nps = 0;
        if (p.ps_mode && __popc(active) <= kPsMax && cnt > 0) {
          int sum = 0;
          for (uint32_t a = active; a; a &= a - 1u, ++nps) {
            const int sl = __ffs(a) - 1;
            int ck = 0;
            for (int yb = 0; yb < n; yb += 32) {
              const int y = yb + lane;
              const bool in = y < n && ((chgof(y) >> sl) & 1u);
              const uint32_t bal = __ballot_sync(0xffffffffu, in);
              if (in) psl[(size_t)nps * ps_stride + ck + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)y;
              ck += __popc(bal);
            }
            if (lane == 0) {
              s_psc[nps] = ck;
              s_pslane[nps] = sl;
            }
            sum += ck;
          }
          if (!(p.ps_mode == 2 || sum < 3 * cnt)) nps = 0;
        }
        if (lane == 0) {
          s_cnt = cnt;
          s_ps = nps;
        }
      }
      if (nwarps == 1) __syncwarp();
#if RAC_CL_ITEM_TABLES
      {
        constexpr int NI = L::TSB / 64;  // 16-entry blocks per column
        const int tb = nwarps > 1 ? tid - 32 : tid, TT = nwarps > 1 ? T - 32 : T;
        if (tb >= 0)
          for (int i = tb; i < n * NI; i += TT) {
            const int y = i / NI;
            if (t == 1 || chgof(y) != 0u) build_item<W>(Tb, X, y, i - y * NI, dmax);
          }
      }
#else
      {
        // one warp per rebuilt column (warps 1.. while warp 0 builds the list)
        const int wb = nwarps > 1 ? warp - 1 : warp, NWB = nwarps > 1 ? nwarps - 1 : nwarps;
        if (wb >= 0)
          for (int y = wb; y < n; y += NWB)
            if (t == 1 || chgof(y) != 0u) build_column<W>(Tb, X, y, dmax, lane);
      }
#endif
      __syncthreads();
      const int cnt = s_cnt;
      const int nps = groups ? 0 : s_ps;
      if (nps) {
        // D_s(y) of every listed (state, column): one warp per entry, lane b reads
        // X[(y, b)] and a ballot of bit s gives the W-bit domain
        for (int k = 0; k < nps; ++k) {
          const int ck = s_psc[k], sl = s_pslane[k];
          for (int i = warp; i < ck; i += nwarps) {
            const int y = psl[(size_t)k * ps_stride + i];
            const bool bit = lane < dmax && ((X[y * dmax + lane] >> sl) & 1u);
            const uint32_t dv = __ballot_sync(0xffffffffu, bit);
            if (lane == 0) psd[(size_t)k * ps_stride + i] = dv;
          }
        }
        __syncthreads();
      }
      // everybody's rows and my chg_in are read: peers may overwrite them once
      // they have waited on this arrival
      cluster_arrive_relaxed();
      CL_MARK();
      // ---- sweep: my rows against the tested columns
      const bool cp = (E & active) != 0u;  // some active state has an empty domain
      uint32_t my_or0;
      if (nps)
        my_or0 = cp ? sweep_states<W, true>(p.M, p.col_stride, p.P, p.pw, X, psl, psd, s_psc, s_pslane, nps,
                                            ps_stride, r0, r1, dmax, active, chgn)
                    : sweep_states<W, false>(p.M, p.col_stride, p.P, p.pw, X, psl, psd, s_psc, s_pslane, nps,
                                             ps_stride, r0, r1, dmax, active, chgn);
      else if (groups)
        my_or0 = cp ? sweep_groups<W, true>(p.Mg, p.gstride, p.P, p.pw, X, tb0, cgrp, gtst, (cnt + 3) & ~3, r0, r1,
                                            dmax, active, chgn)
                    : sweep_groups<W, false>(p.Mg, p.gstride, p.P, p.pw, X, tb0, cgrp, gtst, (cnt + 3) & ~3, r0, r1,
                                             dmax, active, chgn);
      else
        my_or0 = cp ? sweep_list<W, true>(p.M, p.P, p.pw, X, tb0, ci, ctst, (cnt + 7) & ~7, r0, r1, dmax, active, chgn)
                    : sweep_list<W, false>(p.M, p.P, p.pw, X, tb0, ci, ctst, (cnt + 7) & ~7, r0, r1, dmax, active, chgn);
      const uint32_t my_or = __reduce_or_sync(0xffffffffu, my_or0);
      if (lane == 0 && my_or) atomicOr(&s_red[par][0], my_or);
      __syncthreads();  // my rows and change masks are final
      {
        // lanes in which one of my variables became empty (only changed ones can)
        uint32_t emp = 0u;
        for (int x = x0 + tid; x < x1; x += T) {
          if (!chgn[x]) continue;
          uint32_t ne = 0u;
          for (int a = 0; a < dmax; ++a) ne |= X[x * dmax + a];
          emp |= ~ne;
        }
        emp = __reduce_or_sync(0xffffffffu, emp);
        if (lane == 0 && emp) atomicOr(&s_red[par][1], emp);
      }
      __syncthreads();
      CL_MARK();
      // ---- push: wait until every CTA has read the old rows, then store my
      // rows, my change masks and my partial into every other CTA (fixed sizes:
      // each peer's mbarrier expects exactly these bytes)
      cluster_wait();
      for (int x = x0 + tid; x < x1; x += T) chgn2[(size_t)(par ^ 1) * n4 + x] = 0u;  // read by this pass's prep only
      if (C > 1) {
        // same layout in every CTA: the peer address is mapa(local address, q)
        const uint32_t xs = (uint32_t)__cvta_generic_to_shared(X + r0), cs = (uint32_t)__cvta_generic_to_shared(chg_in);
        const uint32_t ps = (uint32_t)__cvta_generic_to_shared(&s_part[par][k][0]);
        const int nv4 = (r1 - r0 + 3) / 4;
        for (int q = 0; q < C; ++q) {
          if (q == k) continue;
          const uint32_t bq = mapa(mbar, (uint32_t)q);
          for (int i = tid; i < nv4; i += T)
            st_async_v4(mapa(xs + 16u * (uint32_t)i, (uint32_t)q), *reinterpret_cast<const uint4*>(X + r0 + 4 * i), bq);
          for (int x = x0 + tid; x < x1; x += T) st_async_b32(mapa(cs + 4u * (uint32_t)x, (uint32_t)q), chgn[x], bq);
          if (tid == 0) st_async_v2(mapa(ps, (uint32_t)q), s_red[par][0], s_red[par][1], bq);
        }
      }
      if (tid == 0) {
        s_part[par][k][0] = s_red[par][0];
        s_part[par][k][1] = s_red[par][1];
      }
      CL_MARK();
      if (C > 1) mbar_wait(mbar, ph);
      ph ^= 1u;
      __syncthreads();  // s_part[par][k] (own slot) for everybody
      // the next pass's incoming bytes (peers push them only after my next arrival)
      if (C > 1 && tid == 0) mbar_expect_tx(mbar, in_bytes);
      CL_MARK();
      // ---- per-state loop control (Alg. 1): wipeout first, then "changed"
      uint32_t changed = 0u;
      for (int q = 0; q < C; ++q) {
        changed |= s_part[par][q][0];
        E |= s_part[par][q][1];
      }
      const uint32_t stop_wipe = full ? 0u : (E & active);
      const uint32_t stop_conv = ~changed & active & ~stop_wipe;
      if (tid < 32) {
        const uint32_t bit = 1u << tid;
        if (active & bit) s_iters[tid] = t;
        if (stop_wipe & bit) s_status[tid] = 1;
        if (stop_conv & bit) s_status[tid] = (E & bit) ? 1 : 0;
      }
      active &= ~(stop_wipe | stop_conv);
      // (the next pass's prep reads the change masks in place -- mine from chgn,
      // the others' from chg_in -- so no copy and no block barrier here)
      CL_MARK();
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
  const int TSB = W == 1 ? Lut<1>::TSB : W == 2 ? Lut<2>::TSB : Lut<4>::TSB;
  const size_t CPI = 32 / W;
  const size_t npad = (n + CPI - 1) / CPI * CPI, n4 = ((size_t)n + 3) & ~(size_t)3;
  const size_t rows4 = (((size_t)n * dmax) + 3) & ~(size_t)3;
  const size_t tb_bytes = std::max(npad * TSB, (size_t)32 * (n + 1) * 8);  // tables, or the staged d_in block
  return (size_t)TSB + tb_bytes + rows4 * 4 + 4 * n4 * 4 + ((((size_t)n + 8 + 3) & ~(size_t)3) * 4) +
         (((size_t)n + 8 + 1) & ~(size_t)1) * 8 +
         ((((size_t)n + 8 / W - 1) / (8 / W) + 4) * (8 / W) + 3) / 4 * 16 +
         ((((size_t)n + 8 / W - 1) / (8 / W) + 4 + 3) & ~(size_t)3) * 4 +
         (size_t)kPsMax * ((((size_t)n + 8) + 7) & ~(size_t)7) * 6 + 16;
}

// Column groups for the batched sweep: Mg[g][r] = the 8 bytes of masks of columns
// g*8/W .. g*8/W + 8/W - 1 at row r (columns >= n: all ones -- never tested).
__global__ void pack_groups_kernel(const uint8_t* __restrict__ M, size_t col_stride, int n, int W, int rows_pad,
                                   uint8_t* __restrict__ Mg) {
  const int cpg = 8 / W, ngr = (n + cpg - 1) / cpg;
  const size_t total = (size_t)ngr * rows_pad;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / rows_pad), r = (int)(i - (size_t)g * rows_pad);
    uint8_t b[8];
    for (int j = 0; j < cpg; ++j) {
      const int y = g * cpg + j;
      for (int k = 0; k < W; ++k) b[j * W + k] = y < n ? M[(size_t)y * col_stride + (size_t)r * W + k] : 0xFF;
    }
    uint2 v;
    v.x = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
    v.y = (uint32_t)b[4] | ((uint32_t)b[5] << 8) | ((uint32_t)b[6] << 16) | ((uint32_t)b[7] << 24);
    *reinterpret_cast<uint2*>(Mg + i * 8) = v;
  }
}

cudaError_t launch_pack_groups(const uint8_t* M, size_t col_stride, int n, int W, int rows_pad, uint8_t* Mg,
                               cudaStream_t s) {
  if (W != 1 && W != 2 && W != 4) return cudaErrorInvalidValue;
  const int cpg = 8 / W;
  const size_t total = (size_t)((n + cpg - 1) / cpg) * rows_pad;
  const int blocks = (int)std::min<size_t>(4096, (total + 255) / 256);
  pack_groups_kernel<<<blocks, 256, 0, s>>>(M, col_stride, n, W, rows_pad, Mg);
  return cudaGetLastError();
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
  if (C > kMaxC) return cudaErrorInvalidValue;
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
  if (C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
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
