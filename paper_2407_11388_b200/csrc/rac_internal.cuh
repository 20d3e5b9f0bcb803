// rac_internal.cuh -- internal declarations and device helpers of librac (sm_100a).
//
// Data layout in HBM:
//   W          bytes per support mask: 1, 2, 4 or 8 (smallest >= max dom bits).
//   rows       local rows (x,a): r = (x - x_lo)*dmax + a, padded to a multiple of
//              kSlabRows(W) = 32 lanes x 16/W rows (one warp-wide 512-byte slab).
//   M          COLUMN-major: column y (every variable y = 0..n-1) is a contiguous
//              array of `rows` W-byte masks, M + y*col_stride + r*W holds
//              c_xy|(x,a) as a d_y-bit set.  Absent pairs and
//              y == x hold all-ones; padding rows hold 0xFF.  Reading the columns
//              of the changed variables is Alg. 1's Cons[:, @changed] gather
//               as contiguous streams.
//   Mr         optional ROW-major copy: row r = n W-byte masks M[(x,a)][y], padded
//              to dbytes (16-byte multiple, 0xFF); a full pass over the live rows
//              streams whole rows with per-row early exit and dead-row skip.
//              Each pass picks the layout that reads fewer bytes (live rows x n
//              vs all rows x changed columns).
//   P          presence bitmap, [local x][pw = ceil(n/32)] u32; bit y of
//              variable x set iff c_xy is declared (C_x).
//   D (smem)   the alive bitvector D_t, variable y at bytes [y*W, y*W+W),
//              padded to 16 bytes (dbytes).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace rac {

#ifndef RAC_THREADS
#define RAC_THREADS 512
#endif
constexpr int kThreads = RAC_THREADS;  // CTA size of the support-pass kernels
#ifndef RAC_MIN_BLOCKS
#define RAC_MIN_BLOCKS 1
#endif
constexpr int kMinBlocks = RAC_MIN_BLOCKS;  // CTAs per SM the register budget is sized for
#ifndef RAC_UNROLL_C
#define RAC_UNROLL_C 8
#endif
constexpr int kUnroll = RAC_UNROLL_C;   // 16-byte loads in flight per lane (column sweep)
#ifndef RAC_UNROLL_S
#define RAC_UNROLL_S 16
#endif
constexpr int kUnrollS = RAC_UNROLL_S;  // 16-byte loads in flight per lane (sparse arc-block sweep)
#ifndef RAC_UNROLL_R
#define RAC_UNROLL_R 8
#endif
constexpr int kUnrollR = RAC_UNROLL_R;  // 16-byte row loads in flight per lane (row-major sweep)

__host__ __device__ constexpr int slab_rows(int W) { return 32 * (16 / W); }

// ---------------------------------------------------------------------------- params
struct PassGeom {
  const uint8_t* M;       // column-major masks of the local rows
  size_t col_stride;      // bytes per column = rows_pad * W
  const uint8_t* Mr;      // nullable: row-major copy (row stride dbytes)
  int force;              // 0 = pick per pass, 1 = rows, 2 = columns (testing knob)
  int n;                  // variables (= columns)
  int dmax;               // rows per variable
  int x_lo, x_hi;         // rows of variables [x_lo, x_hi) are tested
  int x_lo_alloc;         // first variable of the local row block
  const uint32_t* P;      // presence bits of variable x_lo_alloc onward
  int pw;                 // u32 words per presence row
  int dbytes;             // bytes of D in smem (n*W rounded up to 16)
  // Sparse arc-block layout (S != nullptr; NEXT-3): only declared arcs are
  // stored.  Block b = the dpad masks c_xy|(x,a), a < dpad, of one arc x -> y
  // (16-byte multiple); the blocks of column y are contiguous (Cons[:, y] of
  // Alg. 1), columns in order.
  const uint8_t* S;
  const uint32_t* s_off;  // [n+1] first block of column y
  const uint32_t* s_arc;  // [nblk] x | y << 16
  const uint32_t* s_ipref;  // [n+1] work items of columns 0..y-1 (full-pass item prefix)
  uint32_t s_nblk;        // blocks (local arcs)
  int s_vb;               // 16-byte vectors per block
};

// Peer-memory exchange of the row-sharded fused kernel (world > 1, RAC_OPT_PEER):
// after each pass a rank writes the removal words of its own rows into every
// peer's removal buffer (NVLink P2P stores), so after the cross-rank barrier
// each rank holds the complete R of the pass.  Entries of self are NULL.
constexpr int kMaxRanks = 8;
struct Mirror {
  int world, rank;
  int n;                               // words per removal buffer
  unsigned long long* R[kMaxRanks];    // peer q's R[3][n]
  unsigned* flag[kMaxRanks];           // peer q's per-pass removal flags [3]
};

// Removal epochs mirrored to the peers (peer path with removed_at): an epoch
// written for a local row is also stored into every peer's epoch array of the
// call, so after the last cross-rank barrier every rank holds all epochs.
struct EpochMirror {
  int world, rank;
  int32_t* E[kMaxRanks];  // peer q's epoch array of this call (NULL for self)
};

__device__ __forceinline__ void put_epoch(int32_t* ra, const EpochMirror* em, size_t i, int t) {
  ra[i] = t;
  if (em)
    for (int q = 0; q < em->world; ++q)
      if (q != em->rank) em->E[q][i] = t;
}

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
  unsigned* wctr;           // [3] per-pass dynamic row counters (rotating like R)
  unsigned* rflag;          // [3] per-pass "some value was removed" flags (rotating like R)
  uint32_t* clist;          // nullable [3][n+1] per-pass change lists ([0] = count; rotating like R)
  const int32_t* seeds;     // device [n_seeds]: Alg. 1 initial @changed (read only if n_seeds > 0)
  int n_seeds;              // < 0: root call (every column in pass 1); 0: no pass
  uint32_t flags;
  uint32_t ab;              // A/B knobs (tooling, RAC_FUSED_AB): bit 0 legacy grid barrier, bit 1 listed apply, bit 2 no removal-flag check before the R read
  int list_max;             // dense layout: passes testing <= list_max columns keep a change list (apply reads only its R words, no compaction)
  int row_agg;              // dense: the row sweep ORs removals into a per-CTA copy of R in shared memory (after the
                            // fused_smem region, n words) and flushes one atomic per (CTA, variable)
  unsigned* cctr;           // nullable [3][32 parts][32]: partitioned tail-claim counters of the column sweep (RAC_COL_CLAIM == 2 builds)
  unsigned long long* dbg;  // nullable: phase timestamps of CTA 0 (RAC_DEBUG_TIMELINE)
  // Global pass counter (persists across launches): pass t of this launch is
  // pass *seq + t; it selects the rotating buffers and is the cross-rank
  // barrier's sequence number.
  unsigned long long* seq;
  // world > 1 (peer exchange) only:
  Mirror mir;
  unsigned long long* arrive;                  // own arrival words [kMaxRanks] (written by peers)
  unsigned long long* peer_arrive[kMaxRanks];  // peer q's arrival words (NULL for self)
  unsigned long long timeout_ns;               // give up waiting for a peer after this long
  int32_t* xerr;                               // set to 1 on a peer timeout
  // world > 1 with removed_at: epoch arrays [2][n*64] in every rank's exchange
  // region (double-buffered by the parity of *calls, the count of such calls)
  int32_t* E;                                  // own
  int32_t* Epeer[kMaxRanks];                   // peer q's (NULL for self)
  unsigned long long* calls;
};

struct ShardState {
  uint64_t* Dcur;            // [n] current D_t (u64 per variable)
  uint64_t* Dg;              // [world*blk] gathered D_{t+1}
  uint8_t* Dw;               // [dbytes] D_t in the W-byte smem layout (TMA source)
  unsigned long long* R;     // [n] removal masks of the current pass
  int32_t* iters;            // device scalars
  int32_t* status;
  int32_t* done;
  int32_t* vcnt;             // length of vlist (variables changed in the last pass)
  int32_t* seeded;           // 1: pass 1 tests vlist (a seeded call), 0: every column
  uint16_t* vlist;           // [n] Prop. 2 incremental column list
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
  int32_t* removed_at;      // nullable, single-state launches only: [n*64] removal epochs (pre-zeroed)
  uint32_t flags;
};

// rac_state (rac_state.cu): one block per domain state.
struct StateParams {
  const uint8_t* M;         // column-major masks (all rows of the instance)
  size_t col_stride;        // bytes per column
  int n, dmax;
  const uint32_t* P;        // presence bitmap [n][pw]
  int pw;
  const uint64_t* dommask;  // [n]
  const uint64_t* d_in;     // [.][n] states (state s0 + blockIdx.x)
  uint64_t* d_out;
  int32_t* iters;
  int32_t* status;
  const int32_t* seed_var;  // nullable [.]: per-state seed variable (-1 = all)
  const int32_t* seeds;     // single-state seeded call: device [n_seeds] (read if n_seeds > 0)
  int n_seeds;              // < 0: not a seed-list call; 0: empty @changed (no pass)
  int32_t* removed_at;      // nullable (single-state launches): [n*64], pre-zeroed
  uint32_t flags;
  int s0;                   // first state of this launch in the caller's arrays
  int nvec;                 // 16-byte vectors per column
  uint32_t off_R, off_live, off_vx, off_list, off_nlist, off_P, off_M;  // shared-memory layout (state_layout)
  unsigned long long* dbg;  // nullable: phase stamps of block 0 (RAC_DEBUG_TIMELINE)
};
// Offsets of rac_state's shared memory; P staged if <= p_cap bytes, the whole
// mask tensor if <= m_cap bytes (0 = not staged).  Returns the total bytes.
size_t state_layout(StateParams& p, int n, int dmax, int W, int rows_pad, int pw, size_t p_cap, size_t m_cap);
cudaError_t launch_state(int W, int T, const StateParams& p, int n_states, size_t smem, cudaStream_t s);
// rac_tiny: one warp per state for n <= 64 (the mask tensor in shared memory)
size_t tiny_smem(int n, size_t col_stride);
cudaError_t launch_tiny(int W, const StateParams& p, int n_states, size_t smem, cudaStream_t s);
// Blocking calls: copy the pinned host staging (d_in | seeds) into device memory
// with one small kernel reading host memory (instead of a copy-engine transfer).
cudaError_t launch_stage_copy(const void* host_src, void* dev_dst, size_t bytes, cudaStream_t s);

// rac_batch_cl (rac_batch_cl.cu): one 32-state bit-sliced word per cluster.
struct BatchCLParams {
  const uint8_t* M;         // column-major masks
  size_t col_stride;
  const uint8_t* Mg;        // nullable: 8-byte column groups, Mg + g*gstride + r*8 = masks of columns g*8/W.. of row r
  size_t gstride;
  int ps_mode;              // 0: union sweep only; 1: per-state sweep when <= 8 states are active and cheaper; 2: always when <= 8
  int n, dmax;
  const uint32_t* P;
  int pw;
  const uint64_t* dommask;
  const uint64_t* d_in;     // [S][n]
  uint64_t* d_out;
  int32_t* iters;           // [S]
  int32_t* status;          // [S]
  const int32_t* seed_var;  // nullable [S]
  int S;
  int RPC;                  // rows per CTA of a cluster (a multiple of dmax)
  uint32_t flags;
  unsigned long long* dbg;  // nullable (RAC_DEBUG_TIMELINE): [clusters][256] %globaltimer stamps
};
// CTA size cap of rac_batch_cl: 800 threads = 25 warps, so ptxas may use 80
// registers (the software-pipelined sweep needs ~70; at 1024 threads it spilled).
constexpr int kBatchClThreads = 800;
size_t batch_cl_smem(int n, int dmax, int W);
cudaError_t launch_pack_groups(const uint8_t* M, size_t col_stride, int n, int W, int rows_pad, uint8_t* Mg,
                               cudaStream_t s);
cudaError_t launch_batch_cl(int W, const BatchCLParams& p, int clusters, int C, int threads, size_t smem,
                            cudaStream_t s);
cudaError_t batch_cl_max_clusters(int W, int C, int threads, size_t smem, int* out);

struct BatchBSParams {
  const uint8_t* M;
  size_t col_stride;
  const uint8_t* Mr;        // nullable row-major copy (row stride row_bytes)
  int row_bytes;
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
  unsigned long long* dbg;  // nullable: [grid][64] per-CTA pass-end timestamps (RAC_DEBUG_TIMELINE)
};

struct TcPassParams {
  const uint8_t* M;        // column-major masks
  size_t col_stride;
  int W;
  int n, dmax, rows;
  const uint32_t* P;
  int pw;
  const uint32_t* Xin;     // [NW][rows4] state bit slices
  uint32_t* Xout;          // [NW][rows4]
  int rows4, NW;
};

// Dynamic smem of rac_fused / rac_pass / rac_batch: D (dbytes), then the
// incremental column list (u16[n]) and the per-variable "changed" flags (u8[n]).
__host__ __device__ constexpr size_t list_offset(int dbytes) { return (size_t)dbytes; }
__host__ __device__ constexpr size_t need_offset(int dbytes, int n) {
  return (size_t)dbytes + (((size_t)n * 2 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t fused_smem(int dbytes, int n) {
  return need_offset(dbytes, n) + (((size_t)n + 15) & ~(size_t)15);
}
// Sparse layout: + the work-item prefix over the tested columns (u32[n+1]).
__host__ __device__ constexpr size_t pref_offset(int dbytes, int n) { return fused_smem(dbytes, n); }
__host__ __device__ constexpr size_t sparse_smem(int dbytes, int n) {
  return pref_offset(dbytes, n) + (((size_t)(n + 1) * 4 + 15) & ~(size_t)15);
}

// ---------------------------------------------------------------------------- host launchers
// (defined in rac_kernels.cu / rac_pack.cu; return cudaError_t of the launch)
int choose_group(int nvec);  // lanes per row of the row-major sweep
cudaError_t launch_fused(int W, int G, const FusedParams& p, int grid, size_t smem, cudaStream_t s, bool cooperative);
cudaError_t fused_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
cudaError_t launch_pass(int W, int G, const PassParams& p, int grid, size_t smem, cudaStream_t s);
cudaError_t pass_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
cudaError_t launch_shard_init(const ShardState& s, const uint64_t* d_in, const uint64_t* dommask, int n, int W,
                              int dbytes, int total_g, cudaStream_t st);
cudaError_t launch_shard_seed(const ShardState& s, const int32_t* seeds, int n_seeds, int n, cudaStream_t st);
cudaError_t launch_shard_slice(const ShardState& s, int x_lo, int x_hi, int n, cudaStream_t st);
cudaError_t launch_shard_update(const ShardState& s, int n, int W, uint32_t flags, cudaStream_t st);
cudaError_t launch_shard_finalize(const ShardState& s, int n, uint64_t* d_out, int32_t* iters, int32_t* status,
                                  cudaStream_t st);
cudaError_t launch_batch(int W, int G, const BatchParams& p, int n_states, size_t smem, cudaStream_t s);
cudaError_t batch_occupancy(int W, int G, size_t smem, int* blocks_per_sm);
size_t batch_bs_smem(int n, int dmax, int W, bool use_table);
struct TcPassParams;
cudaError_t launch_batch_pass_eval(int impl, const TcPassParams& p, const uint64_t* d_in, const uint64_t* dommask,
                                   int S, uint64_t* d_out, cudaStream_t st);
cudaError_t batch_bs_occupancy(int W, size_t smem, int* blocks_per_sm);
cudaError_t launch_batch_bs(int W, const BatchBSParams& p, int grid, size_t smem, cudaStream_t s);

struct PackGeom {
  uint8_t* M;             // column-major masks of the local rows
  size_t col_stride;
  uint8_t* Mr;            // nullable row-major copy
  size_t row_bytes;       // = dbytes
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
// Sparse arc-block packer: pair r = (xs[r], ys[r]) (x < y for generated
// instances); its forward masks c_xy|(x,a) go to block fwd[r], the transposed
// masks c_yx|(y,b) to block bwd[r] (either may be UINT32_MAX: not local).
// rows == nullptr: rows come from the seeded generator (d, t_q16, seed).
struct SparsePack {
  uint8_t* S;
  int bbytes;             // bytes per block
  int W;
  const int32_t* dom;     // device [n]
  int n;
};
cudaError_t launch_pack_sparse(const SparsePack& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                               int row_words, const uint32_t* fwd, const uint32_t* bwd, long n_pairs, int d,
                               uint32_t t_q16, uint64_t seed, cudaStream_t s);

// ---------------------------------------------------------------------------- wide domains (rac_wide.cu)
// NEXT-4: 65..256 values.  Masks WS = 2 or 4 words per (x,a,y), row-major
// M[((x*dmax + a)*n + y)*WS]; boundary domain states n x wq words, wq = ceil(dmax/64).
struct WideParams {
  const uint64_t* M;
  const uint32_t* P;       // presence bitmap [n][pw]
  const int32_t* dom;      // device [n]
  int n, dmax, wq, WS, pw;
  int full;                // RAC_FULL_FIXPOINT
  const uint64_t* d_in;    // [n * wq]
  uint64_t* d_out;         // [n * wq]
  uint64_t* D;             // [n * WS] current state
  uint64_t* R;             // [n * WS] removal bits of the pass
  uint32_t* clist;         // [3][n] change lists
  unsigned* slots;         // [3][2] {count, wipe}
  int32_t* removed_at;     // nullable [n * 64 * wq]
  int32_t* iters;
  int32_t* status;
  const int32_t* seeds;    // device [n_seeds], each in [0, n) (seeded calls)
  int n_seeds;             // -1: unseeded (pass 1 tests every column)
};
struct WidePack {
  uint64_t* M;
  uint32_t* P;
  const int32_t* dom;      // device [n]
  int n, dmax, wq, WS, pw;
  uint64_t dens_q32;
};
struct WideStateParams {  // wide_state: one block per domain state
  const uint64_t* M;
  const uint32_t* P;
  const int32_t* dom;
  int n, dmax, wq, WS, pw;
  int full;
  const uint64_t* d_in;     // [S][n * wq]
  uint64_t* d_out;
  int32_t* iters;
  int32_t* status;
  const int32_t* seed_var;  // nullable [S]
  int s0;                   // first state of this launch
};
// rac_wide_tc.cu: one batched pass on wide domains, bit-sliced (impl 2) or
// tcgen05 (impl 3, d <= 128), for the A/B of rac_batch_pass_eval.
struct WideTcParams {
  const uint64_t* M;        // wide row-major masks
  const uint32_t* P;
  int pw;
  const int32_t* dom;       // device [n]
  int n, dmax, wq, WS;
  int S;                    // states
  const uint64_t* d_in;     // [S][n * wq]
  uint64_t* d_out;          // [S][n * wq]
  const uint32_t* Xin;      // [NW][rows4] state slices (impl 2)
  uint32_t* Xout;           // [NW][rows4] rows kept per state
  int rows4, NW;
};
cudaError_t launch_wide_pass_eval(int impl, const WideTcParams& p, cudaStream_t st);
cudaError_t launch_fill_i32(int32_t* p, int32_t v, int n, cudaStream_t st);
cudaError_t launch_wide_mask_copy(const uint64_t* d_in, const int32_t* dom, int S, int n, int wq, uint64_t* Dc,
                                  cudaStream_t st);
cudaError_t launch_wide_tc_update(const int32_t* dom, int n, int wq, int full, uint64_t* Dc, const uint64_t* Dn,
                                  int32_t* active, int32_t* iters, int32_t* status, int32_t* n_active, int S,
                                  cudaStream_t st);
size_t wide_state_smem(int n, int WS);
cudaError_t launch_wide_state(const WideStateParams& p, int n_states, cudaStream_t s);
cudaError_t wide_fused_grid(int WS, size_t smem, int sm_count, int* grid);
cudaError_t launch_wide_fused(const WideParams& p, int grid, size_t smem, cudaStream_t s);
// rows: [n_rel][dmax][wq] (row a of rel(c_{xs[r] ys[r]}))
cudaError_t launch_wide_pack(const WidePack& g, const int32_t* xs, const int32_t* ys, const uint64_t* rows,
                             int n_rel, cudaStream_t s);
cudaError_t launch_wide_generate(const WidePack& g, int d, uint32_t t_q16, uint64_t seed, cudaStream_t s);

// ---------------------------------------------------------------------------- device helpers
#ifdef __CUDACC__

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
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

// D(y) replicated over the 16/W lanes of a 16-byte vector.
template <int W>
__device__ __forceinline__ uint4 rep16(uint64_t d) {
  if constexpr (W == 8) {
    const uint32_t lo = (uint32_t)d, hi = (uint32_t)(d >> 32);
    return make_uint4(lo, hi, lo, hi);
  } else {
    uint32_t v = (uint32_t)d;
    if constexpr (W == 2) v = v | (v << 16);
    if constexpr (W == 1) v = v * 0x01010101u;
    return make_uint4(v, v, v, v);
  }
}

// Bit i set iff the i-th W-byte lane of t is zero (16/W lanes).
template <int W>
__device__ __forceinline__ uint32_t zero_lanes(uint4 t) {
  if constexpr (W == 8) {
    return (uint32_t)((t.x | t.y) == 0u) | ((uint32_t)((t.z | t.w) == 0u) << 1);
  } else if constexpr (W == 4) {
    return (uint32_t)(t.x == 0u) | ((uint32_t)(t.y == 0u) << 1) | ((uint32_t)(t.z == 0u) << 2) |
           ((uint32_t)(t.w == 0u) << 3);
  } else if constexpr (W == 2) {
    const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = __vcmpeq2(w4[k], 0u);
      m |= ((c & 1u) | ((c >> 15) & 2u)) << (2 * k);
    }
    return m;
  } else {
    const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = __vcmpeq4(w4[k], 0u);
      m |= ((c & 1u) | ((c >> 7) & 2u) | ((c >> 14) & 4u) | ((c >> 21) & 8u)) << (4 * k);
    }
    return m;
  }
}

// Support test of column y for the 16/W rows r0.. of one lane against D(y):
// returns the rows (bits) among `cand` that lose support, i.e. whose mask &
// D(y) == 0 (Eq. 1 condition, intersection form of line
// 59) -- but only on a declared c_xy (reading R2): absent pairs store
// all-ones, so they can only "fail" when D(y) is empty, and then P decides.
template <int W>
__device__ __forceinline__ uint32_t column_fail(uint4 m, uint64_t d, uint32_t cand, int y, int r0, int dmax,
                                                const uint32_t* P, int pw) {
  const uint32_t z = zero_lanes<W>(and4(m, rep16<W>(d))) & cand;
  if (z == 0u || d != 0ull) return z;
  uint32_t f = 0;
  for (uint32_t zz = z; zz; zz &= zz - 1u) {
    const int i = __ffs(zz) - 1;
    const int xl = (r0 + i) / dmax;  // local variable of row r0+i
    if ((P[(size_t)xl * pw + (y >> 5)] >> (y & 31)) & 1u) f |= 1u << i;
  }
  return f;
}

// column_fail with the AND already taken (t = mask & D(y) over the 16/W rows):
// the rows among `cand` whose test failed on a declared c_xy.
template <int W>
__device__ __forceinline__ uint32_t column_fail_t(uint4 t, uint64_t d, uint32_t cand, int y, int r0, int dmax,
                                                  const uint32_t* P, int pw) {
  const uint32_t z = zero_lanes<W>(t) & cand;
  if (z == 0u || d != 0ull) return z;
  uint32_t f = 0;
  for (uint32_t zz = z; zz; zz &= zz - 1u) {
    const int i = __ffs(zz) - 1;
    const int xl = (r0 + i) / dmax;
    if ((P[(size_t)xl * pw + (y >> 5)] >> (y & 31)) & 1u) f |= 1u << i;
  }
  return f;
}

// ---- row-major sweep helpers
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

// A 16-byte vector v of row (x,a) had some mask & D == 0: is it a real loss of
// support?  Only on a declared c_xy (reading R2); padding lanes never fail.
template <int W>
__device__ __noinline__ bool vec_real_fail(uint4 m, uint4 d, int v, int n, const uint32_t* Prow) {
  constexpr int L = 16 / W;
  const uint32_t mw[4] = {m.x, m.y, m.z, m.w}, dw[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
  for (int i = 0; i < L; ++i) {
    const int y = v * L + i;
    if (y >= n) break;
    uint64_t mi, di;
    if constexpr (W == 8) {
      mi = (uint64_t)mw[2 * i] | ((uint64_t)mw[2 * i + 1] << 32);
      di = (uint64_t)dw[2 * i] | ((uint64_t)dw[2 * i + 1] << 32);
    } else {
      const int sh = (8 * W * i) & 31, k = (W * i) >> 2;
      const uint32_t msk = W == 4 ? 0xffffffffu : ((1u << (8 * W)) - 1u);
      mi = (mw[k] >> sh) & msk;
      di = (dw[k] >> sh) & msk;
    }
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

// Support test of one (x,a) row segment [vb, ve) (16-byte vectors) against D
// in smem: true iff some declared c_xy has c_xy|(x,a) ∩ D(y) = ∅ (Eq. 1
// condition).  G lanes cooperate, kUnrollR loads per lane in flight, early exit.
template <int W, int G>
__device__ __forceinline__ bool row_fails(const uint4* __restrict__ row, const uint4* Ds, int vb, int ve, int gl,
                                          unsigned gmask, int n, const uint32_t* Prow) {
  bool fail = false;
  for (int v0 = vb; v0 < ve; v0 += G * kUnrollR) {
    uint4 m[kUnrollR];
#pragma unroll
    for (int u = 0; u < kUnrollR; ++u) {
      const int v = v0 + u * G + gl;
      if (v < ve) m[u] = ldg_stream(row + v);
    }
#pragma unroll
    for (int u = 0; u < kUnrollR; ++u) {
      const int v = v0 + u * G + gl;
      if (v < ve) {
        const uint4 d = Ds[v];
        if (vec_any_zero<W>(and4(m[u], d))) fail |= vec_real_fail<W>(m[u], d, v, n, Prow);
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

// Block-wide inclusive scan of one u32 per thread (every thread gets its
// exclusive prefix and the total).
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t c, uint32_t* total, int* scratch) {
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t v = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  __syncthreads();  // scratch may still be read by a previous helper
  if (lane == 31) scratch[w] = (int)v;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < (T >> 5) ? (uint32_t)scratch[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    if (lane < (T >> 5)) scratch[lane] = (int)s;
  }
  __syncthreads();
  const uint32_t excl = v - c + (w > 0 ? (uint32_t)scratch[w - 1] : 0u);
  *total = (uint32_t)scratch[(T >> 5) - 1];
  __syncthreads();
  return excl;
}

// Sparse layout, listed columns: choose the vectors per lane per item `upl`
// (U, fewer when the pass is too small to give every warp an item) and write
// ipref[i] = work items of list[0..i) (column y has ceil((s_off[y+1] -
// s_off[y]) * VB / (32 upl)) items), ipref[cnt] = total.  Block-wide; every
// CTA computes it redundantly from its own list.  Returns upl.
__device__ __forceinline__ uint32_t block_prefix_items(const uint16_t* list, int cnt, const uint32_t* s_off,
                                                       uint32_t VB, uint32_t U, long nwarps, uint32_t* ipref,
                                                       int* scratch) {
  const int T = blockDim.x, t = threadIdx.x;
  const int chunk = (cnt + T - 1) / T;
  const int b = min(cnt, t * chunk), e = min(cnt, b + chunk);
  uint32_t c = 0;
  for (int i = b; i < e; ++i) c += __ldg(s_off + list[i] + 1) - __ldg(s_off + list[i]);
  uint32_t tot_blocks;
  block_scan_u32(c, &tot_blocks, scratch);
  const uint64_t upl64 = (uint64_t)tot_blocks * VB / (32ull * (uint64_t)nwarps);
  const uint32_t upl = upl64 < 1 ? 1u : (upl64 > U ? U : (uint32_t)upl64);
  const uint32_t per_item = 32u * upl;
  auto items_of = [&](int i) {
    const int y = list[i];
    return ((__ldg(s_off + y + 1) - __ldg(s_off + y)) * VB + per_item - 1u) / per_item;
  };
  c = 0;
  for (int i = b; i < e; ++i) c += items_of(i);
  uint32_t total;
  uint32_t pos = block_scan_u32(c, &total, scratch);
  for (int i = b; i < e; ++i) {
    ipref[i] = pos;
    pos += items_of(i);
  }
  if (t == 0) ipref[cnt] = total;
  __syncthreads();
  return upl;
}

__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mb)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// One elected lane: arm `mb` for `bytes` and start `cnt` 512-byte bulk copies.
__device__ __forceinline__ void bulk_arm(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy_512(void* dst, const void* src, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"((uint32_t)__cvta_generic_to_shared(mb))
      : "memory");
}

// Stage `bytes` (a multiple of 16, both addresses 16-byte aligned) from global
// into shared memory with bulk copies (TMA engine): thread 0 initialises the
// mbarrier, arms it with the byte count and issues <= 32 KB copies; every
// thread then calls bulk_stage_wait (phase 0).  The mbarrier must not be
// reused within the launch.
__device__ __forceinline__ void bulk_stage_start(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mb);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes) : "memory");
    const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst);
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t sz = bytes - off < 32768u ? bytes - off : 32768u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d0 + off),
          "l"(static_cast<const uint8_t*>(src) + off), "r"(sz), "r"(m)
          : "memory");
    }
  }
}
__device__ __forceinline__ void bulk_stage_wait(uint64_t* mb) {
  __syncwarp();
  // thread 0 initialised the barrier before any thread can observe phase 0 complete
  if (blockDim.x > 32) __syncthreads();
  mbar_wait(mb, 0);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin-wait loads: relaxed (an acquire load invalidates the SM's L1 on every
// poll -- CCTL.IVALL in the SASS -- which evicted the L1-cached operands of the
// other CTAs sharing the SM); the fence after the loop gives the acquire.
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_release_add_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Software grid barrier for a co-resident (cooperative) grid.  bar[0] counts
// arrivals over the whole launch.  Each CTA arrives with a release reduction
// (no return value, no separate fence) and polls the counter itself until all
// nblocks * epoch arrivals are in (relaxed polls, one fence after: an acquire
// load per poll would invalidate the SM's L1 every time), so the release does
// not wait for a last arriver to publish a flag.  legacy != 0: the previous
// form (fenced atomicAdd; the last arriver releases bar[1]) for A/B runs.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned epoch, int legacy = 0) {
  if (!legacy) {
    __syncthreads();
    if (nblocks > 1 && threadIdx.x == 0) {
      red_release_add_gpu(&bar[0], 1u);
      const unsigned target = nblocks * epoch;
      while (ld_relaxed_gpu(&bar[0]) < target) {
      }
      __threadfence();
    }
    __syncthreads();
    return;
  }
  __syncthreads();
  if (nblocks > 1 && threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(&bar[0], 1u);
    if (prev + 1u == nblocks * epoch) {
      st_release_gpu(&bar[1], epoch);
    } else {
      while (ld_relaxed_gpu(&bar[1]) < epoch) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// The grid barrier extended across ranks (world > 1, peer exchange).  Every
// CTA fences at system scope (covering its mirrored removals on the peers)
// before it counts itself in; the CTA that completes the local count
// publishes "this rank finished global pass seqv" on every peer and waits
// for every peer's arrival before it releases the local grid.  The wait gives
// up after p.timeout_ns (a peer that never launched) and sets *p.xerr.
static __device__ __noinline__ void grid_sync_peer(unsigned* bar, unsigned nblocks, unsigned epoch, const FusedParams& p,
                                               unsigned long long seqv) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const bool last = nblocks == 1 || atomicAdd(&bar[0], 1u) + 1u == nblocks * epoch;
    if (last) {
      __threadfence_system();  // acquire the other CTAs' arrivals before publishing ours
      for (int q = 0; q < p.mir.world; ++q)
        if (q != p.mir.rank) st_release_sys64(p.peer_arrive[q] + p.mir.rank, seqv);
      const unsigned long long t0 = globaltimer();
      for (int q = 0; q < p.mir.world; ++q) {
        if (q == p.mir.rank) continue;
        while (ld_relaxed_sys64(p.arrive + q) < seqv) {
          if (*reinterpret_cast<volatile int32_t*>(p.xerr)) break;
          if (globaltimer() - t0 > p.timeout_ns) {
            atomicExch(p.xerr, 1);
            break;
          }
          __nanosleep(64);
        }
      }
      __threadfence_system();
      if (nblocks > 1) st_release_gpu(&bar[1], epoch);
    } else {
      while (ld_relaxed_gpu(&bar[1]) < epoch) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

#endif  // __CUDACC__

}  // namespace rac
