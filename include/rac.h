/*
 * rac.h -- C ABI of librac.so: Recurrent Arc Consistency (RAC) enforcement on
 * NVIDIA B200 (sm_100a).  arXiv 2407.11388, "Paralleling and Accelerating Arc
 * Consistency Enforcement with Recurrent Tensor Computations".
 *
 * The operation (PAPER.md, reference lines cited as P:n):
 *   A binary CSP has variables x with domains dom(x) and binary constraints
 *   c_xy with relations rel(c_xy).  c_xy|(x,a) = { tau[y] | tau in rel(c_xy),
 *   tau[x] = a } is the support set of (x,a) on c_xy; C_x is the set of
 *   constraints involving x.  A domain set D is arc consistent iff every
 *   (x,a) in D has c_xy|(x,a) ∩ D(y) ≠ ∅ for every c_xy in C_x.
 *   D_ac = the union of all arc-consistent subsets of D.
 *   rac_enforce computes D_ac by the RAC recurrence, Eq. 1:
 *     D_0 = D_in;  D_k = { (x,a) in D_{k-1} : ∀ c_xy ∈ C_x, c_xy|(x,a) ∩ D_{k-1}(y) ≠ ∅ }
 *   (the complement form of D~(k) = D~(k-1) ∪ {(x,a) | ∃y c_xy|(x,a) ⊆ D~(k-1)}),
 *   iterated with the loop control of Alg. 1 tensorAC: after each
 *   pass, if some D_k(x) = ∅ stop with RAC_WIPEOUT ("throw inconsistency",
 *   P:203-204), else if D_k = D_{k-1} stop with RAC_OK (Prop. 1 end condition,
 *   D_ac = D \ D~(K)).
 *   The reported iteration count is the number of passes executed, including
 *   the final no-change pass and the wipeout-detecting pass (the number of
 *   Alg. 1 loop bodies; reading R3).  Every pass reads only D_{k-1}
 *   (synchronous / Jacobi update; reading R4).
 *
 * Data formats
 *   Domain state D: uint64_t[n_vars]; bit a of word x set iff (x,a) ∈ D.
 *     Bits at positions >= dom_sizes[x] must be 0.
 *   Relation: for a constraint on (x, y), rows[a] (a < dom[x]) is a uint64_t
 *     whose bit b is set iff (a, b) ∈ rel(c_xy); i.e. rows[a] = c_xy|(x,a).
 *     Bits >= dom[y] must be 0.  The (y, x) orientation is derived (transpose).
 *   Domain sizes: 1 <= dom_sizes[x] <= 256 (RAC_MAX_DOM_WIDE).
 *   Wide domains (max dom > 64; SURVEY §8(f) NEXT-4 -- the paper fixes no
 *   domain-size limit, its Cons is a dense [n,d,n,d] tensor):
 *     every domain state is wq = ceil(max dom / 64) words per variable
 *     (rac_words_per_var): bit a of x is bit a%64 of word D[x*wq + a/64]; a
 *     relation's rows are dom[x] x wq words (row a at rows + a*wq); removal
 *     epochs are [n_vars * 64 * wq] (x,a) at x*64*wq + a.  With max dom <= 64,
 *     wq = 1 and every format below is unchanged.  Wide contexts support
 *     rac_create / rac_create_random / rac_enforce / rac_enforce_ex /
 *     rac_enforce_async / rac_enforce_seeded / rac_enforce_seeded_async /
 *     rac_search on one GPU (world == 1, dense layout); the sharded and peer
 *     calls return RAC_EUNSUPPORTED.
 *
 * Return values: every int-returning call returns >= 0 on success (RAC_OK or
 * RAC_WIPEOUT for enforcement calls) and a negative RAC_E* code on error.
 * Nothing is thrown or aborted across the ABI.  After RAC_ECUDA / RAC_ENCCL /
 * RAC_EPEER the context is unusable and every later call returns RAC_ESTATE.
 * rac_last_error(ctx) gives a message (ctx == NULL: the thread's last failed
 * create).
 *
 * Ownership: inputs are borrowed for the duration of the call; rac_create
 * deep-copies and packs relations, so callers may free them on return.  The
 * context owns all its device memory (and, for world > 1, its NCCL
 * communicator).  Callers own every D / iteration / status buffer.  d_out may
 * equal d_in (in place); any other overlap is undefined.
 *
 * Concurrency: calls on one context must be serialized by the caller;
 * distinct contexts are independent.
 *
 * Multi-GPU (world > 1): rac_create* and every rac_enforce* call are
 * COLLECTIVE over the `world` ranks (one process per GPU).  The relation tensor
 * is row-sharded: rank r holds the masks of variables [x_lo, x_hi) given by
 * rac_shard_range.  Two exchange paths (neither is in the paper, which is
 * single-GPU; BASELINE.json north_star asks for the row sharding):
 *   NCCL (default): one rac_pass launch per pass over the local rows, then an
 *     NCCL all-gather of the new alive bitvector; the host polls a done flag.
 *   Peer memory (RAC_OPT_PEER): the whole enforcement is ONE persistent kernel
 *     per rank.  Every removal bit found on the local rows is also OR-ed into
 *     the same word of every peer's removal buffer (NVLink P2P atomics), and
 *     the grid barrier between passes is extended across ranks with
 *     system-scope release/acquire arrival words; no host round trip and no
 *     separate collective per pass.  Needs rac_connect_peers (one process per
 *     GPU, IPC handles) or rac_connect_peers_local (one process driving
 *     several ranks) before the first enforcement.
 * Every rank derives the same stop decision from the same data, so all ranks
 * return identical d_out, iterations and status.  Every rank must pass
 * identical n_vars, dom_sizes and d_in, and make the same sequence of calls.
 */
#ifndef RAC_H
#define RAC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------- */
#define RAC_OK 0             /* fixpoint, no empty domain: d_out == D_ac(d_in)            */
#define RAC_WIPEOUT 1        /* some domain empty: d_out = D after the detecting pass     */
#define RAC_BUDGET 2         /* rac_search: assignment budget exhausted before a verdict  */
#define RAC_EINVAL (-1)      /* invalid argument (see each call)                          */
#define RAC_ENOMEM (-2)      /* host or device allocation failed                          */
#define RAC_ECUDA (-3)       /* CUDA error; context now unusable                          */
#define RAC_ENCCL (-4)       /* NCCL error (or NCCL unavailable for world > 1)            */
#define RAC_ESTATE (-5)      /* context unusable after an earlier CUDA/NCCL error         */
#define RAC_EUNSUPPORTED (-6)/* valid request this build does not support                 */
#define RAC_EPEER (-7)       /* peer-memory exchange failed (IPC open, or a rank did not
                                arrive within RAC_PEER_TIMEOUT_MS, default 20000 ms);
                                context now unusable                                     */

/* ---- flags -------------------------------------------------------------- */
/* Do not stop at the first wipeout: iterate to the definitional fixpoint D_ac
 * (in which a wiped component is emptied).  Status is RAC_WIPEOUT iff some
 * domain of the fixpoint is empty. */
#define RAC_FULL_FIXPOINT (1u << 0)

#define RAC_MAX_DOM 64       /* one-word domains: every call                 */
#define RAC_MAX_DOM_WIDE 256 /* multi-word domains: see "Wide domains" above */
#define RAC_NCCL_ID_BYTES 128

typedef struct rac_ctx rac_ctx;

/* One binary constraint c_xy.  0 <= x, y < n_vars, x != y; at most one
 * relation per unordered pair (either orientation).  rows has dom[x] words. */
typedef struct {
  int32_t x, y;
  const uint64_t* rows;
} rac_relation;

/* rac_options.flags: run a world == 1 context through the multi-GPU exchange
 * path with a one-rank NCCL communicator (exercises the NCCL all-gather leg on
 * a single GPU; results are identical to the fused path). */
#define RAC_OPT_NCCL_SELF (1u << 0)
/* rac_options.flags: world > 1 exchanges through peer memory inside the fused
 * kernel instead of NCCL (see "Multi-GPU" above); 2 <= world <= RAC_MAX_RANKS. */
#define RAC_OPT_PEER (1u << 1)
/* rac_options.flags: relation layout (NEXT-3).  Dense (default for instances
 * whose dense tensor is L2-sized or that are nearly complete): every (x,a) row
 * holds n masks, absent pairs all-ones.  Sparse arc blocks: only declared arcs
 * are stored -- block = the masks c_xy|(x,a) of one arc for all a, the blocks
 * of column y contiguous (Cons[:, y]) -- so a pass reads only declared
 * constraints (the paper's density grid 0.1-0.75).  Without either
 * flag the library picks sparse on one GPU when the dense column tensor is
 * >= 64 MB and the sparse one is <= 0.7 of it.  Sparse contexts need
 * world == 1 without virtual shards / NCCL_SELF (RAC_EINVAL otherwise) and do
 * not support the batched calls (RAC_EUNSUPPORTED); results are identical. */
#define RAC_OPT_SPARSE (1u << 2)
#define RAC_OPT_DENSE (1u << 3)
#define RAC_LAYOUT_DENSE 0
#define RAC_LAYOUT_SPARSE 1
#define RAC_MAX_RANKS 8
#define RAC_IPC_HANDLE_BYTES 64

typedef struct {
  int32_t device;             /* CUDA device ordinal (rank's GPU)                     */
  uint32_t flags;             /* RAC_OPT_* bits (0: defaults)                         */
  int32_t rank, world;        /* world <= 1: single GPU                               */
  const void* nccl_unique_id; /* world > 1: RAC_NCCL_ID_BYTES bytes, identical on all
                                 ranks (from rac_get_nccl_unique_id on rank 0)        */
  int32_t virtual_shards;     /* world <= 1 only.  > 1: run the sharded per-pass path
                                 over this many row blocks on one GPU, a device copy
                                 standing in for the all-gather (tests the partition
                                 without NCCL).  0 or 1: fused single-GPU path.      */
  int32_t max_ctas;           /* > 0: cap the CTAs of the enforcement kernels (and
                                 launch the fused kernel without the cooperative
                                 API): lets several RAC_OPT_PEER ranks share one GPU,
                                 whose grids must then fit on it together.  0: all
                                 SMs.                                                */
} rac_options;

/* Fill *opt with defaults: device 0, single GPU, fused path. */
void rac_default_options(rac_options* opt);

/*
 * Create a context from explicit relations ("Prepare Cons"; Fig. 1).
 * Packs, on the device, every relation into per-(x,a) support masks (both
 * orientations) plus a constraint-presence bitmap.
 * RAC_EINVAL: n_vars < 1; dom size outside [1,256]; x == y or out of range;
 * duplicate unordered pair; bits beyond the domain sizes; NULL pointers
 * (rels may be NULL iff n_rel == 0); bad options.
 */
int rac_create(int32_t n_vars, const int32_t* dom_sizes, int32_t n_rel, const rac_relation* rels,
               const rac_options* opt, rac_ctx** out);

/*
 * Create a context holding the seeded random CSP of synth/csp_synth.h, generated
 * directly into the packed layout on the device (no host relation copy; needed at
 * 30+ GB).  Workload shape: PAPER.md §5.2 P:232-236.  Uniform domain size d.
 * dens_q32 in [0, 2^32] (pair constrained iff 32-bit draw < dens_q32);
 * t_q16 in [0, 65536] (value pair forbidden iff 16-bit draw < t_q16).
 */
int rac_create_random(int32_t n_vars, int32_t d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                      const rac_options* opt, rac_ctx** out);

/* Blocking enforcement, host buffers: d_in, d_out = uint64_t[n_vars * wq]
 * (wq = rac_words_per_var(ctx): 1 unless the domains are wider than 64 values;
 * bit a of x is bit a%64 of word x*wq + a/64).
 * Returns RAC_OK / RAC_WIPEOUT (and *iterations) or an error.
 * RAC_EINVAL: NULL pointers; bits of d_in beyond dom sizes. */
int rac_enforce(rac_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations);

/* As rac_enforce, plus flags (RAC_FULL_FIXPOINT) and, if removed_at != NULL,
 * removed_at[x*64*wq + a] (int32_t[n_vars * 64 * wq]) = the pass that removed
 * (x,a), 0 if kept or absent (the per-step sets V^(k) of Prop. 2).
 * With world > 1 every rank receives all epochs (gathered with the exchange);
 * removed_at is then collective: all ranks pass it or none does. */
int rac_enforce_ex(rac_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations,
                   int32_t* removed_at, uint32_t flags);

/* Asynchronous enforcement, DEVICE buffers (d_in_dev / d_out_dev:
 * uint64_t[n_vars * wq]), enqueued on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  Writes *status_dev (RAC_OK / RAC_WIPEOUT) and
 * *iterations_dev on the device; returns 0 once enqueued.  Bits of d_in
 * beyond dom sizes are ignored.  removed_at_dev is nullable
 * (int32_t[n_vars * 64 * wq], as in rac_enforce_ex).  On the single-GPU fused path
 * the host is not involved per iteration; on the sharded path (world > 1 or
 * virtual_shards > 1) the host reads a device flag once per chunk of passes. */
int rac_enforce_async(rac_ctx* ctx, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                      int32_t* iterations_dev, int32_t* status_dev, int32_t* removed_at_dev,
                      uint32_t flags, void* stream);

/* Batched enforcement of n_states independent domain states (search-tree nodes)
 * on one instance, DEVICE buffers: d_in_dev/d_out_dev = uint64_t[n_states][n_vars * wq],
 * iterations_dev/status_dev = int32_t[n_states].  State s's results are exactly
 * those of rac_enforce on state s alone (each state stops at its own pass).
 * world == 1 only (batches are sharded by the caller). */
int rac_enforce_batch(rac_ctx* ctx, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                      int32_t* iterations_dev, int32_t* status_dev, uint32_t flags, void* stream);

/* Seeded (incremental) enforcement: Alg. 1 tensorAC(Vars, @changed = seeds)
 * (P:198-221), the paper's per-assignment call tensorAC(Vars, [idx]).
 * PRECONDITION: d_in is arc consistent on every constraint c_xy whose y is not
 * a seed -- e.g. the D_ac of a parent search node after the seed variables'
 * domains were reduced (an assignment).  Under it the result
 * (status, d_out, iterations) equals rac_enforce(d_in): by Prop. 2
 * the trajectory is the same, but pass 1 reads only the masks of the seed
 * variables instead of the whole relation tensor.  Without the precondition the
 * result is sound (every removal is justified by Lemma 1) but may keep values
 * D_ac removes.  n_seeds == 0: no pass, iterations = 0, status RAC_WIPEOUT iff
 * some domain of d_in is empty.  seeds: host int32[n_seeds], each in [0, n)
 * (RAC_EINVAL otherwise).  d_in, d_out: uint64_t[n_vars * wq]. */
int rac_enforce_seeded(rac_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations,
                       const int32_t* seeds, int32_t n_seeds, uint32_t flags);

/* As rac_enforce_seeded, device buffers (seeds_dev: device int32[n_seeds];
 * NULL allowed when n_seeds == 0), asynchronous on `stream` like
 * rac_enforce_async.  Out-of-range entries of seeds_dev are skipped (the
 * device cannot report them); duplicates test their column once. */
int rac_enforce_seeded_async(rac_ctx* ctx, const uint64_t* d_in_dev, uint64_t* d_out_dev, int32_t* iterations_dev,
                             int32_t* status_dev, const int32_t* seeds_dev, int32_t n_seeds, uint32_t flags,
                             void* stream);

/* Batched seeded enforcement: state s is seeded with the single variable
 * seed_var_dev[s] (device int32[n_states]; -1 = all variables, i.e. a root
 * call), under the precondition above (search-tree children after one
 * assignment each).  Results equal rac_enforce of each state alone.  Off the
 * precondition, the one-word kernels (max dom <= 32: 32-state words per
 * thread-block cluster, every state gated to its own changed columns) and the
 * per-state kernels give exactly rac_enforce_seeded(state, [seed]); the wide
 * tensor-core pass (max dom 65..128, >= 256 states) tests every column in every
 * pass, which agrees under the precondition. */
int rac_enforce_batch_seeded(rac_ctx* ctx, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                             int32_t* iterations_dev, int32_t* status_dev, const int32_t* seed_var_dev,
                             uint32_t flags, void* stream);

/* Measurement of the batched contraction alone: ONE pass of Eq. 1 (every
 * column tested, no loop control) for n_states device states, d_out[s] = D_1.
 * One-word contexts: impl 0 = bit-sliced ALU pass (32 states per u32 OR);
 * impl 1 = tcgen05 tensor-core pass (tcgen05.mma.kind::f16: per column y, 128
 * rows x 16 mask bits times 16 values x 256 states, fp32 counts in TMEM, count
 * > 0 tested in the epilogue; max dom <= 16).  Wide contexts (max dom > 64):
 * impl 2 = bit-sliced byte-table pass; impl 3 = pipelined tcgen05 pass (K =
 * 128 per column as 8 kind::f16 MMAs, two TMEM accumulators, producer / MMA /
 * epilogue warps; max dom <= 128); impl 4 = the same with fp8 (e4m3) 0/1
 * operands (kind::f8f6f4, 4 MMAs of K = 32 per column, half the operand bytes).  world == 1 only.  This is the A/B behind the
 * batched-mode choice, not an enforcement API. */
int rac_batch_pass_eval(rac_ctx* ctx, int32_t impl, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                        void* stream);

/* ---- search (Alg. 2) ---------------------------------------- */
typedef struct {
  int64_t assignments;      /* assign + seeded enforcement events (Table 1's unit) */
  int64_t recurrences;      /* sum of their iteration counts (Table 1's #Recurrence x assignments) */
  int64_t wipeouts;         /* assignments whose enforcement ended in RAC_WIPEOUT               */
  int64_t solutions;        /* complete assignments reached                                    */
  int64_t max_depth;        /* deepest level reached                                            */
  int32_t root_iterations;  /* passes of the root enforcement tensorAC(Vars, all)       */
  int32_t root_status;
  double enforce_seconds;   /* host wall time spent in the per-assignment enforcements          */
} rac_search_stats;

#define RAC_SEARCH_ALL (1u << 8) /* count every solution instead of stopping at the first */

/* Backtracking search maintaining arc consistency (Alg. 2) on the
 * device-resident instance: root enforcement tensorAC(Vars, all),
 * then depth-first: pick the unassigned variable with the smallest current
 * domain (lowest index on ties -- the paper leaves heuristics() open, P:389;
 * SPEC S:396-404), try its values in ascending order, assign (row overwrite,
 * P:410-416) on a copy of the parent's domains, enforce with @changed = [idx]
 * (rac_enforce_seeded), recurse unless wiped out.
 * Returns RAC_OK (a solution: solution[x] = value of x, unless NULL;
 * with RAC_SEARCH_ALL the whole tree is explored and RAC_OK means >= 1
 * solution), RAC_WIPEOUT (unsatisfiable: tree exhausted with no solution) or
 * RAC_BUDGET (max_assignments reached first; max_assignments <= 0 = no limit).
 * d_in: host uint64_t[n_vars].  world == 1 only. */
int rac_search(rac_ctx* ctx, const uint64_t* d_in, int64_t max_assignments, uint32_t flags, int32_t* solution,
               rac_search_stats* stats);

/* ---- introspection ------------------------------------------------------ */
int32_t rac_n_vars(const rac_ctx* ctx);
int32_t rac_max_dom(const rac_ctx* ctx);
/* Bytes per packed support mask (1, 2, 4 or 8: the smallest width >= max dom bits;
 * 16 or 32 for wide domains: max dom <= 128 or <= 256). */
int32_t rac_mask_bytes(const rac_ctx* ctx);
/* Words per variable of every domain state of this context: ceil(max dom / 64)
 * (1 for max dom <= 64).  RAC_EINVAL if ctx is NULL. */
int32_t rac_words_per_var(const rac_ctx* ctx);
/* Bytes of packed support masks held by this rank (rows x row stride). */
int64_t rac_relation_bytes(const rac_ctx* ctx);
/* Row block [*x_lo, *x_hi) of variables owned by `rank` of `world` (host only,
 * no GPU needed): contiguous blocks of ceil(n_vars/world). */
int rac_shard_range(int32_t n_vars, int32_t world, int32_t rank, int32_t* x_lo, int32_t* x_hi);
/* This context's row block. */
int rac_local_range(const rac_ctx* ctx, int32_t* x_lo, int32_t* x_hi);
/* Copy the packed support masks of row (x, a) (x in the local block) to host:
 * out_masks[y] = mask M[x][a][y] widened to uint64 (all ones for absent pairs and
 * y == x), out_present[y] = 1 iff c_xy is declared.  Either output may be NULL. */
int rac_read_row(const rac_ctx* ctx, int32_t x, int32_t a, uint64_t* out_masks, uint8_t* out_present);
/* NCCL unique id for rac_options.nccl_unique_id (call on rank 0, broadcast). */
int rac_get_nccl_unique_id(void* out /* RAC_NCCL_ID_BYTES */);
/* Peer-memory exchange (RAC_OPT_PEER contexts).  Each rank exposes one device
 * region (its removal buffers, removal flags, arrival words and pass counter;
 * layout private to the library, identical on all ranks).
 * rac_peer_handle: the region's CUDA IPC handle (RAC_IPC_HANDLE_BYTES bytes) to
 *   all-gather over the host transport (e.g. torch.distributed).
 * rac_connect_peers: handles = world x RAC_IPC_HANDLE_BYTES bytes in rank order
 *   (own entry ignored); opens every peer's region (cudaIpcOpenMemHandle, peer
 *   access enabled lazily).  RAC_EPEER if a handle cannot be opened.
 * rac_peer_region / rac_connect_peers_local: the same for ranks driven by ONE
 *   process: regions[q] = rank q's region pointer (rac_peer_region), devices[q]
 *   = its device; enables peer access between distinct devices
 *   (RAC_EUNSUPPORTED if the devices cannot access each other).  Ranks may
 *   share a device (then size max_ctas so that all grids fit together).
 * Connect once, before the first enforcement; destroy the ranks' contexts only
 * after every rank's work has completed. */
int rac_peer_handle(const rac_ctx* ctx, void* out /* RAC_IPC_HANDLE_BYTES */);
int rac_connect_peers(rac_ctx* ctx, const void* handles /* world x RAC_IPC_HANDLE_BYTES */);
int rac_peer_region(const rac_ctx* ctx, void** region_dev);
int rac_connect_peers_local(rac_ctx* ctx, void* const* regions /* [world] */, const int32_t* devices /* [world] */);
/* RAC_LAYOUT_DENSE or RAC_LAYOUT_SPARSE (see RAC_OPT_SPARSE). */
int32_t rac_layout(const rac_ctx* ctx);
/* Which kernel runs a single-state enforcement on this context:
 *   RAC_PATH_FUSED     persistent cooperative kernel (dense one-word layout)
 *   RAC_PATH_ONE_BLOCK one thread block per state (small instances: the whole
 *                      mask tensor is L2-sized; also the batched calls' kernel)
 *   RAC_PATH_SPARSE    persistent cooperative kernel over the sparse layout
 *   RAC_PATH_SHARDED   per-pass launches + exchange (world > 1 / virtual shards)
 *   RAC_PATH_PEER      persistent kernel + peer-memory exchange (RAC_OPT_PEER)
 *   RAC_PATH_WIDE      wide-domain persistent kernel (max dom > 64)
 * RAC_EINVAL if ctx is NULL. */
#define RAC_PATH_FUSED 0
#define RAC_PATH_ONE_BLOCK 1
#define RAC_PATH_SPARSE 2
#define RAC_PATH_SHARDED 3
#define RAC_PATH_PEER 4
#define RAC_PATH_WIDE 5
int32_t rac_path(const rac_ctx* ctx);
/* Kernel launches enqueued by the last rac_enforce* call on this context. */
int64_t rac_last_launch_count(const rac_ctx* ctx);
/* Sweep used for full passes (every live row against every column: pass 1 of a
 * root call) of a dense single-GPU context: 0 = row-major sweep, 1 = column
 * sweep.  Both read the same bytes; HBM-resident contexts time one root
 * enforcement with each at rac_create and keep the faster (*ms_cols, *ms_rows:
 * best times in ms, 0 when not measured; either pointer may be NULL). */
int32_t rac_full_pass_layout(const rac_ctx* ctx, float* ms_cols, float* ms_rows);

const char* rac_last_error(const rac_ctx* ctx);
void rac_destroy(rac_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* RAC_H */
