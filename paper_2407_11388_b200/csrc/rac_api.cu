// rac_api.cu -- the C ABI of librac.so (declared and documented in include/rac.h).
//
// Host side: validation, device memory ownership, the loop drivers and the
// NCCL communicator.  Every step of the method runs in the kernels of
// rac_kernels.cu / rac_pack.cu; there is no CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>

#include <numeric>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <vector>

#include "../../include/rac.h"
#include "../../synth/csp_synth.h"  // presence of generated pairs (rac_create_random, sparse layout)
#include "rac_internal.cuh"

using namespace rac;

// ----------------------------------------------------------------------------- NCCL (dlopen)
namespace {

typedef int ncclResult_t;
typedef void* ncclComm_t;
typedef struct { char internal[RAC_NCCL_ID_BYTES]; } ncclUniqueId;
constexpr int kNcclUint64 = 5;  // ncclUint64 in nccl.h
constexpr int kNcclInt32 = 2;   // ncclInt32

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (!api.loaded) {
    // Prefer the copy torch already loaded (same soname), else load it.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.loaded = api.GetUniqueId && api.CommInitRank && api.AllGather && api.CommDestroy;
    }
  }
  return api;
}

thread_local std::string g_create_error;

}  // namespace

// ----------------------------------------------------------------------------- context
struct rac_ctx {
  int device = 0;
  int rank = 0, world = 1, vshards = 1;
  bool nccl_self = false;  // world == 1 through the NCCL exchange path (RAC_OPT_NCCL_SELF)
  bool peer = false;       // world > 1 through the fused kernel + peer-memory exchange (RAC_OPT_PEER)
  bool connected = false;  // peer regions known (rac_connect_peers*)
  int max_ctas = 0;        // rac_options.max_ctas
  bool use_nccl() const { return (world > 1 && !peer) || nccl_self; }
  int n = 0, dmax = 0, W = 0;
  int rows_pad = 0;        // local rows padded to a warp slab
  size_t col_stride = 0;   // bytes per column of the mask tensor
  uint8_t* Mg = nullptr;   // batched mode: 8-byte column groups of the mask tensor (built on first use)
  unsigned* cctr = nullptr;  // partitioned tail-claim counters of the column sweep [3][32][32]
  int dbytes = 0;          // bytes of D in smem
  int x_lo = 0, x_hi = 0, blk = 0;
  int pw = 0;
  std::vector<int32_t> dom;
  std::vector<uint64_t> dommask_h;
  // device
  uint8_t* M = nullptr;     // column-major masks
  uint8_t* Mr = nullptr;    // row-major copy (nullable)
  int G = 1;                // lanes per row of the row-major sweep
  int force_layout = 0;     // RAC_FORCE_LAYOUT=rows|cols|tiecols (testing knob); 3 after calibrate_tie picks columns
  bool row_agg = false;     // row sweep aggregates removals per CTA in shared memory (dense, when n words fit)
  float tie_ms[2] = {0.f, 0.f};  // calibrate_tie: best root enforcement with ties to columns / rows
  uint32_t* P = nullptr;
  // Sparse arc-block layout (NEXT-3; rac.h RAC_OPT_SPARSE): only declared arcs
  bool sparse = false;
  uint8_t* S = nullptr;          // [s_nblk][s_bbytes]
  uint32_t* s_off = nullptr;     // [n+1]
  uint32_t* s_arc = nullptr;     // [s_nblk] x | y << 16
  uint32_t* s_ipref = nullptr;   // [n+1] full-pass work-item prefix (sparse_sweep)
  uint32_t s_nblk = 0;
  int s_dpad = 0, s_bbytes = 0, s_vb = 0;
  std::vector<uint32_t> s_off_h, s_arc_h;
  int32_t* dom_d = nullptr;
  uint64_t* dommask = nullptr;
  // Exchange region (one allocation so that one IPC handle maps it): the
  // fused kernel's rotating removal buffers R[3][n], per-pass removal flags,
  // the arrival words peers write, and the global pass counter.
  uint8_t* xr = nullptr;
  unsigned long long* R3 = nullptr;  // = xr
  uint8_t* peer_base[RAC_MAX_RANKS] = {};  // every rank's region as seen from this device (self = xr)
  bool peer_ipc[RAC_MAX_RANKS] = {};       // opened with cudaIpcOpenMemHandle (closed at destroy)
  unsigned* bar = nullptr;
  uint32_t* clist = nullptr;  // fused path: per-pass change lists [3][n+1]
  ShardState sh{};
  uint64_t* buf_in = nullptr;   // blocking-API staging
  uint64_t* buf_out = nullptr;
  int32_t* buf_scalars = nullptr;  // [iters, status]
  int32_t* buf_removed = nullptr;  // [n*64]
  int32_t* ra_g = nullptr;         // world > 1 (NCCL): padded epoch all-gather buffer
  int32_t* buf_seeds = nullptr;    // [seed_cap]
  size_t seed_cap = 0;
  uint32_t* bs_X2 = nullptr;       // bit-sliced batch exchange buffers
  size_t bs_X2_cap = 0;            // bytes
  unsigned* bs_bar = nullptr;      // per-word barrier words
  size_t bs_bar_cap = 0;           // words
  unsigned long long* dbg = nullptr;  // RAC_DEBUG_TIMELINE phase timestamps [256]
  unsigned long long* bs_dbg = nullptr;  // bit-sliced batch: [ctas][64] pass-end timestamps
  uint32_t* eval_buf = nullptr;          // rac_batch_pass_eval scratch
  uint8_t* tc_buf = nullptr;             // wide tensor-core batch scratch
  size_t tc_cap = 0;
  size_t eval_cap = 0;
  int bs_dbg_ctas = 0;
  uint64_t* h_in = nullptr;        // pinned staging: [d_in words | seeds (seed_cap int32)]
  uint64_t* h_out = nullptr;       // pinned + mapped: [d_out words | iters, status] written by the kernel
  uint64_t* d_hout = nullptr;      // device view of h_out (zero-copy: no D2H copy in the blocking API)
  int32_t* h_scalars = nullptr;    // pinned [iters, status, done]
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  int fused_grid = 0;
  int pass_grid = 0;
  ncclComm_t comm = nullptr;
  // Wide domains (NEXT-4, rac_wide.cu): dmax > 64.  M / P / dom_d / clist /
  // staging buffers are shared with the one-word layout's fields.
  bool wide = false;
  int wq = 1, WS = 0;       // boundary words per variable, mask words per (x,a,y)
  uint64_t* wD = nullptr;   // [n*WS] current state
  uint64_t* wR = nullptr;   // [n*WS] removal bits
  unsigned* wslots = nullptr;
  int wide_grid = 0;
  size_t wide_smem = 0;
  // rac_state (one block per state): batched mode and small single instances
  StateParams state_geom{};  // shared-memory layout (state_layout)
  size_t state_smem = 0;
  int state_T = 128;         // threads per block
  bool small = false;        // single instance small enough for one block
  bool tiny = false;         // ... and for one warp (n <= 64): rac_tiny
  // Blocking calls on small instances: [H2D of d_in (+ seeds), kernel] replayed
  // as one CUDA graph per (seed count, flags) -- one launch instead of a copy
  // and a kernel launch (graphs[] keyed by gkey[]; cleared when the staging
  // buffers move).
  static constexpr int kGraphs = 8;
  cudaGraphExec_t graphs[kGraphs] = {};
  int64_t gkey[kGraphs] = {};
  int ngraphs = 0;
  bool graphs_off = false;
  int64_t launches = 0;
  bool broken = false;
  std::string err;
};

namespace {

int fail(rac_ctx* c, int code, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (code == RAC_ECUDA || code == RAC_ENCCL || code == RAC_EPEER) c->broken = true;
  } else {
    g_create_error = msg;
  }
  return code;
}

#define CK(ctx, call)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail((ctx), RAC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)

uint64_t dom_mask(int k) { return k >= 64 ? ~0ull : ((1ull << k) - 1ull); }

int mask_bytes(int dmax) { return dmax <= 8 ? 1 : dmax <= 16 ? 2 : dmax <= 32 ? 4 : 8; }

// Blocking-API staging: pinned h_in / device buf_in hold [d_in | seeds] so one
// H2D copy moves both; h_out is pinned AND mapped: the kernels write D_out and
// [iters, status] straight into it (zero-copy), so no D2H copy is enqueued.
// (Re)allocates the input staging with room for `seeds` seed entries.
void drop_graphs(rac_ctx* c);

cudaError_t alloc_staging(rac_ctx* c, size_t nb, size_t seeds) {
  drop_graphs(c);  // captured graphs point at the old buffers
  cudaFree(c->buf_in);
  cudaFreeHost(c->h_in);
  c->buf_in = nullptr;
  c->h_in = nullptr;
  c->buf_seeds = nullptr;
  c->seed_cap = 0;
  cudaError_t e = cudaMalloc(&c->buf_in, nb + seeds * 4);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_in, nb + seeds * 4);
  if (e != cudaSuccess) return e;
  c->buf_seeds = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(c->buf_in) + nb);
  c->seed_cap = seeds;
  if (!c->h_out) {
    e = cudaHostAlloc(&c->h_out, nb + 16, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_hout), c->h_out, 0);
  }
  return e;
}

// cudaSetDevice only when another device is current (the call is not free).
cudaError_t ensure_device(const rac_ctx* c) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e == cudaSuccess && cur == c->device) return cudaSuccess;
  return cudaSetDevice(c->device);
}

void drop_graphs(rac_ctx* c) {
  for (int i = 0; i < c->ngraphs; ++i)
    if (c->graphs[i]) cudaGraphExecDestroy(c->graphs[i]);
  c->ngraphs = 0;
}

void free_ctx(rac_ctx* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  drop_graphs(c);
  if (c->comm && nccl().loaded) nccl().CommDestroy(c->comm);
  for (int q = 0; q < RAC_MAX_RANKS; ++q)
    if (c->peer_ipc[q]) cudaIpcCloseMemHandle(c->peer_base[q]);
  cudaFree(c->M);
  cudaFree(c->Mr);
  cudaFree(c->Mg);
  cudaFree(c->cctr);
  cudaFree(c->S);
  cudaFree(c->s_off);
  cudaFree(c->s_arc);
  cudaFree(c->s_ipref);
  cudaFree(c->P);
  cudaFree(c->dom_d);
  cudaFree(c->dommask);
  cudaFree(c->xr);
  cudaFree(c->bar);
  cudaFree(c->clist);
  cudaFree(c->sh.Dcur);
  cudaFree(c->sh.Dg);
  cudaFree(c->sh.Dw);
  cudaFree(c->sh.R);
  cudaFree(c->sh.iters);
  cudaFree(c->sh.vlist);
  cudaFree(c->buf_in);
  cudaFree(c->buf_out);
  cudaFree(c->buf_scalars);
  cudaFree(c->buf_removed);
  cudaFree(c->ra_g);
  cudaFree(c->bs_X2);
  cudaFree(c->bs_bar);
  cudaFree(c->dbg);
  cudaFree(c->bs_dbg);
  cudaFree(c->eval_buf);
  cudaFree(c->tc_buf);
  cudaFree(c->wD);
  cudaFree(c->wR);
  cudaFree(c->wslots);
  cudaFreeHost(c->h_in);
  cudaFreeHost(c->h_out);
  cudaFreeHost(c->h_scalars);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// Exchange region layout (identical on every rank: it depends on n only).
size_t xr_rflag_off(int n) { return (size_t)3 * n * 8; }                 // u32[4]
size_t xr_arrive_off(int n) { return xr_rflag_off(n) + 16; }             // u64[RAC_MAX_RANKS]
size_t xr_seq_off(int n) { return xr_arrive_off(n) + 8 * RAC_MAX_RANKS; }  // u64
size_t xr_calls_off(int n) { return xr_seq_off(n) + 8; }                     // u64: calls with removal epochs
size_t xr_epoch_off(int n) { return xr_calls_off(n) + 8; }                   // int32 [2][n*64]
size_t xr_bytes(int n) { return xr_epoch_off(n) + (size_t)2 * n * 64 * 4; }

size_t kernel_smem(const rac_ctx* c) {
  return c->sparse ? sparse_smem(c->dbytes, c->n)
                   : fused_smem(c->dbytes, c->n) + (c->row_agg ? (((size_t)c->n * 8 + 15) & ~(size_t)15) : 0);
}

// Sparse arc-block geometry: dpad rows per block so that a block is a whole
// number of 16-byte vectors.
int sparse_dpad(int dmax, int W) {
  const int L = 16 / W;
  return (dmax + L - 1) / L * L;
}

// Common part of rac_create / rac_create_random up to (not including) packing.
int setup_ctx(rac_ctx* c, int32_t n, const int32_t* dom, const rac_options* opt, double n_pairs) {
  rac_options o;
  rac_default_options(&o);
  if (opt) o = *opt;
  if (o.flags & ~(RAC_OPT_NCCL_SELF | RAC_OPT_PEER | RAC_OPT_SPARSE | RAC_OPT_DENSE))
    return fail(nullptr, RAC_EINVAL, "unknown options.flags");
  if ((o.flags & RAC_OPT_SPARSE) && (o.flags & RAC_OPT_DENSE))
    return fail(nullptr, RAC_EINVAL, "RAC_OPT_SPARSE and RAC_OPT_DENSE together");
  if ((o.flags & RAC_OPT_SPARSE) && (o.world > 1 || o.virtual_shards > 1 || (o.flags & RAC_OPT_NCCL_SELF)))
    return fail(nullptr, RAC_EINVAL, "RAC_OPT_SPARSE needs world == 1 without virtual shards / NCCL_SELF");
  if ((o.flags & RAC_OPT_NCCL_SELF) && o.world > 1) return fail(nullptr, RAC_EINVAL, "RAC_OPT_NCCL_SELF needs world == 1");
  if ((o.flags & RAC_OPT_PEER) && (o.world < 2 || o.world > RAC_MAX_RANKS))
    return fail(nullptr, RAC_EINVAL, "RAC_OPT_PEER needs 2 <= world <= RAC_MAX_RANKS");
  if (o.max_ctas < 0) return fail(nullptr, RAC_EINVAL, "max_ctas < 0");
  c->nccl_self = (o.flags & RAC_OPT_NCCL_SELF) != 0;
  c->peer = (o.flags & RAC_OPT_PEER) != 0;
  c->max_ctas = o.max_ctas;
  c->device = o.device;
  c->world = o.world < 1 ? 1 : o.world;
  c->rank = c->world > 1 ? o.rank : 0;
  c->vshards = (c->world == 1 && o.virtual_shards > 1) ? o.virtual_shards : 1;
  if (c->world > 1 && (o.rank < 0 || o.rank >= c->world))
    return fail(nullptr, RAC_EINVAL, "world > 1 needs 0 <= rank < world");
  if (c->world > 1 && !c->peer && !o.nccl_unique_id)
    return fail(nullptr, RAC_EINVAL, "world > 1 needs nccl_unique_id (or RAC_OPT_PEER)");
  if (c->vshards > n) c->vshards = n;
  c->n = n;
  c->dom.assign(dom, dom + n);
  c->dmax = 0;
  for (int x = 0; x < n; ++x) c->dmax = std::max(c->dmax, (int)dom[x]);
  c->dommask_h.resize(n);
  for (int x = 0; x < n; ++x) c->dommask_h[x] = dom_mask(dom[x]);
  c->W = mask_bytes(c->dmax);
  c->dbytes = (int)(((size_t)n * c->W + 15) / 16 * 16);
  c->pw = (n + 31) / 32;
  c->blk = (n + c->world - 1) / c->world;
  rac_shard_range(n, c->world, c->rank, &c->x_lo, &c->x_hi);
  {
    const int rows = (c->x_hi - c->x_lo) * c->dmax;
    const int slab = slab_rows(c->W);
    c->rows_pad = std::max(slab, (rows + slab - 1) / slab * slab);
    c->col_stride = (size_t)c->rows_pad * c->W;
  }
  if (n > 65535) return fail(nullptr, RAC_EUNSUPPORTED, "n_vars > 65535");
  {
    // Layout: the sparse arc-block tensor stores 2 * pairs blocks of dpad masks
    // instead of n columns x rows_pad masks (twice, with the row-major copy).
    // Auto: sparse on one GPU when the dense tensor would not be L2-resident
    // and the sparse one is at most 0.7 of it.
    const double dense_b = (double)n * (double)c->col_stride;
    const int dpad = sparse_dpad(c->dmax, c->W);
    const double sparse_b = 2.0 * n_pairs * dpad * c->W;
    const bool single = c->world == 1 && c->vshards == 1 && !c->nccl_self;
    if (o.flags & RAC_OPT_SPARSE) c->sparse = true;
    else if (o.flags & RAC_OPT_DENSE) c->sparse = false;
    else c->sparse = single && dense_b >= 64.0 * (1 << 20) && sparse_b <= 0.7 * dense_b;
    if (c->sparse) {
      c->s_dpad = dpad;
      c->s_bbytes = dpad * c->W;
      c->s_vb = c->s_bbytes / 16;
      if (2.0 * n_pairs * c->s_vb >= 4294967295.0)
        return fail(nullptr, RAC_EUNSUPPORTED, "sparse layout: more than 2^32 16-byte vectors");
    }
  }

  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(nullptr, RAC_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  if (cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess)
    return fail(nullptr, RAC_ECUDA, "cudaDeviceGetAttribute");
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(nullptr, RAC_ECUDA, "cudaStreamCreate");

  const size_t local_vars = (size_t)(c->x_hi - c->x_lo);
  const size_t mbytes = (size_t)n * c->col_stride;
#define CKC(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      return fail(nullptr, e_ == cudaErrorMemoryAllocation ? RAC_ENOMEM : RAC_ECUDA,                \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                              \
  } while (0)
  CKC(cudaMalloc(&c->M, c->sparse ? 16 : std::max<size_t>(mbytes, 16)));
  CKC(cudaMemsetAsync(c->M, 0xFF, c->sparse ? 16 : std::max<size_t>(mbytes, 16), c->stream));
  if (!c->sparse) {
    // Row-major copy for full passes (dead-row skip, early exit).  Optional:
    // without room for it every pass uses the column-major tensor.
    const size_t rbytes = (size_t)c->rows_pad * c->dbytes;
    const char* fl = getenv("RAC_FORCE_LAYOUT");
    c->force_layout = fl ? (strcmp(fl, "rows") == 0 ? 1 : strcmp(fl, "cols") == 0 ? 2
                                : strcmp(fl, "tiecols") == 0 ? 3 : 0) : 0;
    const char* nr = getenv("RAC_NO_ROW_LAYOUT");
    if (!(nr && *nr && strcmp(nr, "0") != 0) && c->force_layout != 2) {
      if (cudaMalloc(&c->Mr, rbytes) != cudaSuccess) {
        cudaGetLastError();
        c->Mr = nullptr;
      } else {
        CKC(cudaMemsetAsync(c->Mr, 0xFF, rbytes, c->stream));
      }
    }
    c->G = choose_group(c->dbytes / 16);
  }
  CKC(cudaMalloc(&c->P, std::max<size_t>(local_vars * c->pw * 4, 4)));
  CKC(cudaMemsetAsync(c->P, 0, std::max<size_t>(local_vars * c->pw * 4, 4), c->stream));
  CKC(cudaMalloc(&c->dom_d, (size_t)n * 4));
  CKC(cudaMemcpyAsync(c->dom_d, dom, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CKC(cudaMalloc(&c->dommask, (size_t)n * 8));
  CKC(cudaMemcpyAsync(c->dommask, c->dommask_h.data(), (size_t)n * 8, cudaMemcpyHostToDevice, c->stream));
  CKC(cudaMalloc(&c->xr, xr_bytes(n)));
  CKC(cudaMemsetAsync(c->xr, 0, xr_bytes(n), c->stream));
  c->R3 = reinterpret_cast<unsigned long long*>(c->xr);
  if (c->rank < RAC_MAX_RANKS) c->peer_base[c->rank] = c->xr;
  CKC(cudaMalloc(&c->clist, (size_t)3 * (n + 1) * 4));
  CKC(cudaMalloc(&c->cctr, (size_t)3 * 32 * 32 * 4));
  CKC(cudaMemsetAsync(c->cctr, 0, (size_t)3 * 32 * 32 * 4, c->stream));
  CKC(cudaMemsetAsync(c->clist, 0, (size_t)3 * (n + 1) * 4, c->stream));
  CKC(cudaMalloc(&c->bar, 64));
  CKC(cudaMemsetAsync(c->bar, 0, 64, c->stream));  // [0..3] grid barrier, [4..6] row counters, [12] peer error
  const size_t gtot = (size_t)c->world * c->blk;
  CKC(cudaMalloc(&c->sh.Dcur, (size_t)n * 8));
  CKC(cudaMalloc(&c->sh.Dg, gtot * 8));
  CKC(cudaMalloc(&c->sh.Dw, (size_t)c->dbytes));
  CKC(cudaMalloc(&c->sh.R, (size_t)n * 8));
  CKC(cudaMemsetAsync(c->sh.R, 0, (size_t)n * 8, c->stream));
  CKC(cudaMalloc(&c->sh.iters, 32));
  c->sh.status = c->sh.iters + 1;
  c->sh.done = c->sh.iters + 2;
  c->sh.vcnt = c->sh.iters + 3;
  c->sh.seeded = c->sh.iters + 4;
  CKC(cudaMalloc(&c->sh.vlist, (size_t)n * 2 + 16));
  CKC(cudaMalloc(&c->buf_out, (size_t)n * 8));
  CKC(cudaMalloc(&c->buf_scalars, 16));
  CKC(cudaMalloc(&c->buf_removed, (size_t)n * 64 * 4));
  CKC(alloc_staging(c, (size_t)n * 8, 64));
  CKC(cudaMallocHost(&c->h_scalars, 16));

  // A/B knob RAC_ROW_AGG=1: row-sweep removals aggregated per CTA in shared memory
  // (one atomic per (CTA, variable) instead of one per failing row).  Off: it
  // shortened the barrier waits of C3 W-seed's removal-heavy passes (8.6 / 13.3 ->
  // 3.6 / 4.3 us) but lengthened their sweeps as much (119.2 vs 120.2 us, r02aw).
  c->row_agg = !c->sparse && fused_smem(c->dbytes, n) + (size_t)n * 8 <= 160 * 1024 && getenv("RAC_ROW_AGG") != nullptr;
  // Launch geometry.  Fused path: a co-resident grid (cooperative launch),
  // as many CTAs as fit, but no more than the work of a full pass can feed
  // (about 4 items of kUnroll columns x one 512-byte slab per warp).
  const long slabs = c->rows_pad / slab_rows(c->W);
  const long items = c->sparse ? (long)((2.0 * n_pairs * c->s_vb + 32.0 * kUnrollS - 1) / (32.0 * kUnrollS))
                               : slabs * ((n + kUnroll - 1) / kUnroll);
  int occ = 0;
  CKC(fused_occupancy(c->W, c->sparse ? 0 : c->G, kernel_smem(c), &occ));
  if (occ < 1) return fail(nullptr, RAC_EUNSUPPORTED, "support-pass kernel does not fit on an SM (n too large)");
  // about one item per warp (small problems are latency-bound: spread them)
  const long want = (items + (kThreads / 32) - 1) / (kThreads / 32);
  c->fused_grid = (int)std::max(1L, std::min((long)c->sm_count * occ, want));
  int pocc = 0;
  CKC(pass_occupancy(c->W, c->G, kernel_smem(c), &pocc));
  c->pass_grid = (int)std::max(1L, std::min((long)c->sm_count * std::max(1, pocc), want));
  if (c->max_ctas > 0) {
    c->fused_grid = std::min(c->fused_grid, c->max_ctas);
    c->pass_grid = std::min(c->pass_grid, c->max_ctas);
  }
  // rac_state geometry (dense layout, one GPU): the whole mask tensor of a
  // small instance is at most a few hundred KB, which one block streams from L2
  // faster than a cooperative grid can be launched and synchronised
  if (!c->sparse && c->world == 1 && n <= 8192) {
    c->state_smem = state_layout(c->state_geom, n, c->dmax, c->W, c->rows_pad, c->pw, 48 * 1024, 96 * 1024);
    if (c->state_smem > 200 * 1024) c->state_smem = 0;
    const char* st = getenv("RAC_STATE_T");  // A/B knob (tooling only)
    if (st) c->state_T = atoi(st);
    const char* sm = getenv("RAC_SMALL_BYTES");  // A/B knob (tooling only)
    const double small_bytes = sm ? atof(sm) : 256.0 * 1024;
    c->small = c->state_smem > 0 && c->vshards == 1 && !c->nccl_self && (double)mbytes <= small_bytes;
    const char* tn = getenv("RAC_NO_TINY");  // A/B knob (tooling only)
    c->tiny = c->small && n <= 64 && c->pw <= 2 && tiny_smem(n, c->col_stride) <= 96 * 1024 && !(tn && *tn == '1');
  }
  CKC(cudaStreamSynchronize(c->stream));
#undef CKC
  return 0;
}

StateParams state_params(const rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iters, int32_t* status,
                         uint32_t flags) {
  StateParams sp = c->state_geom;
  sp.M = c->M;
  sp.col_stride = c->col_stride;
  sp.n = c->n;
  sp.dmax = c->dmax;
  sp.P = c->P;
  sp.pw = c->pw;
  sp.dommask = c->dommask;
  sp.d_in = d_in;
  sp.d_out = d_out;
  sp.iters = iters;
  sp.status = status;
  sp.seed_var = nullptr;
  sp.seeds = nullptr;
  sp.n_seeds = -1;
  sp.removed_at = nullptr;
  sp.flags = flags;
  sp.dbg = nullptr;
  sp.s0 = 0;
  return sp;
}

PassGeom geom_for(const rac_ctx* c, int x_lo, int x_hi) {
  PassGeom g{};
  g.M = c->M;
  g.col_stride = c->col_stride;
  g.Mr = c->Mr;
  g.force = c->force_layout;
  g.n = c->n;
  g.dmax = c->dmax;
  g.x_lo = x_lo;
  g.x_hi = x_hi;
  g.x_lo_alloc = c->x_lo;
  g.P = c->P;
  g.pw = c->pw;
  g.dbytes = c->dbytes;
  g.S = c->S;
  g.s_off = c->s_off;
  g.s_arc = c->s_arc;
  g.s_ipref = c->s_ipref;
  g.s_nblk = c->s_nblk;
  g.s_vb = c->s_vb;
  return g;
}

// Sparse layout: order the arcs of the pairs (xs[r], ys[r]) by column then x,
// upload the block index, pack the masks (host rows or the generator when
// drows == nullptr) and set the presence bits.
int build_sparse(rac_ctx* c, const std::vector<int32_t>& xs, const std::vector<int32_t>& ys, const uint64_t* drows,
                 int row_words, int d, uint32_t t_q16, uint64_t seed) {
  const long np = (long)xs.size();
  const int n = c->n;
  // arc key = column << 16 | x; value = r << 1 | (1 = the y -> x arc of pair r)
  std::vector<std::pair<uint32_t, uint32_t>> arcs;
  arcs.reserve(2 * np);
  for (long r = 0; r < np; ++r) {
    const uint32_t x = (uint32_t)xs[r], y = (uint32_t)ys[r];
    arcs.push_back({(y << 16) | x, (uint32_t)(r << 1)});      // x -> y: rows of x, column y
    arcs.push_back({(x << 16) | y, (uint32_t)(r << 1) | 1u}); // y -> x: rows of y, column x
  }
  std::sort(arcs.begin(), arcs.end());
  c->s_nblk = (uint32_t)arcs.size();
  c->s_off_h.assign(n + 1, 0u);
  c->s_arc_h.resize(arcs.size());
  std::vector<uint32_t> fwd(np), bwd(np);
  std::vector<uint32_t> pres((size_t)n * c->pw, 0u);
  for (size_t b = 0; b < arcs.size(); ++b) {
    const uint32_t col = arcs[b].first >> 16, row = arcs[b].first & 0xffffu;
    c->s_off_h[col + 1]++;
    c->s_arc_h[b] = row | (col << 16);
    const uint32_t r = arcs[b].second >> 1;
    if (arcs[b].second & 1u) bwd[r] = (uint32_t)b; else fwd[r] = (uint32_t)b;
    pres[(size_t)row * c->pw + (col >> 5)] |= 1u << (col & 31);
  }
  for (int y = 0; y < n; ++y) c->s_off_h[y + 1] += c->s_off_h[y];
  std::vector<uint32_t> ipref(n + 1, 0u);  // full-pass work items (32 x kUnrollS vectors, within a column)
  const uint32_t per_item = 32u * kUnrollS;
  for (int y = 0; y < n; ++y)
    ipref[y + 1] = ipref[y] + ((c->s_off_h[y + 1] - c->s_off_h[y]) * (uint32_t)c->s_vb + per_item - 1u) / per_item;
  const size_t sbytes = std::max<size_t>((size_t)c->s_nblk * c->s_bbytes, 16);
  int32_t *dxs = nullptr, *dys = nullptr;
  uint32_t *dfwd = nullptr, *dbwd = nullptr;
  cudaError_t e = cudaMalloc(&c->S, sbytes);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->S, 0xFF, sbytes, c->stream);
  if (e == cudaSuccess) e = cudaMalloc(&c->s_off, (size_t)(n + 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->s_arc, std::max<size_t>(arcs.size(), 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->s_ipref, (size_t)(n + 1) * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->s_ipref, ipref.data(), (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMalloc(&dxs, (size_t)np * 4);
  if (e == cudaSuccess && np > 0) e = cudaMalloc(&dys, (size_t)np * 4);
  if (e == cudaSuccess && np > 0) e = cudaMalloc(&dfwd, (size_t)np * 4);
  if (e == cudaSuccess && np > 0) e = cudaMalloc(&dbwd, (size_t)np * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->s_off, c->s_off_h.data(), (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMemcpyAsync(c->s_arc, c->s_arc_h.data(), arcs.size() * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMemcpyAsync(dxs, xs.data(), (size_t)np * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMemcpyAsync(dys, ys.data(), (size_t)np * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMemcpyAsync(dfwd, fwd.data(), (size_t)np * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess && np > 0) e = cudaMemcpyAsync(dbwd, bwd.data(), (size_t)np * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->P, pres.data(), pres.size() * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
  SparsePack g{c->S, c->s_bbytes, c->W, c->dom_d, n};
  if (e == cudaSuccess) e = launch_pack_sparse(g, dxs, dys, drows, row_words, dfwd, dbwd, np, d, t_q16, seed, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dxs);
  cudaFree(dys);
  cudaFree(dfwd);
  cudaFree(dbwd);
  if (e != cudaSuccess)
    return fail(nullptr, e == cudaErrorMemoryAllocation ? RAC_ENOMEM : RAC_ECUDA,
                std::string("sparse packing: ") + cudaGetErrorString(e));
  return 0;
}



// Wide-domain context (NEXT-4): one GPU, dense row-major masks of WS words.
int setup_wide(rac_ctx* c, int32_t n, const int32_t* dom, const rac_options* opt) {
  rac_options o;
  rac_default_options(&o);
  if (opt) o = *opt;
  if (o.flags & ~(RAC_OPT_NCCL_SELF | RAC_OPT_PEER | RAC_OPT_SPARSE | RAC_OPT_DENSE))
    return fail(nullptr, RAC_EINVAL, "unknown options.flags");
  if (o.world > 1 || o.virtual_shards > 1 || (o.flags & (RAC_OPT_NCCL_SELF | RAC_OPT_PEER | RAC_OPT_SPARSE)))
    return fail(nullptr, RAC_EUNSUPPORTED, "domains > 64 values: single GPU, dense layout only");
  if (o.max_ctas < 0) return fail(nullptr, RAC_EINVAL, "max_ctas < 0");
  if (n > 65535) return fail(nullptr, RAC_EUNSUPPORTED, "n_vars > 65535");
  c->wide = true;
  c->device = o.device;
  c->max_ctas = o.max_ctas;
  c->n = n;
  c->dom.assign(dom, dom + n);
  c->dmax = 0;
  for (int x = 0; x < n; ++x) c->dmax = std::max(c->dmax, (int)dom[x]);
  c->wq = (c->dmax + 63) / 64;
  c->WS = c->dmax <= 128 ? 2 : 4;
  c->W = c->WS * 8;
  c->pw = (n + 31) / 32;
  c->x_lo = 0;
  c->x_hi = n;
  c->wide_smem = (size_t)n * c->WS * 8;
  if (c->wide_smem > 200 * 1024) return fail(nullptr, RAC_EUNSUPPORTED, "n * mask words too large for the smem D");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(nullptr, RAC_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  if (cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess)
    return fail(nullptr, RAC_ECUDA, "cudaDeviceGetAttribute");
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(nullptr, RAC_ECUDA, "cudaStreamCreate");
  const size_t mbytes = (size_t)n * c->dmax * n * c->WS * 8;
  const size_t nw = (size_t)n * c->wq;
#define CKC(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      return fail(nullptr, e_ == cudaErrorMemoryAllocation ? RAC_ENOMEM : RAC_ECUDA,                \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                              \
  } while (0)
  CKC(cudaMalloc(&c->M, mbytes));
  CKC(cudaMemsetAsync(c->M, 0xFF, mbytes, c->stream));  // absent pairs / diagonal: all ones, P = 0
  CKC(cudaMalloc(&c->P, (size_t)n * c->pw * 4));
  CKC(cudaMemsetAsync(c->P, 0, (size_t)n * c->pw * 4, c->stream));
  CKC(cudaMalloc(&c->dom_d, (size_t)n * 4));
  CKC(cudaMemcpyAsync(c->dom_d, dom, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
  CKC(cudaMalloc(&c->wD, (size_t)n * c->WS * 8));
  CKC(cudaMalloc(&c->wR, (size_t)n * c->WS * 8));
  CKC(cudaMalloc(&c->wslots, 64));
  CKC(cudaMalloc(&c->clist, (size_t)3 * n * 4));
  CKC(cudaMalloc(&c->buf_out, nw * 8));
  CKC(cudaMalloc(&c->buf_scalars, 16));
  CKC(cudaMalloc(&c->buf_removed, nw * 64 * 4));
  CKC(alloc_staging(c, nw * 8, 64));
  CKC(cudaMallocHost(&c->h_scalars, 16));
  CKC(wide_fused_grid(c->WS, c->wide_smem, c->sm_count, &c->wide_grid));
  // about four live rows per warp at most: small instances keep fewer CTAs
  const long rows = (long)n * c->dmax;
  c->wide_grid = (int)std::max(1L, std::min((long)c->wide_grid, (rows + 16 * 4 - 1) / (16 * 4)));
  if (c->max_ctas > 0) c->wide_grid = std::min(c->wide_grid, c->max_ctas);
  CKC(cudaStreamSynchronize(c->stream));
#undef CKC
  return 0;
}

WidePack wide_pack_geom(const rac_ctx* c, uint64_t dens_q32) {
  return WidePack{reinterpret_cast<uint64_t*>(c->M), c->P, c->dom_d, c->n, c->dmax, c->wq, c->WS, c->pw, dens_q32};
}

int enforce_wide(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iters, int32_t* status,
                 int32_t* removed_at, uint32_t flags, cudaStream_t s, const int32_t* seeds = nullptr,
                 int n_seeds = -1) {
  WideParams p{reinterpret_cast<const uint64_t*>(c->M), c->P, c->dom_d, c->n, c->dmax, c->wq, c->WS, c->pw,
               (flags & RAC_FULL_FIXPOINT) ? 1 : 0, d_in, d_out, c->wD, c->wR, c->clist, c->wslots, removed_at,
               iters, status, seeds, n_seeds};
  CK(c, launch_wide_fused(p, c->wide_grid, c->wide_smem, s));
  c->launches = 1;
  return 0;
}

bool wide_bits_ok(const rac_ctx* c, const uint64_t* D) {
  for (int x = 0; x < c->n; ++x)
    for (int w = 0; w < c->wq; ++w) {
      const int bits = std::min(64, std::max(0, c->dom[x] - 64 * w));
      const uint64_t dm = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
      if (D[(size_t)x * c->wq + w] & ~dm) return false;
    }
  return true;
}

// Padding bits of a host domain state (bits at or beyond dom(x) must be 0).
bool bits_ok(const rac_ctx* c, const uint64_t* D) {
  if (c->wide) return wide_bits_ok(c, D);
  uint64_t bad = 0;  // no early exit: a branch-free OR the compiler vectorises
  for (int x = 0; x < c->n; ++x) bad |= D[x] & ~c->dommask_h[x];
  return bad == 0;
}

int check_usable(rac_ctx* c) {
  if (!c) return RAC_EINVAL;
  if (c->broken) return RAC_ESTATE;
  return 0;
}

// n_seeds < 0: root call (every column in pass 1); >= 0: seeded call
// (Alg. 1 @changed = seeds; 0 = empty @changed, no pass, whatever `seeds` is).
int enforce_fused(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iters, int32_t* status,
                  int32_t* removed_at, uint32_t flags, cudaStream_t s, const int32_t* seeds = nullptr,
                  int n_seeds = -1) {
  FusedParams p{};
  p.g = geom_for(c, c->x_lo, c->x_hi);  // world == 1: every row
  p.dommask = c->dommask;
  p.d_in = d_in;
  p.d_out = d_out;
  p.iters = iters;
  p.status = status;
  p.removed_at = removed_at;
  p.R = c->R3;
  p.bar = c->bar;
  static const bool no_claim = getenv("RAC_NO_CLAIM") != nullptr;  // A/B knob (tooling only)
  p.wctr = no_claim ? nullptr : c->bar + 4;
  p.rflag = reinterpret_cast<unsigned*>(c->xr + xr_rflag_off(c->n));
  static const bool no_clist = getenv("RAC_NO_CLIST") != nullptr;  // A/B knob (tooling only)
  p.clist = no_clist ? nullptr : c->clist;
  p.seq = reinterpret_cast<unsigned long long*>(c->xr + xr_seq_off(c->n));
  p.mir.world = c->peer ? c->world : 1;
  p.mir.rank = c->rank;
  p.mir.n = c->n;
  p.xerr = reinterpret_cast<int32_t*>(c->bar + 12);
  if (c->peer) {
    for (int q = 0; q < c->world; ++q) {
      if (q == c->rank) continue;
      p.mir.R[q] = reinterpret_cast<unsigned long long*>(c->peer_base[q]);
      p.mir.flag[q] = reinterpret_cast<unsigned*>(c->peer_base[q] + xr_rflag_off(c->n));
      p.peer_arrive[q] = reinterpret_cast<unsigned long long*>(c->peer_base[q] + xr_arrive_off(c->n));
    }
    p.arrive = reinterpret_cast<unsigned long long*>(c->xr + xr_arrive_off(c->n));
    p.E = reinterpret_cast<int32_t*>(c->xr + xr_epoch_off(c->n));
    p.calls = reinterpret_cast<unsigned long long*>(c->xr + xr_calls_off(c->n));
    for (int q = 0; q < c->world; ++q)
      if (q != c->rank) p.Epeer[q] = reinterpret_cast<int32_t*>(c->peer_base[q] + xr_epoch_off(c->n));
    const char* to = getenv("RAC_PEER_TIMEOUT_MS");
    p.timeout_ns = (unsigned long long)(to ? atoll(to) : 20000) * 1000000ull;
  }
  p.flags = flags;
  static const uint32_t ab = getenv("RAC_FUSED_AB") ? (uint32_t)atoi(getenv("RAC_FUSED_AB")) : 0u;  // tooling
  p.ab = ab;
  // passes t > 1 testing <= 16 columns keep a change list (c3-prop 281 -> 277 us,
  // profiles/r02v; A/B knob RAC_LIST_MAX, 0 = off)
  static const int list_max = getenv("RAC_LIST_MAX") ? atoi(getenv("RAC_LIST_MAX")) : 16;
  p.list_max = list_max;
  p.row_agg = c->row_agg ? 1 : 0;
  static const bool no_cclaim = getenv("RAC_NO_CCLAIM") != nullptr;  // A/B knob (tooling only)
  p.cctr = no_cclaim ? nullptr : c->cctr;
  p.seeds = seeds;
  p.n_seeds = n_seeds;
  if (getenv("RAC_DEBUG_TIMELINE") && !c->dbg) CK(c, cudaMalloc(&c->dbg, (256 + 3000) * 8));
  p.dbg = c->dbg;
  if (removed_at) CK(c, cudaMemsetAsync(removed_at, 0, (size_t)c->n * 64 * 4, s));
  if (c->small && !c->peer && !c->sparse) {
    // A small instance is latency-bound: one block runs the whole enforcement
    // (rac_state: D, removal bits and column lists in shared memory,
    // __syncthreads as the pass barrier, an ordinary launch).
    StateParams sp = state_params(c, d_in, d_out, iters, status, flags);
    sp.seeds = seeds;
    sp.n_seeds = n_seeds;
    sp.removed_at = removed_at;
    if (getenv("RAC_DEBUG_TIMELINE") && !c->dbg) CK(c, cudaMalloc(&c->dbg, (256 + 3000) * 8));
    sp.dbg = c->dbg;
    if (c->tiny) CK(c, launch_tiny(c->W, sp, 1, tiny_smem(c->n, c->col_stride), s));
    else CK(c, launch_state(c->W, c->state_T, sp, 1, c->state_smem, s));
    c->launches++;
    return 0;
  }
  // R[1] (pass 1's removal buffer) is clean: zeroed at create and by the last
  // CTA of every previous launch.
  static const bool no_coop = getenv("RAC_NO_COOP") != nullptr;  // A/B knob (tooling only)
  // max_ctas > 0 (several ranks sharing a GPU): ordinary launch, co-residency
  // is the caller's sizing
  CK(c, launch_fused(c->W, c->sparse ? 0 : c->G, p, c->fused_grid, kernel_smem(c), s,
                     c->fused_grid > 1 && !no_coop && c->max_ctas == 0));
  c->launches++;
  return 0;
}

int enforce_sharded(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iters, int32_t* status,
                    int32_t* removed_at, uint32_t flags, cudaStream_t s, const int32_t* seeds = nullptr,
                    int n_seeds = -1) {
  const int total_g = c->world * c->blk;
  // world > 1: each rank's passes write the epochs of its own rows into a
  // padded [world*blk][64] buffer, all-gathered after the loop (collective)
  int32_t* ra = removed_at;
  if (removed_at && c->world > 1) {
    if (!c->ra_g) CK(c, cudaMalloc(&c->ra_g, (size_t)total_g * 64 * 4));
    ra = c->ra_g;
    CK(c, cudaMemsetAsync(ra, 0, (size_t)total_g * 64 * 4, s));
  } else if (removed_at) {
    CK(c, cudaMemsetAsync(removed_at, 0, (size_t)c->n * 64 * 4, s));
  }
  CK(c, launch_shard_init(c->sh, d_in, c->dommask, c->n, c->W, c->dbytes, total_g, s));
  c->launches++;
  if (n_seeds >= 0) {
    // seeded call: pass 1 tests Cons[:, seeds] (Alg. 1 @changed = seeds);
    // an empty list marks the call done with no pass
    CK(c, launch_shard_seed(c->sh, seeds, n_seeds, c->n, s));
    c->launches++;
  }
  const int nb = c->use_nccl() ? 1 : c->vshards;
  std::vector<PassParams> pp(nb);
  for (int b = 0; b < nb; ++b) {
    int lo, hi;
    if (c->use_nccl()) { lo = c->x_lo; hi = c->x_hi; }
    else rac_shard_range(c->n, c->vshards, b, &lo, &hi);
    pp[b].g = geom_for(c, lo, std::min(hi, c->n));
    pp[b].s = c->sh;
    pp[b].removed_at = ra;
  }
  const long max_passes = (long)c->n * c->dmax + 2;
  long enq = 0;
  int chunk = 1;  // a one-pass enforcement (W-stream) needs no speculative pass
  for (;;) {
    for (int k = 0; k < chunk; ++k) {
      for (int b = 0; b < nb; ++b) {
        if (pp[b].g.x_hi <= pp[b].g.x_lo) continue;
        CK(c, launch_pass(c->W, c->G, pp[b], c->pass_grid, kernel_smem(c), s));
        c->launches++;
      }
      if (c->use_nccl()) {
        CK(c, launch_shard_slice(c->sh, c->x_lo, c->x_lo + c->blk, c->n, s));
        c->launches++;
        ncclResult_t r = nccl().AllGather(c->sh.Dg + (size_t)c->rank * c->blk, c->sh.Dg, (size_t)c->blk,
                                          kNcclUint64, c->comm, s);
        if (r != 0)
          return fail(c, RAC_ENCCL, std::string("ncclAllGather: ") +
                                        (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
      } else {
        CK(c, launch_shard_slice(c->sh, 0, c->n, c->n, s));
        c->launches++;
      }
      CK(c, launch_shard_update(c->sh, c->n, c->W, flags, s));
      c->launches++;
    }
    enq += chunk;
    CK(c, cudaMemcpyAsync(c->h_scalars + 2, c->sh.done, 4, cudaMemcpyDeviceToHost, s));
    CK(c, cudaStreamSynchronize(s));
    if (c->h_scalars[2]) break;
    if (enq > max_passes) return fail(c, RAC_ECUDA, "sharded loop did not converge (internal error)");
    chunk = std::min(chunk * 2, 64);
  }
  CK(c, launch_shard_finalize(c->sh, c->n, d_out, iters, status, s));
  c->launches++;
  if (removed_at && c->world > 1) {
    ncclResult_t r = nccl().AllGather(ra + (size_t)c->rank * c->blk * 64, ra, (size_t)c->blk * 64, kNcclInt32, c->comm,
                                      s);
    if (r != 0)
      return fail(c, RAC_ENCCL, std::string("ncclAllGather(epochs): ") +
                                    (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
    CK(c, cudaMemcpyAsync(removed_at, ra, (size_t)c->n * 64 * 4, cudaMemcpyDeviceToDevice, s));
  }
  return 0;
}

int enforce_async_impl(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iters, int32_t* status,
                       int32_t* removed_at, uint32_t flags, cudaStream_t s, const int32_t* seeds = nullptr,
                       int n_seeds = -1) {
  if (flags & ~RAC_FULL_FIXPOINT) return fail(c, RAC_EINVAL, "unknown flags");
  CK(c, ensure_device(c));
  c->launches = 0;
  if (c->wide) return enforce_wide(c, d_in, d_out, iters, status, removed_at, flags, s, seeds, n_seeds);
  if (c->peer) {
    if (!c->connected) return fail(c, RAC_EINVAL, "RAC_OPT_PEER context: call rac_connect_peers first");
    // removal epochs are exchanged through the peers' epoch arrays (collective:
    // every rank passes removed_at or none does)
    return enforce_fused(c, d_in, d_out, iters, status, removed_at, flags, s, seeds, n_seeds);
  }
  if (c->use_nccl() || c->vshards > 1)
    return enforce_sharded(c, d_in, d_out, iters, status, removed_at, flags, s, seeds, n_seeds);
  return enforce_fused(c, d_in, d_out, iters, status, removed_at, flags, s, seeds, n_seeds);
}

}  // namespace

namespace {
// Full passes over every live row read the same bytes in either dense sweep, and
// which one streams faster depends on the box (profiles/r02an/r02ao: column
// sweep 88 vs row sweep 92 us on one B200, 110 vs 90 us on another, same C3
// W-stream).  So an HBM-resident single-GPU context times both once at create
// -- a root enforcement from full domains with ties sent to columns, then to
// rows, best of three -- and keeps the faster for ties (RAC_FORCE_LAYOUT
// overrides; RAC_NO_TIE_CALIB=1 keeps the row sweep without measuring).
void calibrate_tie(rac_ctx* c) {
  if (c->sparse || c->world > 1 || c->vshards > 1 || c->nccl_self || c->peer || !c->Mr || c->small ||
      c->force_layout != 0 || (double)c->rows_pad * c->dbytes <= 64.0 * (1 << 20))
    return;
  if (getenv("RAC_NO_TIE_CALIB")) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  float best[2] = {1e30f, 1e30f};  // [0] ties -> columns (force 3), [1] ties -> rows (force 0)
  int32_t* res = reinterpret_cast<int32_t*>(c->buf_scalars);
  for (int rep = 0; rep < 4; ++rep)
    for (int v = 0; v < 2; ++v) {
      c->force_layout = v == 0 ? 3 : 0;
      cudaEventRecord(e0, c->stream);
      if (enforce_fused(c, c->dommask, c->buf_out, res, res + 1, nullptr, 0u, c->stream) != 0) {
        c->force_layout = 0;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaGetLastError();
        c->broken = false;
        return;
      }
      cudaEventRecord(e1, c->stream);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best[v]) best[v] = ms;  // rep 0 warms up both
    }
  c->force_layout = best[0] < best[1] ? 3 : 0;
  c->tie_ms[0] = best[0];
  c->tie_ms[1] = best[1];
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// rac_create with max dom > 64: rows of relation r are dom[x] x wq words
// (wq = ceil(max dom / 64)); validated here, packed on the device.
int create_wide(int32_t n_vars, const int32_t* dom_sizes, int32_t n_rel, const rac_relation* rels,
                const rac_options* opt, rac_ctx** out) {
  int dmax = 0;
  for (int x = 0; x < n_vars; ++x) dmax = std::max(dmax, (int)dom_sizes[x]);
  const int wq = (dmax + 63) / 64;
  std::vector<int32_t> xs(n_rel), ys(n_rel);
  std::vector<uint64_t> keys(n_rel);
  std::vector<uint64_t> rows((size_t)std::max(n_rel, 1) * dmax * wq, 0ull);
  for (int r = 0; r < n_rel; ++r) {
    const int x = rels[r].x, y = rels[r].y;
    if (x < 0 || y < 0 || x >= n_vars || y >= n_vars || x == y || !rels[r].rows)
      return fail(nullptr, RAC_EINVAL, "relation " + std::to_string(r) + ": bad (x, y) or NULL rows");
    for (int a = 0; a < dom_sizes[x]; ++a)
      for (int w = 0; w < wq; ++w) {
        const uint64_t v = rels[r].rows[(size_t)a * wq + w];
        const int bits = std::min(64, std::max(0, dom_sizes[y] - 64 * w));
        const uint64_t dm = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
        if (v & ~dm) return fail(nullptr, RAC_EINVAL, "relation " + std::to_string(r) + ": bits beyond dom(y)");
        rows[((size_t)r * dmax + a) * wq + w] = v;
      }
    xs[r] = x;
    ys[r] = y;
    keys[r] = ((uint64_t)std::min(x, y) << 32) | (uint64_t)std::max(x, y);
  }
  std::sort(keys.begin(), keys.end());
  if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
    return fail(nullptr, RAC_EINVAL, "duplicate constraint on one unordered pair");
  rac_ctx* c = new rac_ctx();
  int rc = setup_wide(c, n_vars, dom_sizes, opt);
  if (rc) { free_ctx(c); return rc; }
  if (n_rel > 0) {
    int32_t *dxs = nullptr, *dys = nullptr;
    uint64_t* drows = nullptr;
    cudaError_t e = cudaMalloc(&dxs, (size_t)n_rel * 4);
    if (e == cudaSuccess) e = cudaMalloc(&dys, (size_t)n_rel * 4);
    if (e == cudaSuccess) e = cudaMalloc(&drows, rows.size() * 8);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dxs, xs.data(), (size_t)n_rel * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e == cudaSuccess) e = cudaMemcpyAsync(dys, ys.data(), (size_t)n_rel * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e == cudaSuccess) e = cudaMemcpyAsync(drows, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e == cudaSuccess) e = launch_wide_pack(wide_pack_geom(c, 0), dxs, dys, drows, n_rel, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(dxs);
    cudaFree(dys);
    cudaFree(drows);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(nullptr, RAC_ECUDA, std::string("packing relations: ") + cudaGetErrorString(e));
    }
  }
  *out = c;
  return 0;
}
}  // namespace

// ----------------------------------------------------------------------------- C ABI
extern "C" {

void rac_default_options(rac_options* opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
  opt->device = 0;
  opt->world = 1;
  opt->rank = 0;
  opt->virtual_shards = 0;
  opt->max_ctas = 0;
}

int rac_peer_region(const rac_ctx* c, void** region_dev) {
  if (!c || !region_dev) return RAC_EINVAL;
  *region_dev = c->xr;
  return 0;
}

int rac_peer_handle(const rac_ctx* c, void* out) {
  if (!c || !out) return RAC_EINVAL;
  if (!c->peer) return RAC_EINVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAC_ECUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->xr) != cudaSuccess) {
    cudaGetLastError();
    return RAC_ECUDA;
  }
  static_assert(sizeof(h) == RAC_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(out, &h, sizeof(h));
  return 0;
}

int rac_connect_peers(rac_ctx* c, const void* handles) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (c->wide) return fail(c, RAC_EUNSUPPORTED, "domains > 64 values: rac_enforce[_ex / _async / _seeded / _seeded_async] only");
  if (!handles || !c->peer) return fail(c, RAC_EINVAL, "rac_connect_peers needs a RAC_OPT_PEER context and handles");
  if (c->connected) return fail(c, RAC_EINVAL, "peers already connected");
  CK(c, cudaSetDevice(c->device));
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)q * RAC_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, RAC_EPEER, std::string("cudaIpcOpenMemHandle(rank ") + std::to_string(q) +
                                     "): " + cudaGetErrorString(e));
    }
    c->peer_base[q] = static_cast<uint8_t*>(ptr);
    c->peer_ipc[q] = true;
  }
  c->connected = true;
  return 0;
}

int rac_connect_peers_local(rac_ctx* c, void* const* regions, const int32_t* devices) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (c->wide) return fail(c, RAC_EUNSUPPORTED, "domains > 64 values: rac_enforce[_ex / _async / _seeded / _seeded_async] only");
  if (!regions || !devices || !c->peer)
    return fail(c, RAC_EINVAL, "rac_connect_peers_local needs a RAC_OPT_PEER context, regions and devices");
  if (c->connected) return fail(c, RAC_EINVAL, "peers already connected");
  if (regions[c->rank] != c->xr || devices[c->rank] != c->device)
    return fail(c, RAC_EINVAL, "regions[rank] / devices[rank] must be this context's");
  CK(c, cudaSetDevice(c->device));
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    if (!regions[q]) return fail(c, RAC_EINVAL, "NULL peer region");
    if (devices[q] != c->device) {
      int can = 0;
      CK(c, cudaDeviceCanAccessPeer(&can, c->device, devices[q]));
      if (!can) return fail(c, RAC_EUNSUPPORTED, "no peer access between the devices");
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else CK(c, e);
    }
    c->peer_base[q] = static_cast<uint8_t*>(regions[q]);
  }
  c->connected = true;
  return 0;
}

int rac_shard_range(int32_t n_vars, int32_t world, int32_t rank, int32_t* x_lo, int32_t* x_hi) {
  if (n_vars < 0 || world < 1 || rank < 0 || rank >= world || !x_lo || !x_hi) return RAC_EINVAL;
  const int blk = (n_vars + world - 1) / world;
  *x_lo = std::min(n_vars, rank * blk);
  *x_hi = std::min(n_vars, (rank + 1) * blk);
  return 0;
}

static int init_comm(rac_ctx* c, const rac_options* opt) {
  if (!c->use_nccl()) return 0;
  if (!nccl().loaded) return fail(nullptr, RAC_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  if (c->nccl_self) {
    if (nccl().GetUniqueId(&id) != 0) return fail(nullptr, RAC_ENCCL, "ncclGetUniqueId failed");
  } else {
    memcpy(id.internal, opt->nccl_unique_id, RAC_NCCL_ID_BYTES);
  }
  ncclResult_t r = nccl().CommInitRank(&c->comm, c->world, id, c->rank);
  if (r != 0) {
    c->comm = nullptr;
    return fail(nullptr, RAC_ENCCL,
                std::string("ncclCommInitRank: ") + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
  }
  return 0;
}

int rac_create(int32_t n_vars, const int32_t* dom_sizes, int32_t n_rel, const rac_relation* rels,
               const rac_options* opt, rac_ctx** out) {
  if (!out) return fail(nullptr, RAC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_vars < 1 || !dom_sizes || n_rel < 0 || (n_rel > 0 && !rels))
    return fail(nullptr, RAC_EINVAL, "bad n_vars / dom_sizes / rels");
  for (int x = 0; x < n_vars; ++x)
    if (dom_sizes[x] < 1 || dom_sizes[x] > RAC_MAX_DOM_WIDE)
      return fail(nullptr, RAC_EINVAL, "dom size outside [1,256]");
  int dmax = 0;
  for (int x = 0; x < n_vars; ++x) dmax = std::max(dmax, (int)dom_sizes[x]);
  if (dmax > RAC_MAX_DOM) return create_wide(n_vars, dom_sizes, n_rel, rels, opt, out);
  // validate relations: range, x != y, padding bits, duplicate unordered pairs
  std::vector<uint64_t> keys(n_rel);
  std::vector<int32_t> xs(n_rel), ys(n_rel);
  std::vector<uint64_t> rows((size_t)n_rel * dmax, 0ull);
  for (int r = 0; r < n_rel; ++r) {
    const int x = rels[r].x, y = rels[r].y;
    if (x < 0 || y < 0 || x >= n_vars || y >= n_vars || x == y || !rels[r].rows)
      return fail(nullptr, RAC_EINVAL, "relation " + std::to_string(r) + ": bad (x, y) or NULL rows");
    const uint64_t my = dom_mask(dom_sizes[y]);
    for (int a = 0; a < dom_sizes[x]; ++a) {
      const uint64_t v = rels[r].rows[a];
      if (v & ~my) return fail(nullptr, RAC_EINVAL, "relation " + std::to_string(r) + ": bits beyond dom(y)");
      rows[(size_t)r * dmax + a] = v;
    }
    xs[r] = x;
    ys[r] = y;
    keys[r] = ((uint64_t)std::min(x, y) << 32) | (uint64_t)std::max(x, y);
  }
  {
    std::vector<uint64_t> k2 = keys;
    std::sort(k2.begin(), k2.end());
    if (std::adjacent_find(k2.begin(), k2.end()) != k2.end())
      return fail(nullptr, RAC_EINVAL, "duplicate constraint on one unordered pair");
  }
  rac_ctx* c = new rac_ctx();
  int rc = setup_ctx(c, n_vars, dom_sizes, opt, (double)n_rel);
  if (rc) { free_ctx(c); return rc; }
  if (c->sparse) {
    uint64_t* drows = nullptr;
    cudaError_t e = n_rel > 0 ? cudaMalloc(&drows, rows.size() * 8) : cudaSuccess;
    if (e == cudaSuccess && n_rel > 0) e = cudaMemcpyAsync(drows, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e != cudaSuccess) {
      cudaFree(drows);
      free_ctx(c);
      return fail(nullptr, RAC_ENOMEM, std::string("relation upload: ") + cudaGetErrorString(e));
    }
    rc = build_sparse(c, xs, ys, drows, dmax, 0, 0u, 0ull);
    cudaFree(drows);
    if (rc) { free_ctx(c); return rc; }
  } else if (n_rel > 0) {
    int32_t *dxs = nullptr, *dys = nullptr;
    uint64_t* drows = nullptr;
    cudaError_t e = cudaMalloc(&dxs, (size_t)n_rel * 4);
    if (e == cudaSuccess) e = cudaMalloc(&dys, (size_t)n_rel * 4);
    if (e == cudaSuccess) e = cudaMalloc(&drows, rows.size() * 8);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dxs, xs.data(), (size_t)n_rel * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e == cudaSuccess) e = cudaMemcpyAsync(dys, ys.data(), (size_t)n_rel * 4, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    if (e == cudaSuccess) e = cudaMemcpyAsync(drows, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice, c->stream);  // stream-ordered (pageable H2D may outlive cudaMemcpy)
    PackGeom g{c->M, c->col_stride, c->Mr, (size_t)c->dbytes, c->W, c->n, c->dmax, c->x_lo, c->x_hi, c->P, c->pw,
               c->dom_d};
    if (e == cudaSuccess) e = launch_pack_relations(g, dxs, dys, drows, n_rel, dmax, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(dxs);
    cudaFree(dys);
    cudaFree(drows);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(nullptr, RAC_ECUDA, std::string("packing relations: ") + cudaGetErrorString(e));
    }
  }
  rc = init_comm(c, opt);
  if (rc) { free_ctx(c); return rc; }
  calibrate_tie(c);
  *out = c;
  return 0;
}

int rac_create_random(int32_t n_vars, int32_t d, uint64_t dens_q32, uint32_t t_q16, uint64_t seed,
                      const rac_options* opt, rac_ctx** out) {
  if (!out) return fail(nullptr, RAC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_vars < 1 || d < 1 || d > RAC_MAX_DOM_WIDE || dens_q32 > (1ull << 32) || t_q16 > 65536u)
    return fail(nullptr, RAC_EINVAL, "bad generator parameters");
  std::vector<int32_t> dom(n_vars, d);
  if (d > RAC_MAX_DOM) {
    rac_ctx* c = new rac_ctx();
    int rc = setup_wide(c, n_vars, dom.data(), opt);
    if (rc) { free_ctx(c); return rc; }
    cudaError_t e = launch_wide_generate(wide_pack_geom(c, dens_q32), d, t_q16, seed, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(nullptr, RAC_ECUDA, std::string("generating instance: ") + cudaGetErrorString(e));
    }
    *out = c;
    return 0;
  }
  rac_ctx* c = new rac_ctx();
  const double est_pairs = (double)dens_q32 / 4294967296.0 * 0.5 * (double)n_vars * (double)(n_vars - 1);
  int rc = setup_ctx(c, n_vars, dom.data(), opt, est_pairs);
  if (rc) { free_ctx(c); return rc; }
  if (c->sparse) {
    // the present pairs (x < y) from the generator's presence hash
    std::vector<int32_t> xs, ys;
    xs.reserve((size_t)(est_pairs * 1.05) + 16);
    ys.reserve((size_t)(est_pairs * 1.05) + 16);
    for (int x = 0; x < n_vars; ++x)
      for (int y = x + 1; y < n_vars; ++y)
        if (synth_present(seed, (uint32_t)n_vars, (uint32_t)x, (uint32_t)y, dens_q32)) {
          xs.push_back(x);
          ys.push_back(y);
        }
    rc = build_sparse(c, xs, ys, nullptr, 0, d, t_q16, seed);
    if (rc) { free_ctx(c); return rc; }
    rc = init_comm(c, opt);
    if (rc) { free_ctx(c); return rc; }
    *out = c;
    return 0;
  }
  PackGeom g{c->M, c->col_stride, c->Mr, (size_t)c->dbytes, c->W, c->n, c->dmax, c->x_lo, c->x_hi, c->P, c->pw,
               c->dom_d};
  cudaError_t e = launch_generate(g, d, dens_q32, t_q16, seed, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    free_ctx(c);
    return fail(nullptr, RAC_ECUDA, std::string("generating instance: ") + cudaGetErrorString(e));
  }
  rc = init_comm(c, opt);
  if (rc) { free_ctx(c); return rc; }
  calibrate_tie(c);
  *out = c;
  return 0;
}

int rac_enforce_async(rac_ctx* c, const uint64_t* d_in_dev, uint64_t* d_out_dev, int32_t* iterations_dev,
                      int32_t* status_dev, int32_t* removed_at_dev, uint32_t flags, void* stream) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (!d_in_dev || !d_out_dev || !iterations_dev || !status_dev) return fail(c, RAC_EINVAL, "NULL device buffer");
  return enforce_async_impl(c, d_in_dev, d_out_dev, iterations_dev, status_dev, removed_at_dev, flags,
                            (cudaStream_t)stream);
}

static int enqueue_blocking(rac_ctx* c, size_t nb, int n_seeds, uint32_t flags);

int rac_enforce_ex(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations, int32_t* removed_at,
                   uint32_t flags) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (!d_in || !d_out || !iterations) return fail(c, RAC_EINVAL, "NULL pointer");
  if (!bits_ok(c, d_in)) return fail(c, RAC_EINVAL, "d_in has bits beyond dom sizes");
  CK(c, ensure_device(c));
  const size_t nw = (size_t)c->n * c->wq, nb = nw * 8;
  memcpy(c->h_in, d_in, nb);
  int32_t* h_res = reinterpret_cast<int32_t*>(c->h_out + nw);
  int32_t* d_res = reinterpret_cast<int32_t*>(c->d_hout + nw);
  h_res[1] = -99;  // "no status reported" until the kernel writes one
  if (removed_at) {
    CK(c, cudaMemcpyAsync(c->buf_in, c->h_in, nb, cudaMemcpyHostToDevice, c->stream));
    rc = enforce_async_impl(c, c->buf_in, c->d_hout, d_res, d_res + 1, c->buf_removed, flags, c->stream);
  } else {
    rc = enqueue_blocking(c, nb, -1, flags);
  }
  if (rc) return rc;
  if (removed_at)
    CK(c, cudaMemcpyAsync(removed_at, c->buf_removed, (size_t)c->n * 64 * c->wq * 4, cudaMemcpyDeviceToHost,
                          c->stream));
  // (Polling the mapped status word instead was measured: the system-scope
  // fences it needs in the kernels cost more than the synchronise saves --
  // C1 W-seed device time 5.8 -> 9.8 us, profiles/r02u.)
  CK(c, cudaStreamSynchronize(c->stream));
  memcpy(d_out, c->h_out, nb);
  *iterations = h_res[0];
  const int st = h_res[1];
  if (st == RAC_EPEER) return fail(c, RAC_EPEER, "peer exchange timed out (a rank did not arrive)");
  if (st != RAC_OK && st != RAC_WIPEOUT) return fail(c, RAC_ECUDA, "kernel did not report a status");
  return st;
}

int rac_enforce(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations) {
  return rac_enforce_ex(c, d_in, d_out, iterations, nullptr, 0u);
}

int rac_enforce_seeded_async(rac_ctx* c, const uint64_t* d_in_dev, uint64_t* d_out_dev, int32_t* iterations_dev,
                             int32_t* status_dev, const int32_t* seeds_dev, int32_t n_seeds, uint32_t flags,
                             void* stream) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (!d_in_dev || !d_out_dev || !iterations_dev || !status_dev || n_seeds < 0 || (n_seeds > 0 && !seeds_dev))
    return fail(c, RAC_EINVAL, "bad seeded-enforcement arguments");
  return enforce_async_impl(c, d_in_dev, d_out_dev, iterations_dev, status_dev, nullptr, flags,
                            (cudaStream_t)stream, seeds_dev, n_seeds);
}

// Enqueue the blocking API's input and the enforcement writing into the mapped
// output, as a cached CUDA graph (per seed count and flags; dropped when the
// staging moves).  Small instances (the one-warp / one-block kernels, whose
// launch cost is comparable to the kernel) read d_in and the seeds straight
// from the pinned staging (zero-copy: no copy-engine transfer in the graph);
// larger ones stage them with one H2D copy, since every CTA of the persistent
// kernel reads d_in.
static int enqueue_blocking(rac_ctx* c, size_t nb, int n_seeds, uint32_t flags) {
  const size_t nw = (size_t)c->n * c->wq;
  int32_t* d_res = reinterpret_cast<int32_t*>(c->d_hout + nw);
  static const char* bg = getenv("RAC_BLOCKING_GRAPH");  // A/B knob (tooling only): "0" = no graph, "small"
  const bool no_graph = bg && strcmp(bg, "0") == 0;
  const bool small_only = bg && strcmp(bg, "small") == 0;
  static const bool h2d_small = getenv("RAC_BLOCKING_H2D") != nullptr;  // A/B knob: small instances copy too
  const bool zc = c->small && !c->peer && !c->wide && !h2d_small;
  const uint64_t* din = zc ? c->h_in : c->buf_in;  // pinned host memory is device-accessible (UVA)
  const int32_t* seeds =
      n_seeds >= 0 ? (zc ? reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(c->h_in) + nb)
                         : c->buf_seeds)
                   : nullptr;
  const size_t bytes = nb + (size_t)std::max(0, n_seeds) * 4;
  // d_in (+ seeds) reach device memory through a one-block kernel reading the
  // pinned staging: C3 W-stream blocking call 128.4 -> 122.7 us against the
  // copy-engine transfer (profiles/r02aj; A/B knob RAC_BLOCKING_COPY_ENGINE)
  static const bool stage_kernel = getenv("RAC_BLOCKING_COPY_ENGINE") == nullptr;
  auto enqueue = [&]() -> int {
    if (!zc) {
      // (bytes is a multiple of 4: 8-byte words, then 4-byte seeds)
      cudaError_t e = stage_kernel ? launch_stage_copy(c->h_in, c->buf_in, bytes, c->stream)
                                   : cudaMemcpyAsync(c->buf_in, c->h_in, bytes, cudaMemcpyHostToDevice, c->stream);
      if (e != cudaSuccess) return fail(c, RAC_ECUDA, std::string("input staging: ") + cudaGetErrorString(e));
    }
    return enforce_async_impl(c, din, c->d_hout, d_res, d_res + 1, nullptr, flags, c->stream, seeds, n_seeds);
  };
  if (c->peer || c->wide || c->graphs_off || no_graph || (small_only && !c->small)) return enqueue();
  const int64_t key = ((int64_t)n_seeds << 8) | (int64_t)flags;
  for (int i = 0; i < c->ngraphs; ++i)
    if (c->gkey[i] == key) {
      CK(c, cudaGraphLaunch(c->graphs[i], c->stream));
      c->launches = 1;
      return 0;
    }
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed);
  int rc = 0;
  if (e == cudaSuccess) {
    rc = enqueue();
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
    if (e == cudaSuccess) e = e2;
  }
  if (rc == 0 && e == cudaSuccess) e = cudaGraphInstantiate(&ex, g, 0);
  if (g) cudaGraphDestroy(g);
  if (rc != 0 || e != cudaSuccess) {
    // capture not possible here: remember, and run this call directly
    cudaGetLastError();
    c->broken = false;
    c->graphs_off = true;
    return enqueue();
  }
  if (c->ngraphs == rac_ctx::kGraphs) {
    cudaGraphExecDestroy(c->graphs[0]);
    for (int i = 1; i < c->ngraphs; ++i) {
      c->graphs[i - 1] = c->graphs[i];
      c->gkey[i - 1] = c->gkey[i];
    }
    --c->ngraphs;
  }
  c->graphs[c->ngraphs] = ex;
  c->gkey[c->ngraphs++] = key;
  CK(c, cudaGraphLaunch(ex, c->stream));
  c->launches = 1;
  return 0;
}

int rac_enforce_seeded(rac_ctx* c, const uint64_t* d_in, uint64_t* d_out, int32_t* iterations, const int32_t* seeds,
                       int32_t n_seeds, uint32_t flags) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (!d_in || !d_out || !iterations || n_seeds < 0 || (n_seeds > 0 && !seeds))
    return fail(c, RAC_EINVAL, "bad seeded-enforcement arguments");
  for (int i = 0; i < n_seeds; ++i)
    if (seeds[i] < 0 || seeds[i] >= c->n) return fail(c, RAC_EINVAL, "seed out of range");
  if (!bits_ok(c, d_in)) return fail(c, RAC_EINVAL, "d_in has bits beyond dom sizes");
  CK(c, ensure_device(c));
  const size_t nw = (size_t)c->n * c->wq, nb = nw * 8;
  if ((size_t)n_seeds > c->seed_cap) {
    CK(c, cudaStreamSynchronize(c->stream));  // the staging buffers may still be in use
    CK(c, alloc_staging(c, nb, std::max<size_t>((size_t)n_seeds, 2 * c->seed_cap)));
  }
  memcpy(c->h_in, d_in, nb);
  if (n_seeds > 0) memcpy(reinterpret_cast<uint8_t*>(c->h_in) + nb, seeds, (size_t)n_seeds * 4);
  int32_t* h_res = reinterpret_cast<int32_t*>(c->h_out + nw);
  h_res[1] = -99;
  rc = enqueue_blocking(c, nb, n_seeds, flags);
  if (rc) return rc;
  CK(c, cudaStreamSynchronize(c->stream));
  memcpy(d_out, c->h_out, nb);
  *iterations = h_res[0];
  const int st = h_res[1];
  if (st == RAC_EPEER) return fail(c, RAC_EPEER, "peer exchange timed out (a rank did not arrive)");
  if (st != RAC_OK && st != RAC_WIPEOUT) return fail(c, RAC_ECUDA, "kernel did not report a status");
  return st;
}

static int batch_impl(rac_ctx* c, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                      int32_t* iterations_dev, int32_t* status_dev, const int32_t* seed_var_dev, uint32_t flags,
                      void* stream);

// Batched enforcement on wide domains (d <= 128) with the tensor-core pass:
// every pass is ONE dense contraction of all states against every column
// (wide_tc_pass, the winner of the A/B in DESIGN.md section 8), followed by
// per-state loop control (wide_tc_update: wipeout first, then changed; a
// stopped state is frozen).  Testing every column in every pass is a superset
// of Alg. 1's @changed columns, so seeded states (under rac_enforce_seeded's
// precondition) and root states get their exact results (Prop. 2, reading
// R12).  The host reads the count of running states once per pass.
static int wide_tc_enforce(rac_ctx* c, int32_t S, const uint64_t* d_in, uint64_t* d_out, int32_t* iters,
                           int32_t* status, uint32_t flags, cudaStream_t st) {
  CK(c, ensure_device(c));
  const size_t nw = (size_t)c->n * c->wq;
  const int rows = c->n * c->dmax, rows4 = (rows + 3) & ~3, NW = (S + 31) / 32;
  const size_t need = (size_t)S * nw * 8 + (size_t)NW * rows4 * 4 * 2 + (size_t)S * 4 + 16;
  if (need > c->tc_cap) {
    cudaFree(c->tc_buf);
    c->tc_buf = nullptr;
    CK(c, cudaMalloc(&c->tc_buf, need));
    c->tc_cap = need;
  }
  uint8_t* b = c->tc_buf;
  uint64_t* Dn = reinterpret_cast<uint64_t*>(b);
  uint32_t* X = reinterpret_cast<uint32_t*>(b + (size_t)S * nw * 8);
  int32_t* active = reinterpret_cast<int32_t*>(X + (size_t)NW * rows4 * 2);
  int32_t* n_active = active + S;
  // fp8 e4m3 0/1 operands by default (measured 2.76 vs 3.06 ms per pass at n=200, d=128, 1024 states;
  // profiles/r02o); A/B knob RAC_WIDE_TC=f16
  const char* f8e = getenv("RAC_WIDE_TC");
  const int impl = (f8e && strcmp(f8e, "f16") == 0) ? 3 : 4;
  CK(c, launch_wide_mask_copy(d_in, c->dom_d, S, c->n, c->wq, d_out, st));  // d_out holds D_{t-1}
  CK(c, cudaMemsetAsync(iters, 0, (size_t)S * 4, st));
  CK(c, cudaMemsetAsync(status, 0, (size_t)S * 4, st));
  CK(c, launch_fill_i32(active, 1, S, st));
  c->launches += 2;
  const long max_passes = (long)c->n * c->dmax + 2;
  for (long t = 1; t <= max_passes; ++t) {
    WideTcParams w{reinterpret_cast<const uint64_t*>(c->M), c->P, c->pw, c->dom_d, c->n, c->dmax, c->wq, c->WS, S,
                   d_out, Dn, X, X + (size_t)NW * rows4, rows4, NW};
    CK(c, launch_wide_pass_eval(impl, w, st));
    CK(c, cudaMemsetAsync(n_active, 0, 4, st));
    CK(c, launch_wide_tc_update(c->dom_d, c->n, c->wq, (flags & RAC_FULL_FIXPOINT) ? 1 : 0, d_out, Dn, active, iters,
                                status, n_active, S, st));
    c->launches += 3;
    CK(c, cudaMemcpyAsync(c->h_scalars + 3, n_active, 4, cudaMemcpyDeviceToHost, st));
    CK(c, cudaStreamSynchronize(st));
    if (c->h_scalars[3] == 0) return 0;
  }
  return fail(c, RAC_ECUDA, "wide tensor-core batch did not converge (internal error)");
}

int rac_enforce_batch_seeded(rac_ctx* c, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                             int32_t* iterations_dev, int32_t* status_dev, const int32_t* seed_var_dev,
                             uint32_t flags, void* stream) {
  if (n_states > 0 && !seed_var_dev) return fail(c, RAC_EINVAL, "seed_var_dev is NULL");
  return batch_impl(c, n_states, d_in_dev, d_out_dev, iterations_dev, status_dev, seed_var_dev, flags, stream);
}

int rac_enforce_batch(rac_ctx* c, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                      int32_t* iterations_dev, int32_t* status_dev, uint32_t flags, void* stream) {
  return batch_impl(c, n_states, d_in_dev, d_out_dev, iterations_dev, status_dev, nullptr, flags, stream);
}

static int batch_impl(rac_ctx* c, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                      int32_t* iterations_dev, int32_t* status_dev, const int32_t* seed_var_dev, uint32_t flags,
                      void* stream) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (n_states < 0 || (n_states > 0 && (!d_in_dev || !d_out_dev || !iterations_dev || !status_dev)))
    return fail(c, RAC_EINVAL, "bad batch arguments");
  if (flags & ~RAC_FULL_FIXPOINT) return fail(c, RAC_EINVAL, "unknown flags");
  if (c->wide) {
    // wide domains (NEXT-4)
    c->launches = 0;
    if (n_states == 0) return 0;
    const char* wb = getenv("RAC_WIDE_BATCH");  // A/B knob (tooling only): "state" | "tc"
    const bool want_tc = wb ? strcmp(wb, "tc") == 0 : (c->dmax <= 128 && n_states >= 256);
    if (want_tc && c->dmax <= 128) return wide_tc_enforce(c, n_states, d_in_dev, d_out_dev, iterations_dev,
                                                          status_dev, flags, (cudaStream_t)stream);
    // one block per state (wide_state)
    if (wide_state_smem(c->n, c->WS) > 200 * 1024)
      return fail(c, RAC_EUNSUPPORTED, "wide batched mode: n too large for the per-state shared memory");
    CK(c, ensure_device(c));
    WideStateParams w{reinterpret_cast<const uint64_t*>(c->M), c->P, c->dom_d, c->n, c->dmax, c->wq, c->WS, c->pw,
                      (flags & RAC_FULL_FIXPOINT) ? 1 : 0, d_in_dev, d_out_dev, iterations_dev, status_dev,
                      seed_var_dev, 0};
    for (int s0 = 0; s0 < n_states; s0 += 65535) {
      w.s0 = s0;
      CK(c, launch_wide_state(w, std::min(65535, n_states - s0), (cudaStream_t)stream));
      c->launches++;
    }
    return 0;
  }
  if (c->sparse) return fail(c, RAC_EUNSUPPORTED, "batched mode needs the dense layout (RAC_OPT_DENSE)");
  if (c->world > 1) return fail(c, RAC_EUNSUPPORTED, "batched mode runs per rank (world == 1 contexts)");
  c->launches = 0;
  if (n_states == 0) return 0;
  CK(c, cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const char* impl = getenv("RAC_BATCH_IMPL");  // A/B knob (tooling only): "state" = one block per state
  const bool want_state = impl && strcmp(impl, "state") == 0;
  if (want_state && c->state_smem > 0) {
    // One block per state (rac_state): no cross-state barrier, but every state
    // reads its own masks from L2 -- measured 1.2 ms vs 0.68 ms for the
    // bit-sliced kernel at C5 (profiles/r02b/ab_state.log), which shares each
    // mask load among 32 states.
    StateParams sp = state_params(c, d_in_dev, d_out_dev, iterations_dev, status_dev, flags);
    sp.seed_var = seed_var_dev;
    const int T = getenv("RAC_STATE_T") ? c->state_T : 128;
    // launches of at most 65535 blocks (the grid's x limit is larger, but the
    // state index arithmetic stays in int)
    for (int s0 = 0; s0 < n_states; s0 += 65535) {
      sp.s0 = s0;
      CK(c, launch_state(c->W, T, sp, std::min(65535, n_states - s0), c->state_smem, st));
      c->launches++;
    }
    return 0;
  }
  // Default for d <= 32: one bit-sliced 32-state word per thread-block cluster
  // (rac_batch_cl): cluster barriers and DSMEM exchange between the word's CTAs.
  const bool want_old_bs = impl && strcmp(impl, "bs") == 0;
  if (!want_old_bs && c->W <= 4) {
    const int rows_all = c->n * c->dmax;
    const char* ce = getenv("RAC_BATCH_CL");  // A/B knob (tooling only): cluster size
    int C = ce ? atoi(ce) : 4;
    C = std::max(1, std::min(C, (rows_all + 255) / 256));
    // a thread per row: enough CTAs that a CTA's rows fit its kBatchClThreads
    // threads (up to 16 per cluster; beyond that threads take several rows)
    C = std::min(16, std::max(C, (rows_all + kBatchClThreads - 1) / kBatchClThreads));
    // rows per CTA: whole variables, a multiple of 4 rows (16-byte DSMEM pushes)
    const int unit = c->dmax * 4 / std::gcd(c->dmax, 4);
    int RPC = (rows_all + C - 1) / C;
    RPC = (RPC + unit - 1) / unit * unit;
    C = (rows_all + RPC - 1) / RPC;
    const int threads = std::min(kBatchClThreads, (RPC + 31) / 32 * 32);
    const size_t smem = batch_cl_smem(c->n, c->dmax, c->W);
    int maxcl = 0;
    if (smem <= 200 * 1024) CK(c, batch_cl_max_clusters(c->W, C, threads, smem, &maxcl));
    if (maxcl >= 1) {
      BatchCLParams b{};
      b.M = c->M;
      b.col_stride = c->col_stride;
      // Per-column masks by default.  A/B knob RAC_CL_GROUPS=1: 8-byte column
      // groups (one coalesced 8-byte load per row tests 8/W columns), built from
      // the column-major tensor on the first such call -- measured slower at C5
      // (242 vs 232 us, profiles/r02ac: the heavy sweeps gain 3 %, the light
      // passes lose more testing whole groups for one listed column).
      const bool no_groups = !(getenv("RAC_CL_GROUPS") && atoi(getenv("RAC_CL_GROUPS")) == 1);  // per call
      const int cpg = 8 / c->W, ngr = (c->n + cpg - 1) / cpg;
      const size_t gbytes = (size_t)ngr * c->rows_pad * 8;
      if (!no_groups && !c->Mg && gbytes <= ((size_t)1 << 30)) {
        if (cudaMalloc(&c->Mg, gbytes) != cudaSuccess) {
          cudaGetLastError();
          c->Mg = nullptr;
        } else {
          CK(c, launch_pack_groups(c->M, c->col_stride, c->n, c->W, c->rows_pad, c->Mg, st));
        }
      }
      b.Mg = no_groups ? nullptr : c->Mg;
      b.gstride = (size_t)c->rows_pad * 8;
      // A/B knob (per call) RAC_CL_PS: per-state sweep for words with <= 8 active
      // states, 1 = when cheaper by a test count, 2 = always.  Off: measured 1.8x
      // slower at C5 (232 vs 421 us, profiles/r02al) -- each state pays its own
      // mask loads, which the 32-state union sweep shares.
      const char* pse = getenv("RAC_CL_PS");
      b.ps_mode = pse ? atoi(pse) : 0;
      b.n = c->n;
      b.dmax = c->dmax;
      b.P = c->P;
      b.pw = c->pw;
      b.dommask = c->dommask;
      b.d_in = d_in_dev;
      b.d_out = d_out_dev;
      b.iters = iterations_dev;
      b.status = status_dev;
      b.seed_var = seed_var_dev;
      b.S = n_states;
      b.RPC = RPC;
      b.flags = flags;
      const int NW = (n_states + 31) / 32;
      const int ncl = std::min(NW, maxcl);
      if (getenv("RAC_DEBUG_TIMELINE")) {
        if (!c->bs_dbg) CK(c, cudaMalloc(&c->bs_dbg, (size_t)4096 * 64 * 8));
        CK(c, cudaMemsetAsync(c->bs_dbg, 0, (size_t)4096 * 64 * 8, st));
        b.dbg = ncl <= 1024 ? c->bs_dbg : nullptr;
        c->bs_dbg_ctas = ncl * 4;  // 256 stamps per cluster
      }
      CK(c, launch_batch_cl(c->W, b, ncl, C, threads, smem, st));
      c->launches++;
      return 0;
    }
  }
  // Bit-sliced path (N5, r01 design): 32 states per 32-bit word, per-word CTA groups.
  const bool want_bs = true;
  const int rows = c->n * c->dmax;
  const int RB = (rows + 255) / 256;
  bool use_table = batch_bs_smem(c->n, c->dmax, c->W, true) <= 96 * 1024;
  const size_t smem = batch_bs_smem(c->n, c->dmax, c->W, use_table);
  int occ = 0;
  if (want_bs && smem <= 200 * 1024) CK(c, batch_bs_occupancy(c->W, smem, &occ));
  const int words_per_launch = occ > 0 ? (c->sm_count * occ) / RB : 0;
  if (want_bs && words_per_launch >= 1) {
    const int NWmax = std::min(words_per_launch, (n_states + 31) / 32);
    const size_t x2_bytes = (size_t)2 * NWmax * ((rows + 3) & ~3) * 4;
    if (x2_bytes > c->bs_X2_cap) {
      cudaFree(c->bs_X2);
      c->bs_X2 = nullptr;
      CK(c, cudaMalloc(&c->bs_X2, x2_bytes));
      c->bs_X2_cap = x2_bytes;
    }
    if ((size_t)NWmax * 4 > c->bs_bar_cap) {
      cudaFree(c->bs_bar);
      c->bs_bar = nullptr;
      CK(c, cudaMalloc(&c->bs_bar, (size_t)NWmax * 16));
      CK(c, cudaMemsetAsync(c->bs_bar, 0, (size_t)NWmax * 16, st));
      c->bs_bar_cap = (size_t)NWmax * 4;
    }
    for (int s0 = 0; s0 < n_states; s0 += 32 * NWmax) {
      BatchBSParams b{};
      b.M = c->M;
      b.col_stride = c->col_stride;
      b.Mr = c->Mr;
      b.row_bytes = c->dbytes;
      b.n = c->n;
      b.dmax = c->dmax;
      b.P = c->P;
      b.pw = c->pw;
      b.dommask = c->dommask;
      b.d_in = d_in_dev;
      b.d_out = d_out_dev;
      b.iters = iterations_dev;
      b.status = status_dev;
      b.seed_var = seed_var_dev;
      b.S = std::min(n_states - s0, 32 * NWmax);
      b.s0 = s0;
      b.NW = (b.S + 31) / 32;
      b.RB = RB;
      b.use_table = use_table;
      b.X2 = c->bs_X2;
      b.bar = c->bs_bar;
      b.flags = flags;
      if (getenv("RAC_DEBUG_TIMELINE")) {
        if (!c->bs_dbg) CK(c, cudaMalloc(&c->bs_dbg, (size_t)4096 * 64 * 8));
        CK(c, cudaMemsetAsync(c->bs_dbg, 0, (size_t)4096 * 64 * 8, st));
        b.dbg = (size_t)b.NW * RB <= 4096 ? c->bs_dbg : nullptr;
        c->bs_dbg_ctas = b.NW * RB;
      }
      CK(c, launch_batch_bs(c->W, b, b.NW * RB, smem, st));
      c->launches++;
    }
    return 0;
  }
  // Per-state path: one CTA per state (reference design for comparison).
  BatchParams p{};
  p.g = geom_for(c, 0, c->n);
  p.dommask = c->dommask;
  p.d_in = d_in_dev;
  p.d_out = d_out_dev;
  p.iters = iterations_dev;
  p.status = status_dev;
  p.seed_var = seed_var_dev;
  p.flags = flags;
  const size_t smem1 = fused_smem(c->dbytes, c->n) + (size_t)c->n * 8;
  int occ1 = 0;
  CK(c, batch_occupancy(c->W, c->G, smem1, &occ1));
  if (occ1 < 1) return fail(c, RAC_EUNSUPPORTED, "batched kernel does not fit on an SM (n too large)");
  CK(c, launch_batch(c->W, c->G, p, n_states, smem1, st));
  c->launches = 1;
  return 0;
}

int rac_batch_pass_eval(rac_ctx* c, int32_t impl, int32_t n_states, const uint64_t* d_in_dev, uint64_t* d_out_dev,
                        void* stream) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (c->wide) {
    // wide domains: impl 2 = bit-sliced byte-table pass, impl 3 = tcgen05 pass (d <= 128)
    if (n_states < 1 || !d_in_dev || !d_out_dev || impl < 2 || impl > 4) return fail(c, RAC_EINVAL, "bad arguments");
    if (impl >= 3 && c->dmax > 128) return fail(c, RAC_EUNSUPPORTED, "tensor-core wide pass needs max dom <= 128");
    CK(c, ensure_device(c));
    const int rows = c->n * c->dmax, rows4 = (rows + 3) & ~3, NW = (n_states + 31) / 32;
    const size_t need = (size_t)2 * NW * rows4 * 4;
    if (need > c->eval_cap) {
      cudaFree(c->eval_buf);
      c->eval_buf = nullptr;
      CK(c, cudaMalloc(&c->eval_buf, need));
      c->eval_cap = need;
    }
    WideTcParams w{reinterpret_cast<const uint64_t*>(c->M), c->P, c->pw, c->dom_d, c->n, c->dmax, c->wq, c->WS,
                   n_states, d_in_dev, d_out_dev, c->eval_buf, c->eval_buf + (size_t)NW * rows4, rows4, NW};
    CK(c, launch_wide_pass_eval(impl, w, (cudaStream_t)stream));
    c->launches = impl == 2 ? 3 : 2;
    return 0;
  }
  if (n_states < 1 || !d_in_dev || !d_out_dev || (impl != 0 && impl != 1)) return fail(c, RAC_EINVAL, "bad arguments");
  if (c->use_nccl() || c->x_lo != 0 || c->x_hi != c->n) return fail(c, RAC_EUNSUPPORTED, "single-GPU contexts only");
  if (c->sparse) return fail(c, RAC_EUNSUPPORTED, "batched passes need the dense layout (RAC_OPT_DENSE)");
  if (impl == 1 && c->dmax > 16) return fail(c, RAC_EUNSUPPORTED, "tensor-core pass needs max dom <= 16");
  CK(c, cudaSetDevice(c->device));
  const int rows = c->n * c->dmax, rows4 = (rows + 3) & ~3, NW = (n_states + 31) / 32;
  const size_t need = (size_t)2 * NW * rows4 * 4;
  if (need > c->eval_cap) {
    cudaFree(c->eval_buf);
    c->eval_buf = nullptr;
    CK(c, cudaMalloc(&c->eval_buf, need));
    c->eval_cap = need;
  }
  TcPassParams p{};
  p.M = c->M;
  p.col_stride = c->col_stride;
  p.W = c->W;
  p.n = c->n;
  p.dmax = c->dmax;
  p.rows = rows;
  p.P = c->P;
  p.pw = c->pw;
  p.Xin = c->eval_buf;
  p.Xout = c->eval_buf + (size_t)NW * rows4;
  p.rows4 = rows4;
  p.NW = NW;
  CK(c, launch_batch_pass_eval(impl, p, d_in_dev, c->dommask, n_states, d_out_dev, (cudaStream_t)stream));
  c->launches = 3;
  return 0;
}

int rac_search(rac_ctx* c, const uint64_t* d_in, int64_t max_assignments, uint32_t flags, int32_t* solution,
               rac_search_stats* stats) {
  int rc = check_usable(c);
  if (rc) return rc;
  if (!d_in) return fail(c, RAC_EINVAL, "d_in is NULL");
  if (flags & ~(RAC_SEARCH_ALL | RAC_FULL_FIXPOINT)) return fail(c, RAC_EINVAL, "unknown flags");
  if (c->use_nccl() || c->vshards > 1) return fail(c, RAC_EUNSUPPORTED, "rac_search runs on fused single-GPU contexts");
  const int n = c->n, wq = c->wq;  // domain states are n x wq words (wq > 1: wide domains, NEXT-4)
  const size_t nw = (size_t)n * wq;
  rac_search_stats st;
  memset(&st, 0, sizeof(st));
  const uint32_t ef = flags & RAC_FULL_FIXPOINT;
  // root: tensorAC(Vars, [0 : |Vars|])
  std::vector<uint64_t> root(nw);
  int32_t it = 0;
  rc = rac_enforce_ex(c, d_in, root.data(), &it, nullptr, ef);
  if (rc < 0) return rc;
  st.root_iterations = it;
  st.root_status = rc;
  if (rc == RAC_WIPEOUT) {
    if (stats) *stats = st;
    return RAC_WIPEOUT;
  }
  // explicit DFS stack: frame k holds the domains of depth k and the variable
  // chosen there with its untried values (wq words)
  std::vector<uint64_t> doms((size_t)(n + 1) * nw);
  std::vector<int> fvar(n + 1);
  std::vector<uint64_t> ftodo((size_t)(n + 1) * wq);
  std::vector<char> assigned(n, 0);
  auto count = [&](const uint64_t* v) {
    int k = 0;
    for (int w = 0; w < wq; ++w) k += __builtin_popcountll(v[w]);
    return k;
  };
  auto first = [&](const uint64_t* v) {
    for (int w = 0; w < wq; ++w)
      if (v[w]) return 64 * w + __builtin_ctzll(v[w]);
    return -1;
  };
  auto pick = [&](const uint64_t* D) {
    int best = -1, bc = 1 << 30;
    for (int x = 0; x < n; ++x) {
      if (assigned[x]) continue;
      const int cnt = count(D + (size_t)x * wq);
      if (cnt < bc) { bc = cnt; best = x; }
    }
    return best;
  };
  auto open_frame = [&](int depth, const uint64_t* D) {
    fvar[depth] = pick(D);
    std::copy(D + (size_t)fvar[depth] * wq, D + (size_t)fvar[depth] * wq + wq, ftodo.begin() + (size_t)depth * wq);
    assigned[fvar[depth]] = 1;
  };
  std::copy(root.begin(), root.end(), doms.begin());
  int depth = 0;
  if (pick(doms.data()) < 0) return fail(c, RAC_EINVAL, "no variable to assign");
  open_frame(0, doms.data());
  bool found = false;
  int result = RAC_WIPEOUT;
  std::vector<uint64_t> child(nw);
  while (depth >= 0) {
    uint64_t* todo = ftodo.data() + (size_t)depth * wq;
    const int var = fvar[depth];
    const int val = first(todo);
    if (val < 0) {  // all values of var tried: backtrack
      assigned[var] = 0;
      --depth;
      continue;
    }
    if (max_assignments > 0 && st.assignments >= max_assignments) { result = RAC_BUDGET; break; }
    todo[val >> 6] &= ~(1ull << (val & 63));
    const uint64_t* parent = doms.data() + (size_t)depth * nw;
    std::copy(parent, parent + nw, child.begin());
    for (int w = 0; w < wq; ++w) child[(size_t)var * wq + w] = 0;
    child[(size_t)var * wq + (val >> 6)] = 1ull << (val & 63);  // assign: row overwrite
    int32_t seed = var;
    int32_t cit = 0;
    const auto t0 = std::chrono::steady_clock::now();
    rc = rac_enforce_seeded(c, child.data(), child.data(), &cit, &seed, 1, ef);
    st.enforce_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc < 0) return rc;
    st.assignments++;
    st.recurrences += cit;
    if (rc == RAC_WIPEOUT) { st.wipeouts++; continue; }
    if (depth + 1 > st.max_depth) st.max_depth = depth + 1;
    if (depth + 1 == n) {  // every variable assigned: a solution (Alg. 2 "find answer")
      st.solutions++;
      if (!found && solution)
        for (int x = 0; x < n; ++x) solution[x] = first(child.data() + (size_t)x * wq);
      found = true;
      if (!(flags & RAC_SEARCH_ALL)) { result = RAC_OK; break; }
      continue;
    }
    ++depth;
    std::copy(child.begin(), child.end(), doms.begin() + (size_t)depth * nw);
    open_frame(depth, child.data());
  }
  if (result != RAC_BUDGET && found) result = RAC_OK;
  if (stats) *stats = st;
  return result;
}

int32_t rac_n_vars(const rac_ctx* c) { return c ? c->n : RAC_EINVAL; }
int32_t rac_max_dom(const rac_ctx* c) { return c ? c->dmax : RAC_EINVAL; }
int32_t rac_mask_bytes(const rac_ctx* c) { return c ? c->W : RAC_EINVAL; }
int32_t rac_words_per_var(const rac_ctx* c) { return c ? c->wq : RAC_EINVAL; }
int64_t rac_relation_bytes(const rac_ctx* c) {
  if (!c) return RAC_EINVAL;
  if (c->sparse) return (int64_t)c->s_nblk * c->s_bbytes;
  if (c->wide) return (int64_t)c->n * c->dmax * c->n * c->WS * 8;
  return (int64_t)c->n * (int64_t)c->col_stride + (c->Mr ? (int64_t)c->rows_pad * c->dbytes : 0);
}
int32_t rac_layout(const rac_ctx* c) { return c ? (c->sparse ? RAC_LAYOUT_SPARSE : RAC_LAYOUT_DENSE) : RAC_EINVAL; }
int64_t rac_last_launch_count(const rac_ctx* c) { return c ? c->launches : RAC_EINVAL; }
int32_t rac_full_pass_layout(const rac_ctx* c, float* ms_cols, float* ms_rows) {
  if (!c) return RAC_EINVAL;
  if (ms_cols) *ms_cols = c->tie_ms[0];
  if (ms_rows) *ms_rows = c->tie_ms[1];
  return (c->force_layout == 2 || c->force_layout == 3 || !c->Mr) ? 1 : 0;
}
int32_t rac_path(const rac_ctx* c) {
  if (!c) return RAC_EINVAL;
  if (c->wide) return RAC_PATH_WIDE;
  if (c->peer) return RAC_PATH_PEER;
  if (c->use_nccl() || c->vshards > 1) return RAC_PATH_SHARDED;
  if (c->sparse) return RAC_PATH_SPARSE;
  return c->small ? RAC_PATH_ONE_BLOCK : RAC_PATH_FUSED;
}

int rac_local_range(const rac_ctx* c, int32_t* x_lo, int32_t* x_hi) {
  if (!c || !x_lo || !x_hi) return RAC_EINVAL;
  *x_lo = c->x_lo;
  *x_hi = c->x_hi;
  return 0;
}

int rac_read_row(const rac_ctx* cc, int32_t x, int32_t a, uint64_t* out_masks, uint8_t* out_present) {
  rac_ctx* c = const_cast<rac_ctx*>(cc);
  int rc = check_usable(c);
  if (rc) return rc;
  if (c->wide) return fail(c, RAC_EUNSUPPORTED, "domains > 64 values: rac_enforce[_ex / _async / _seeded / _seeded_async] only");
  if (x < c->x_lo || x >= c->x_hi || a < 0 || a >= c->dmax) return fail(c, RAC_EINVAL, "row not local");
  CK(c, cudaSetDevice(c->device));
  if (out_masks && c->sparse) {
    // arc blocks: the block of arc x -> y in column y (sorted by x), else all ones
    const uint64_t ones = c->W == 8 ? ~0ull : ((1ull << (8 * c->W)) - 1ull);
    for (int y = 0; y < c->n; ++y) {
      out_masks[y] = ones;
      const uint32_t* b0 = c->s_arc_h.data() + c->s_off_h[y];
      const uint32_t* b1 = c->s_arc_h.data() + c->s_off_h[y + 1];
      const uint32_t key = (uint32_t)x | ((uint32_t)y << 16);
      const uint32_t* it = std::lower_bound(b0, b1, key);
      if (it != b1 && *it == key) {
        uint64_t v = 0;
        CK(c, cudaMemcpy(&v, c->S + (size_t)(it - c->s_arc_h.data()) * c->s_bbytes + (size_t)a * c->W, c->W,
                         cudaMemcpyDeviceToHost));
        out_masks[y] = v;
      }
    }
  } else if (out_masks) {
    // column-major: the row's n masks are strided by col_stride
    std::vector<uint8_t> buf((size_t)c->n * c->W);
    const size_t r = (size_t)(x - c->x_lo) * c->dmax + a;
    CK(c, cudaMemcpy2D(buf.data(), c->W, c->M + r * c->W, c->col_stride, c->W, c->n, cudaMemcpyDeviceToHost));
    for (int y = 0; y < c->n; ++y) {
      uint64_t v = 0;
      for (int k = 0; k < c->W; ++k) v |= (uint64_t)buf[(size_t)y * c->W + k] << (8 * k);
      out_masks[y] = v;
    }
  }
  if (out_present) {
    std::vector<uint32_t> pb(c->pw);
    CK(c, cudaMemcpy(pb.data(), c->P + (size_t)(x - c->x_lo) * c->pw, (size_t)c->pw * 4, cudaMemcpyDeviceToHost));
    for (int y = 0; y < c->n; ++y) out_present[y] = (pb[y >> 5] >> (y & 31)) & 1u;
  }
  return 0;
}

// Tooling (not part of include/rac.h): phase timestamps of the last fused
// launch when RAC_DEBUG_TIMELINE is set.  Returns the number written.
int rac_debug_timeline(rac_ctx* c, unsigned long long* out, int cap) {
  if (!c || !c->dbg || !out) return 0;
  unsigned long long buf[256];
  if (cudaMemcpy(buf, c->dbg, sizeof(buf), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  int n = (int)std::min<unsigned long long>(buf[0], (unsigned long long)cap);
  for (int i = 0; i < n; ++i) out[i] = buf[1 + i];
  return n;
}

// Tooling: per-CTA (start, first-barrier arrival, end) stamps of the last fused launch.
int rac_debug_cta_stamps(rac_ctx* c, unsigned long long* out, int cap) {
  if (!c || !c->dbg || !out) return 0;
  const int cnt = std::min(cap, 3 * c->fused_grid);
  if (cudaMemcpy(out, c->dbg + 256, (size_t)cnt * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return cnt;
}

// Tooling: per-CTA pass-end timestamps of the last bit-sliced batch launch.
int rac_debug_batch_timeline(rac_ctx* c, unsigned long long* out, int cap) {
  if (!c || !c->bs_dbg || !out) return 0;
  const int cnt = std::min(cap, c->bs_dbg_ctas * 64);
  if (cudaMemcpy(out, c->bs_dbg, (size_t)cnt * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return cnt;
}

int rac_get_nccl_unique_id(void* out) {
  if (!out) return RAC_EINVAL;
  if (!nccl().loaded) return fail(nullptr, RAC_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != 0) return fail(nullptr, RAC_ENCCL, "ncclGetUniqueId failed");
  memcpy(out, id.internal, RAC_NCCL_ID_BYTES);
  return 0;
}

const char* rac_last_error(const rac_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

void rac_destroy(rac_ctx* c) { free_ctx(c); }

}  // extern "C"

// Tooling (not part of include/rac.h): copy a wide context's mask tensor and
// presence bitmap to the host (tools/wide_debug.py).
extern "C" int rac_debug_wide_dump(rac_ctx* c, uint64_t* M_out, uint32_t* P_out) {
  if (!c || !c->wide) return RAC_EINVAL;
  CK(c, cudaSetDevice(c->device));
  CK(c, cudaStreamSynchronize(c->stream));
  if (M_out)
    CK(c, cudaMemcpy(M_out, c->M, (size_t)c->n * c->dmax * c->n * c->WS * 8, cudaMemcpyDeviceToHost));
  if (P_out) CK(c, cudaMemcpy(P_out, c->P, (size_t)c->n * c->pw * 4, cudaMemcpyDeviceToHost));
  return 0;
}
