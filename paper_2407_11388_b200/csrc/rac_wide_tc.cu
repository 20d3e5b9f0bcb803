// rac_wide_tc.cu -- ONE batched support pass on wide domains (d = 65..128), two
// ways, for the A/B behind the wide batched-mode choice (SURVEY §8(f) NEXT-4:
// "wider domains ... where N6's tensor-core path may finally win"; BASELINE
// north star: the tensor-core contraction is "used only where ncu shows it
// beats the bit-packed path").  Both compute, for S states and every row
// (x,a) of the instance, the states for which (x,a) keeps a support on every
// declared c_xy against D_s (Eq. 1, one step from D_0),
// as 32-state bit slices Xout[w][r]; wide_pass_finish turns them into D_1.
//
//   impl 2, bit-sliced ALU:  32 states per u32; per column y a byte table
//       T[c][v] = OR_{j : bit j of v} X[(y, 8c+j)]  (16 chunks x 256 entries in
//       shared memory), then a row's support for 32 states is the OR of 16
//       byte lookups of its 128-bit mask.
//   impl 3, tcgen05 tensor cores:  per column y,
//       C[(x,a), s] = Σ_b R_y[(x,a), b] · D_s[y, b]  over K = 128 (8 MMAs of
//       tcgen05.mma.cta_group::1.kind::f16, 0/1 operands, fp32 counts in TMEM),
//       tile 128 rows x 256 states; then count > 0 and AND over y in the
//       epilogue.  Warp-specialised and double-buffered: producer warps expand
//       the next column's masks and state bits into f16 operands while one
//       thread issues the MMAs of the current column and the epilogue warps
//       read the previous column's counts from the other TMEM accumulator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ bool pres(const uint32_t* P, int pw, int x, int y) {
  return (__ldg(P + (size_t)x * pw + (y >> 5)) >> (y & 31)) & 1u;
}

}  // namespace

// ---------------------------------------------------------------------------- state slices
// X[w][r] bit j = (x,a) in state 32w+j, r = x*dmax + a (rows4 stride).
__global__ void wide_states_to_slices(const uint64_t* d_in, const int32_t* dom, int S, int n, int dmax, int wq,
                                      int rows4, uint32_t* X) {
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int NW = (S + 31) / 32;
  if (wid >= (long)NW * n) return;
  const int w = (int)(wid / n), x = (int)(wid - (long)w * n);
  const int s = 32 * w + lane;
  for (int k = 0; k < wq; ++k) {
    const int bits = min(64, max(0, dom[x] - 64 * k));
    const uint64_t dm = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
    const uint64_t v = s < S ? d_in[(size_t)s * n * wq + (size_t)x * wq + k] & dm : 0ull;
    for (int b = 0; b < 64 && 64 * k + b < dmax; ++b) {
      const uint32_t bb = __ballot_sync(0xffffffffu, (v >> b) & 1ull);
      if (lane == 0) X[(size_t)w * rows4 + (size_t)x * dmax + 64 * k + b] = bb;
    }
  }
}

// D_1[s] = D_0[s] & (rows kept for s): thread per (state, variable).
__global__ void wide_pass_finish(const uint64_t* d_in, const int32_t* dom, const uint32_t* Xout, int S, int n,
                                 int dmax, int wq, int rows4, uint64_t* d_out) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)S * n) return;
  const int s = (int)(i / n), x = (int)(i - (long)s * n);
  const uint32_t* Xw = Xout + (size_t)(s >> 5) * rows4 + (size_t)x * dmax;
  for (int k = 0; k < wq; ++k) {
    const int bits = min(64, max(0, dom[x] - 64 * k));
    const uint64_t dm = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
    uint64_t keep = 0;
    for (int b = 0; b < 64 && 64 * k + b < dmax; ++b) keep |= (uint64_t)((Xw[64 * k + b] >> (s & 31)) & 1u) << b;
    d_out[(size_t)s * n * wq + (size_t)x * wq + k] = d_in[(size_t)s * n * wq + (size_t)x * wq + k] & dm & keep;
  }
}

// ---------------------------------------------------------------------------- impl 2: bit-sliced ALU
// grid (ceil(rows / blockDim), NW); thread = row; byte tables for one column at a time.
template <int WS>
__global__ void __launch_bounds__(1024) wide_bs_pass(WideTcParams p) {
  __shared__ uint32_t Tb[32 * 256];  // [chunk][byte value] (NC = dmax/8 <= 32 chunks)
  __shared__ uint32_t Xy[256];
  const int w = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = p.n * p.dmax, NC = (p.dmax + 7) / 8;
  const uint32_t* X = p.Xin + (size_t)w * p.rows4;
  const int x = r < rows ? r / p.dmax : 0;
  const uint64_t* row = p.M + (size_t)(r < rows ? r : 0) * p.n * WS;
  uint32_t acc = 0xffffffffu;
  for (int y = 0; y < p.n; ++y) {
    for (int b = threadIdx.x; b < 8 * NC; b += blockDim.x) Xy[b] = b < p.dmax ? __ldg(X + (size_t)y * p.dmax + b) : 0u;
    __syncthreads();
    for (int e = threadIdx.x; e < NC * 256; e += blockDim.x) {
      const int c = e >> 8, v = e & 255;
      uint32_t t = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if ((v >> j) & 1) t |= Xy[8 * c + j];
      Tb[e] = t;
    }
    __syncthreads();
    if (r < rows) {
      uint64_t m[WS];
#pragma unroll
      for (int k = 0; k < WS; ++k) m[k] = __ldg(row + (size_t)y * WS + k);
      uint32_t sup = 0;
      for (int c = 0; c < NC; ++c) sup |= Tb[(c << 8) | (uint32_t)((m[c >> 3] >> (8 * (c & 7))) & 255u)];
      if (pres(p.P, p.pw, x, y)) acc &= sup;  // only a declared c_xy removes (reading R2)
    }
    __syncthreads();
  }
  if (r < rows) p.Xout[(size_t)w * p.rows4 + r] = X[r] & acc;
}

// ---------------------------------------------------------------------------- impl 3: tcgen05
namespace {

constexpr int kTM = 128;     // rows per tile (MMA M)
constexpr int kTN = 256;     // states per tile (MMA N)
constexpr int kK = 128;      // values of y per column (K), 8 MMAs of K = 16
constexpr int kSlabA = kTM * 32;  // bytes of one K = 16 slab of A (128 rows x 16 f16)
constexpr int kSlabB = kTN * 32;
// f16 operands: K = 16 per MMA, 8 slabs per column; fp8 (e4m3): K = 32 per MMA,
// 4 slabs.  A slab row is 32 bytes either way.
template <bool F8> __host__ __device__ constexpr int slabs() { return F8 ? kK / 32 : kK / 16; }
template <bool F8> __host__ __device__ constexpr int stageA() { return kSlabA * slabs<F8>(); }  // 32 KB f16, 16 KB fp8
template <bool F8> __host__ __device__ constexpr int stageB() { return kSlabB * slabs<F8>(); }  // 64 KB f16, 32 KB fp8
constexpr int kStageA = kSlabA * (kK / 16);
constexpr int kStageB = kSlabB * (kK / 16);
// K-major, no-swizzle canonical layout inside a slab: core matrices of 8 rows x
// 16 bytes; row i, K-chunk j (8 f16) at (i/8)*256 + j*128 + (i%8)*16 bytes.
constexpr uint32_t kLBO = 128, kSBO = 256;

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version (Blackwell)
  return d;
}

// 8 f16 (0 or 1.0) from 8 bits
__device__ __forceinline__ uint4 f16x8(uint32_t bits) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = (((bits >> (2 * k)) & 1u) ? 0x3C00u : 0u) | (((bits >> (2 * k + 1)) & 1u) ? 0x3C000000u : 0u);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// 128 bits (2 words) -> row i of an operand tile, all 8 K-slabs (f16).  (A
// 256-entry shared-memory table of the 8 f16 of each byte was slower: random
// 16-byte lookups conflict on the banks -- profiles/r02n, 3.06 -> 4.09 ms.)
__device__ __forceinline__ void put_row(uint8_t* base, int slab_bytes, int i, uint64_t lo, uint64_t hi) {
  uint8_t* p = base + (i >> 3) * kSBO + (i & 7) * 16;
#pragma unroll
  for (int sl = 0; sl < kK / 16; ++sl) {
    const uint64_t word = sl < 4 ? lo : hi;
    const uint32_t bits16 = (uint32_t)(word >> (16 * (sl & 3))) & 0xFFFFu;
    *reinterpret_cast<uint4*>(p + sl * slab_bytes) = f16x8(bits16 & 0xFFu);
    *reinterpret_cast<uint4*>(p + sl * slab_bytes + kLBO) = f16x8(bits16 >> 8);
  }
}

// 8 bits -> 8 fp8 e4m3 (0 or 1.0 = 0x38) with a few 64-bit ALU operations:
// replicate the byte, keep bit j in byte j, turn each non-zero byte into 0x01,
// scale to 0x38 (no carries: 0x38 < 0x100)
__device__ __forceinline__ unsigned long long fp8x8(uint32_t bits) {
  unsigned long long t = ((unsigned long long)(bits & 255u) * 0x0101010101010101ull) & 0x8040201008040201ull;
  t = (((t + 0x7F7F7F7F7F7F7F7Full) | t) >> 7) & 0x0101010101010101ull;
  return t * 0x38ull;
}

// fp8: 128 bits -> row i, 4 K-slabs of 32 elements, each two 16-element chunks
__device__ __forceinline__ void put_row8(uint8_t* base, int slab_bytes, int i, uint64_t lo, uint64_t hi) {
  uint8_t* p = base + (i >> 3) * kSBO + (i & 7) * 16;
#pragma unroll
  for (int sl = 0; sl < kK / 32; ++sl) {
    const uint32_t b32 = (uint32_t)((sl < 2 ? lo : hi) >> (32 * (sl & 1)));
    *reinterpret_cast<ulonglong2*>(p + sl * slab_bytes) = make_ulonglong2(fp8x8(b32), fp8x8(b32 >> 8));
    *reinterpret_cast<ulonglong2*>(p + sl * slab_bytes + kLBO) = make_ulonglong2(fp8x8(b32 >> 16), fp8x8(b32 >> 24));
  }
}

__device__ __forceinline__ void mbar_init1(uint64_t* mb, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mb)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait1(uint64_t* mb, uint32_t parity) {
  const uint32_t a = su32(mb);
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

}  // namespace

// 288 threads: warps 0-3 producers (thread i = row i of the tile and states
// 2i, 2i+1), warps 4-7 epilogue (thread = row = TMEM lane), warp 8 lane 0 issues
// the MMAs.  Dynamic smem: 2 stages x (A 32 KB + B 64 KB).
template <bool F8>
__global__ void __launch_bounds__(288, 1) wide_tc_pass(WideTcParams p) {
  extern __shared__ __align__(1024) uint8_t tsm[];
  __shared__ alignas(8) uint64_t full_bar[2], done_bar[2], free_bar[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int rows = p.n * p.dmax;
  const int row0 = blockIdx.x * kTM;
  const int s0 = blockIdx.y * kTN;
  constexpr int SA = stageA<F8>(), SB = stageB<F8>();
  uint8_t* sA[2] = {tsm, tsm + SA + SB};
  uint8_t* sB[2] = {tsm + SA, tsm + 2 * SA + SB};
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init1(&full_bar[i], 128);
      mbar_init1(&done_bar[i], 1);
      mbar_init1(&free_bar[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp < 4) {
    // ---- producers
    const int i = tid;  // row of the tile, states 2i and 2i+1
    const int r = row0 + i;
    for (int y = 0; y < p.n; ++y) {
      const int st = y & 1;
      if (y >= 2) mbar_wait1(&done_bar[st], (uint32_t)(((y - 2) >> 1) & 1));  // stage consumed by MMA y-2
      uint64_t lo = 0, hi = 0;
      if (r < rows) {
        const uint64_t* mp = p.M + ((size_t)r * p.n + y) * 2;
        lo = __ldg(mp);
        hi = __ldg(mp + 1);
      }
      if constexpr (F8) put_row8(sA[st], kSlabA, i, lo, hi);
      else put_row(sA[st], kSlabA, i, lo, hi);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = s0 + 2 * i + h;
        uint64_t a = 0, b = 0;
        if (s < p.S) {
          const uint64_t* dp = p.d_in + (size_t)s * p.n * p.wq + (size_t)y * p.wq;
          // bits beyond dom(y) meet only all-ones masks of absent pairs, which
          // the presence test ignores: no masking needed
          a = __ldg(dp);
          b = p.wq > 1 ? __ldg(dp + 1) : 0ull;
        }
        if constexpr (F8) put_row8(sB[st], kSlabB, 2 * i + h, a, b);
        else put_row(sB[st], kSlabB, 2 * i + h, a, b);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
      mbar_arrive1(&full_bar[st]);
    }
  } else if (warp < 8) {
    // ---- epilogue: thread = TMEM lane = row of the tile
    const int lane_row = (warp - 4) * 32 + (tid & 31);
    const int r = row0 + lane_row;
    const int x = r < rows ? r / p.dmax : 0;
    uint32_t acc[kTN / 32];
#pragma unroll
    for (int k = 0; k < kTN / 32; ++k) acc[k] = 0xffffffffu;
    for (int y = 0; y < p.n; ++y) {
      const int ab = y & 1;
      mbar_wait1(&done_bar[ab], (uint32_t)((y >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const bool pr = r < rows && pres(p.P, p.pw, x, y);
#pragma unroll
      for (int k = 0; k < kTN / 32; ++k) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)((warp - 4) * 32) << 16) + (uint32_t)(ab * kTN + k * 32);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t nz = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) nz |= (v[j] != 0u ? 1u : 0u) << j;  // fp32 count > 0
        if (pr) acc[k] &= nz;  // only a declared c_xy removes (reading R2)
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive1(&free_bar[ab]);  // accumulator ab may be overwritten (column y+2)
    }
    if (r < rows) {
#pragma unroll
      for (int k = 0; k < kTN / 32; ++k) {
        const int wv = (s0 >> 5) + k;
        if (wv < p.NW) p.Xout[(size_t)wv * p.rows4 + r] = acc[k];
      }
    }
  } else if ((tid & 31) == 0) {
    // ---- MMA issuer
    const uint32_t idesc = (1u << 4) | ((uint32_t)(kTN >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
    for (int y = 0; y < p.n; ++y) {
      const int st = y & 1;
      mbar_wait1(&full_bar[st], (uint32_t)((y >> 1) & 1));
      if (y >= 2) mbar_wait1(&free_bar[st], (uint32_t)(((y - 2) >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t d_tmem = tmem + (uint32_t)(st * kTN);
#pragma unroll
      for (int sl = 0; sl < slabs<F8>(); ++sl) {
        const uint64_t adesc = make_desc(su32(sA[st] + sl * kSlabA));
        const uint64_t bdesc = make_desc(su32(sB[st] + sl * kSlabB));
        const uint32_t accum = sl > 0 ? 1u : 0u;
        if constexpr (F8) {
          // e4m3 x e4m3 -> f32: the a/b format fields of idesc are 0 (E4M3) as for f16
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
              "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
              "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(&done_bar[st])));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------- batched enforcement
// Per-state loop control after one tensor-core pass (Alg. 1):
// Dn = D_t of every state (the pass ran on all of them), Dc = D_{t-1}.  An
// active state counts the pass; wipeout is checked first, then "changed"; a
// state that stops keeps D_t (its result) and is frozen; an active one that
// continues adopts D_t.  One block per state; *n_active counts the states still
// running (the host reads it once per pass).
__global__ void __launch_bounds__(256) wide_tc_update(const int32_t* dom, int n, int wq, int full, uint64_t* Dc,
                                                      const uint64_t* Dn, int32_t* active, int32_t* iters,
                                                      int32_t* status, int32_t* n_active) {
  const int s = blockIdx.x;
  if (!active[s]) return;  // block-uniform
  const size_t base = (size_t)s * n * wq;
  int changed = 0, empty = 0;
  for (int x = threadIdx.x; x < n; x += blockDim.x) {
    uint64_t any = 0;
    for (int k = 0; k < wq; ++k) {
      const uint64_t a = Dc[base + (size_t)x * wq + k], b = Dn[base + (size_t)x * wq + k];
      changed |= a != b;
      any |= b;
    }
    empty |= any == 0ull;
  }
  changed = __syncthreads_or(changed);
  empty = __syncthreads_or(empty);
  for (int i = threadIdx.x; i < n * wq; i += blockDim.x) Dc[base + i] = Dn[base + i];  // D_t (result or next input)
  if (threadIdx.x == 0) {
    iters[s] += 1;
    if (empty && !full) {
      status[s] = 1;  // RAC_WIPEOUT, Alg. 1
      active[s] = 0;
    } else if (!changed) {
      status[s] = empty ? 1 : 0;  // Prop. 1 end condition
      active[s] = 0;
    } else {
      atomicAdd(n_active, 1);
    }
  }
}

// Dc = d_in with the bits beyond each domain cleared (every state)
__global__ void wide_mask_copy(const uint64_t* d_in, const int32_t* dom, int S, int n, int wq, uint64_t* Dc) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)S * n * wq) return;
  const int k = (int)(i % wq), x = (int)((i / wq) % n);
  const int bits = min(64, max(0, dom[x] - 64 * k));
  Dc[i] = d_in[i] & (bits >= 64 ? ~0ull : ((1ull << bits) - 1ull));
}

cudaError_t launch_wide_mask_copy(const uint64_t* d_in, const int32_t* dom, int S, int n, int wq, uint64_t* Dc,
                                  cudaStream_t st) {
  const long tot = (long)S * n * wq;
  wide_mask_copy<<<(int)((tot + 255) / 256), 256, 0, st>>>(d_in, dom, S, n, wq, Dc);
  return cudaGetLastError();
}

__global__ void fill_i32(int32_t* p, int32_t v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

cudaError_t launch_fill_i32(int32_t* p, int32_t v, int n, cudaStream_t st) {
  fill_i32<<<(n + 255) / 256, 256, 0, st>>>(p, v, n);
  return cudaGetLastError();
}

cudaError_t launch_wide_tc_update(const int32_t* dom, int n, int wq, int full, uint64_t* Dc, const uint64_t* Dn,
                                  int32_t* active, int32_t* iters, int32_t* status, int32_t* n_active, int S,
                                  cudaStream_t st) {
  wide_tc_update<<<S, 256, 0, st>>>(dom, n, wq, full, Dc, Dn, active, iters, status, n_active);
  return cudaGetLastError();
}

size_t wide_tc_smem(bool f8) { return (size_t)2 * (f8 ? stageA<true>() + stageB<true>() : kStageA + kStageB); }

cudaError_t launch_wide_pass_eval(int impl, const WideTcParams& p, cudaStream_t st) {
  const int rows = p.n * p.dmax;
  const long warps = (long)p.NW * p.n;
  const int tb = (int)((warps * 32 + 255) / 256);
  if (impl == 2) {
    wide_states_to_slices<<<tb, 256, 0, st>>>(p.d_in, p.dom, p.S, p.n, p.dmax, p.wq, p.rows4,
                                              const_cast<uint32_t*>(p.Xin));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid((rows + 1023) / 1024, p.NW);
    if (p.WS == 2) wide_bs_pass<2><<<grid, 1024, 0, st>>>(p);
    else wide_bs_pass<4><<<grid, 1024, 0, st>>>(p);
  } else {
    const bool f8 = impl == 4;
    const size_t smem = wide_tc_smem(f8);
    const void* k = f8 ? (const void*)wide_tc_pass<true> : (const void*)wide_tc_pass<false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((rows + kTM - 1) / kTM, (p.S + kTN - 1) / kTN);
    if (f8) wide_tc_pass<true><<<grid, 288, smem, st>>>(p);
    else wide_tc_pass<false><<<grid, 288, smem, st>>>(p);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long th = (long)p.S * p.n;
  wide_pass_finish<<<(int)((th + 255) / 256), 256, 0, st>>>(p.d_in, p.dom, p.Xout, p.S, p.n, p.dmax, p.wq, p.rows4,
                                                           p.d_out);
  return cudaGetLastError();
}

}  // namespace rac
