// rac_batch_tc.cu -- tensor-core (tcgen05) formulation of one batched support
// pass, for the A/B against the bit-sliced kernel (BASELINE north star: "a
// batched mode that evaluates many domain states as one dense ... tensor-core
// contraction, used only where ncu shows it beats the bit-packed path").
//
// For a tile of 128 rows (x,a) and 256 states s, per column y:
//   C[(x,a), s] = Σ_b R_y[(x,a), b] · D_s[y, b]      (tcgen05.mma.kind::f16,
//                 A = 128 x 16 f16 0/1 from the masks c_xy|(x,a), B = 16 x 256
//                 f16 0/1 from the states, fp32 accumulator in TMEM)
// and the epilogue (tcgen05.ld) keeps (x,a) for state s iff C > 0 on every
// declared c_xy (Eq. 1).  Domain sizes <= 16 (K = 16).
// One CTA = 4 warps = 128 threads (thread = row = TMEM lane); the column loop
// is serialised (build A and B in smem -> MMA -> commit/mbarrier -> TMEM load):
// a measurement prototype, not the product path (rac_batch_bs is).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rac_internal.cuh"

namespace rac {

namespace {

constexpr int kTM = 128;  // rows per tile (MMA M)
constexpr int kTN = 256;  // states per tile (MMA N)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no-swizzle canonical layout: core matrices of 8 rows x 16 bytes;
// row i, K-chunk j (8 f16) at (i/8)*SBO + j*LBO + (i%8)*16 bytes.
constexpr uint32_t kLBO = 128, kSBO = 256;

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version (Blackwell)
  return d;                 // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}

// 8 f16 values (0 or 1) from 8 mask bits: f16 1.0 = 0x3C00
__device__ __forceinline__ uint4 bits_to_f16x8(uint32_t bits) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = (((bits >> (2 * k)) & 1u) ? 0x3C00u : 0u) | (((bits >> (2 * k + 1)) & 1u) ? 0x3C000000u : 0u);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace

__global__ void __launch_bounds__(128, 1) rac_batch_tc_pass(TcPassParams p) {
  __shared__ alignas(1024) uint8_t sA[kTM * 32];  // 128 rows x 16 f16
  __shared__ alignas(1024) uint8_t sB[kTN * 32];  // 256 states x 16 f16
  __shared__ alignas(8) uint64_t mbar;
  __shared__ uint32_t tmem_base_s;
  __shared__ uint32_t xs[kTN / 32][16];  // state slices of column y: [word][b]
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row0 = blockIdx.x * kTM;
  const int w0 = blockIdx.y * (kTN / 32);  // first state word of this tile
  const int row = row0 + tid;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(kTN >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
  const uint64_t adesc = make_desc(smem_u32(sA)), bdesc = make_desc(smem_u32(sB));
  const int xl = row < p.rows ? row / p.dmax : 0;
  uint32_t acc[kTN / 32];
#pragma unroll
  for (int k = 0; k < kTN / 32; ++k) acc[k] = 0xffffffffu;
  uint32_t phase = 0;
  for (int y = 0; y < p.n; ++y) {
    // A: my row's mask for column y -> 16 f16 in the canonical layout
    uint32_t m = 0;
    if (row < p.rows) {
      const uint8_t* mp = p.M + (size_t)y * p.col_stride + (size_t)row * p.W;
      m = p.W == 1 ? *mp : p.W == 2 ? *reinterpret_cast<const uint16_t*>(mp) : *reinterpret_cast<const uint32_t*>(mp);
    }
    {
      uint8_t* a = sA + (tid >> 3) * kSBO + (tid & 7) * 16;
      *reinterpret_cast<uint4*>(a) = bits_to_f16x8(m & 0xFFu);
      *reinterpret_cast<uint4*>(a + kLBO) = bits_to_f16x8((m >> 8) & 0xFFu);
    }
    // B: states 2*tid, 2*tid+1 of the tile; value b of y = bit of X[w][(y,b)]
    {
      const int k = tid >> 4, b = tid & 15, wv = w0 + k;  // 128 threads = 8 words x 16 values
      xs[k][b] = (wv < p.NW && b < p.dmax) ? __ldg(p.Xin + (size_t)wv * p.rows4 + y * p.dmax + b) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 2 * tid + h, bit = s & 31;
      uint32_t bits = 0;
#pragma unroll
      for (int b = 0; b < 16; ++b) bits |= ((xs[s >> 5][b] >> bit) & 1u) << b;
      uint8_t* bp = sB + (s >> 3) * kSBO + (s & 7) * 16;
      *reinterpret_cast<uint4*>(bp) = bits_to_f16x8(bits & 0xFFu);
      *reinterpret_cast<uint4*>(bp + kLBO) = bits_to_f16x8((bits >> 8) & 0xFFu);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t accumulate = 0u;  // D = A*B (fresh counts per column)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar)));
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: my lane's 256 counts, 32 columns per load
    const bool pres = row < p.rows && ((__ldg(p.P + (size_t)xl * p.pw + (y >> 5)) >> (y & 31)) & 1u);
#pragma unroll
    for (int k = 0; k < kTN / 32; ++k) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(k * 32);
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
      if (pres) acc[k] &= nz;  // only a declared c_xy removes (reading R2)
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM and smem operands are reused by the next column
  }
  if (row < p.rows) {
#pragma unroll
    for (int k = 0; k < kTN / 32; ++k) {
      const int wv = w0 + k;
      if (wv < p.NW) {
        const uint32_t cur = p.Xin[(size_t)wv * p.rows4 + row];
        p.Xout[(size_t)wv * p.rows4 + row] = cur & acc[k];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// Bit-sliced reference pass (same inputs/outputs, ALU, one thread per row and
// state word, all columns): the comparison partner of the tensor-core pass.
__global__ void __launch_bounds__(256) rac_batch_bs_pass(TcPassParams p) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int wv = blockIdx.y;
  if (row >= p.rows) return;
  const int xl = row / p.dmax;
  const uint32_t* X = p.Xin + (size_t)wv * p.rows4;
  uint32_t acc = 0xffffffffu;
  for (int y = 0; y < p.n; ++y) {
    const uint8_t* mp = p.M + (size_t)y * p.col_stride + (size_t)row * p.W;
    uint32_t m = p.W == 1 ? *mp : p.W == 2 ? *reinterpret_cast<const uint16_t*>(mp) : *reinterpret_cast<const uint32_t*>(mp);
    uint32_t sup = 0;
    for (; m; m &= m - 1) sup |= __ldg(X + y * p.dmax + (__ffs(m) - 1));
    if (((__ldg(p.P + (size_t)xl * p.pw + (y >> 5)) >> (y & 31)) & 1u)) acc &= sup;
  }
  p.Xout[(size_t)wv * p.rows4 + row] = X[row] & acc;
}

__global__ void rac_states_to_slices(const uint64_t* d_in, const uint64_t* dommask, int S, int n, int dmax,
                                     int rows4, uint32_t* X) {
  // warp per (word w, variable x): lane j = state 32w + j
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int NW = (S + 31) / 32;
  if (wid >= (long)NW * n) return;
  const int w = (int)(wid / n), x = (int)(wid - (long)w * n);
  const int s = 32 * w + lane;
  const uint64_t v = s < S ? d_in[(size_t)s * n + x] & dommask[x] : 0ull;
  for (int a = 0; a < dmax; ++a) {
    const uint32_t b = __ballot_sync(0xffffffffu, (v >> a) & 1ull);
    if (lane == 0) X[(size_t)w * rows4 + x * dmax + a] = b;
  }
}

__global__ void rac_slices_to_states(const uint32_t* X, int S, int n, int dmax, int rows4, uint64_t* d_out) {
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int NW = (S + 31) / 32;
  if (wid >= (long)NW * n) return;
  const int w = (int)(wid / n), x = (int)(wid - (long)w * n);
  uint64_t v = 0;
  for (int a = 0; a < dmax; ++a) v |= (uint64_t)((X[(size_t)w * rows4 + x * dmax + a] >> lane) & 1u) << a;
  const int s = 32 * w + lane;
  if (s < S) d_out[(size_t)s * n + x] = v;
}

cudaError_t launch_batch_pass_eval(int impl, const TcPassParams& p, const uint64_t* d_in, const uint64_t* dommask,
                                   int S, uint64_t* d_out, cudaStream_t st) {
  const long warps = (long)p.NW * p.n;
  const int tb = (int)((warps * 32 + 255) / 256);
  rac_states_to_slices<<<tb, 256, 0, st>>>(d_in, dommask, S, p.n, p.dmax, p.rows4, const_cast<uint32_t*>(p.Xin));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (impl == 1) {
    dim3 grid((p.rows + kTM - 1) / kTM, (p.NW * 32 + kTN - 1) / kTN);
    rac_batch_tc_pass<<<grid, 128, 0, st>>>(p);
  } else {
    dim3 grid((p.rows + 255) / 256, p.NW);
    rac_batch_bs_pass<<<grid, 256, 0, st>>>(p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  rac_slices_to_states<<<tb, 256, 0, st>>>(p.Xout, S, p.n, p.dmax, p.rows4, d_out);
  return cudaGetLastError();
}

}  // namespace rac
