// Probe (tooling only): can a cooperative launch carry a cluster dimension on
// this B200, how many co-resident clusters does a 512-thread CTA get, and what
// do a software grid barrier (release-add + polling, as rac_fused) and a
// hardware cluster barrier cost per round?
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(512, 1) probe(unsigned* bar, unsigned long long* out, int rounds, int mode) {
  extern __shared__ unsigned sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = gtime();
  for (int r = 1; r <= rounds; ++r) {
    if (mode == 0) {  // grid barrier
      __syncthreads();
      if (threadIdx.x == 0) {
        red_release_add(bar, 1u);
        while (ld_relaxed(bar) < gridDim.x * (unsigned)r) {
        }
        __threadfence();
      }
      __syncthreads();
    } else {  // cluster barrier
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
  const unsigned long long t1 = gtime();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned* bar;
  unsigned long long* out;
  cudaMalloc(&bar, 64);
  cudaMalloc(&out, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const size_t smem = 12 * 1024;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe, 512, smem);
  printf("{\"sms\": %d, \"occ_per_sm\": %d}\n", sms, occ);
  for (int C : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int maxcl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&maxcl, (const void*)probe, &cfg);
    for (int mode = 0; mode < 2; ++mode) {
      if (mode == 1 && C == 1) continue;
      cfg.gridDim = dim3(maxcl * C);
      cfg.numAttrs = 2;
      cudaMemset(bar, 0, 64);
      int rounds = 1000;
      void* args[] = {&bar, &out, &rounds, &mode};
      cudaError_t le = cudaLaunchKernelExC(&cfg, (const void*)probe, args);
      cudaError_t se = cudaDeviceSynchronize();
      unsigned long long ns = 0;
      cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
      printf("{\"cluster\": %d, \"max_clusters\": %d, \"occ_err\": \"%s\", \"grid\": %d, \"mode\": \"%s\", "
             "\"coop_launch\": \"%s\", \"sync\": \"%s\", \"ns_per_barrier\": %.1f}\n",
             C, maxcl, cudaGetErrorString(e), maxcl * C, mode ? "cluster" : "grid", cudaGetErrorString(le),
             cudaGetErrorString(se), ns / 1000.0);
      cudaGetLastError();
    }
  }
  return 0;
}
