// Probe (tooling only): cost per round of software grid barriers on B200, as a
// function of the grid size: (0) one counter, release-add + relaxed polling
// (rac_fused's grid_sync); (1) the arrivals striped over K counters on
// different 128-byte lines, pollers read all K; (2) hierarchical: a cluster
// barrier, one arrival per cluster on a single counter, a cluster barrier.
#include <cstdio>
#include <cuda_runtime.h>

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

template <int K>
__global__ void __launch_bounds__(512, 1) probe(unsigned* bar, unsigned long long* out, int rounds, int mode, int csize) {
  const unsigned long long t0 = gtime();
  for (int r = 1; r <= rounds; ++r) {
    if (mode == 0) {
      __syncthreads();
      if (threadIdx.x == 0) {
        red_release_add(bar, 1u);
        while (ld_relaxed(bar) < gridDim.x * (unsigned)r) {
        }
        __threadfence();
      }
      __syncthreads();
    } else if (mode == 1) {
      __syncthreads();
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) red_release_add(bar + 32 * (blockIdx.x % K), 1u);
        // lane j < K polls counter j: its expected count is the number of CTAs striped onto it
        const unsigned j = threadIdx.x;
        const unsigned per = j < K ? (gridDim.x / K + (j < gridDim.x % K ? 1u : 0u)) * (unsigned)r : 0u;
        bool done = j >= K;
        while (!__all_sync(0xffffffffu, done)) {
          if (!done) done = ld_relaxed(bar + 32 * j) >= per;
        }
        __threadfence();
      }
      __syncthreads();
    } else {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      unsigned rank;
      asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
      if (rank == 0 && threadIdx.x == 0) {
        red_release_add(bar, 1u);
        const unsigned target = (gridDim.x / csize) * (unsigned)r;
        while (ld_relaxed(bar) < target) {
        }
        __threadfence();
      }
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
  const unsigned long long t1 = gtime();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  unsigned* bar;
  unsigned long long* out;
  cudaMalloc(&bar, 32 * 32 * 4);
  cudaMalloc(&out, 64);
  for (int grid : {8, 16, 32, 64, 148, 296, 592}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int K : {4, 8, 16}) {
        if (mode != 1 && K != 8) continue;
        for (int cs : {4, 8}) {
          if (mode != 2 && cs != 4) continue;
          cudaMemset(bar, 0, 32 * 32 * 4);
          int rounds = 2000;
          cudaLaunchConfig_t cfg = {};
          cfg.blockDim = dim3(512);
          cfg.gridDim = dim3(grid);
          cudaLaunchAttribute attr[2];
          attr[0].id = cudaLaunchAttributeCooperative;
          attr[0].val.cooperative = 1;
          attr[1].id = cudaLaunchAttributeClusterDimension;
          attr[1].val.clusterDim.x = mode == 2 ? cs : 1;
          attr[1].val.clusterDim.y = 1;
          attr[1].val.clusterDim.z = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 2;
          void* args[] = {&bar, &out, &rounds, &mode, &cs};
          const void* f = K == 4 ? (const void*)probe<4> : K == 8 ? (const void*)probe<8> : (const void*)probe<16>;
          cudaError_t le = cudaLaunchKernelExC(&cfg, f, args);
          cudaError_t se = cudaDeviceSynchronize();
          unsigned long long ns = 0;
          cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
          printf("{\"grid\": %d, \"mode\": \"%s\", \"K\": %d, \"cluster\": %d, \"launch\": \"%s\", \"sync\": \"%s\", "
                 "\"ns_per_barrier\": %.1f}\n",
                 grid, mode == 0 ? "one_counter" : mode == 1 ? "striped" : "hier_cluster", K, mode == 2 ? cs : 1,
                 cudaGetErrorString(le), cudaGetErrorString(se), ns / (double)rounds);
          cudaGetLastError();
        }
      }
    }
  }
  return 0;
}
