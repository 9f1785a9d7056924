// Microbenchmark: cost of a cooperative-groups grid barrier on this GPU
// (148 SMs).  Used to size the persistent FISTA design.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int *out) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    g.sync();
  }
  if (acc == -1) out[0] = acc;
}

// hand-rolled sense-reversal barrier: one atomic per CTA, spin on a flag
__global__ void k_flag(int iters, unsigned *count, volatile unsigned *gen, int *out) {
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned g0 = *gen;
      __threadfence();
      if (atomicAdd(count, 1) == gridDim.x - 1) {
        *count = 0;
        __threadfence();
        atomicAdd((unsigned *)gen, 1);
      } else {
        while (*gen == g0) {
        }
      }
      __threadfence();
    }
    __syncthreads();
  }
  if (acc == -1) out[0] = acc;
}

int main() {
  int *out;
  unsigned *cnt, *gen;
  cudaMalloc(&out, 4);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {146, 148, 296}) {
    for (int variant = 0; variant < 2; ++variant) {
      int iters = 2000;
      void *args0[] = {&iters, &out};
      void *args1[] = {&iters, &cnt, &gen, &out};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (variant == 0)
          cudaLaunchCooperativeKernel((void *)k_sync, grid, 256, args0, 0, 0);
        else
          cudaLaunchCooperativeKernel((void *)k_flag, grid, 256, args1, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid=%d %s: %.3f us per barrier (%s)\n", grid, variant ? "flag" : "cg::grid.sync",
             1000.f * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // back-to-back tiny kernel launches for comparison
  cudaEventRecord(a);
  for (int i = 0; i < 2000; ++i) k_sync<<<148, 256>>>(0, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel launch-to-launch: %.3f us\n", 1000.f * ms / 2000);
  return 0;
}
