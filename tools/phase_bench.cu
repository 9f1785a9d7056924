// Microbenchmark: latency of a "phase" (dependent L2 loads + warp reduction)
// between cooperative grid barriers, 132 CTAs x 512 threads.
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512, 1)
k_phase(int iters, int rounds, const int *__restrict__ ia, const int *__restrict__ ib,
        const double *zd, double *out, unsigned long long *tr, int mode, int mask) {
  cg::grid_group g = cg::this_grid();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    for (int r = 0; r < rounds; ++r) {
      const int p = ((blockIdx.x * 16 + warp) * 2 + r + i * 7 * (mode & 4)) & mask;  // a "pixel"
      const int k0 = ia[p] & mask;
      const int a0 = ib[k0 + lane] & mask;
      double s = zd[a0] * 0.5;
      s = __ldcg(zd + a0) + s;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      acc += s;
    }
    if (mode & 1) g.sync();
    else if (mode & 2) __syncthreads();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) tr[blockIdx.x] = t1 - t0;
  if (acc == -1.0) out[0] = acc;
}

int main() {
  const int n = 1 << 20;
  std::vector<int> ha(n), hb(n + 64);
  for (int i = 0; i < n; ++i) ha[i] = (int)((i * 2654435761u) % (n - 64));
  for (int i = 0; i < n + 64; ++i) hb[i] = (int)((i * 40503u) % n);
  int *ia, *ib;
  double *zd, *out;
  unsigned long long *tr;
  cudaMalloc(&ia, n * 4);
  cudaMalloc(&ib, (n + 64) * 4);
  cudaMalloc(&zd, n * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&tr, 8 * 1024);
  cudaMemcpy(ia, ha.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(ib, hb.data(), (n + 64) * 4, cudaMemcpyHostToDevice);
  cudaMemset(zd, 0, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int cfg = 0; cfg < 12; ++cfg) {
    int rounds = (cfg % 3 == 0) ? 0 : (cfg % 3 == 1 ? 1 : 4);
    int mode = (cfg / 3 == 0) ? 1 : (cfg / 3 == 1 ? 2 : (cfg / 3 == 2 ? 1 : 5));
    int mask = (cfg / 3 == 2) ? 4095 : n - 65;
    int iters = 1000, grid = 132;
    void *args[] = {&iters, &rounds, &ia, &ib, &zd, &out, &tr, &mode, &mask};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void *)k_phase, grid, 512, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("rounds=%d mode=%d mask=%d: %.3f us per iteration (%s)\n", rounds, mode, mask,
           1000.f * ms / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
