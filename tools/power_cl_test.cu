// Standalone check of the cluster power-iteration kernels (debug harness).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -Iinclude -Ipaper_2603_08582_b200/csrc \
//   tools/power_cl_test.cu -o build/power_cl_test
#include "../paper_2603_08582_b200/csrc/sf_geom.cu"
#include <cstdio>
#include <random>
#include <vector>

namespace sf {
std::atomic<int64_t> g_launches{0};
bool debug_sync() { return false; }
sf_status fail(sf_status st, const std::string &msg) {
  fprintf(stderr, "fail: %s\n", msg.c_str());
  return st;
}
}  // namespace sf

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32;
  const int variant = argc > 2 ? atoi(argv[2]) : 0;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double2> G(n * n), K(n * n), u0(n);
  for (auto &g : G) g = make_double2(nd(rng), nd(rng));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double re = 0, im = 0;
      for (int k = 0; k < n; ++k) {  // G G^H
        const double2 a = G[i * n + k], b = G[j * n + k];
        re += a.x * b.x + a.y * b.y;
        im += a.y * b.x - a.x * b.y;
      }
      K[i * n + j] = make_double2(re, im);
    }
  for (auto &u : u0) u = make_double2(nd(rng), nd(rng));
  double2 *dK, *du;
  double *dd, *dL;
  long long *dc;
  cudaMalloc(&dK, n * n * 16);
  cudaMalloc(&du, n * 16);
  cudaMalloc(&dd, 64);
  cudaMalloc(&dL, 8);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dK, K.data(), n * n * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(du, u0.data(), n * 16, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0, 64);
  sf_status s = SF_OK;
  auto run = [&]() {
    switch (variant) {
      case 0: return sf::launch_power_cl<4, 4, 0>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 1: return sf::launch_power_cl<8, 8, 0>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 3: return sf::launch_power_cl<4, 4, 3>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 4: return sf::launch_power_cl<8, 8, 3>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 5: return sf::launch_power_cl<4, 4, 1>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 6: return sf::launch_power_cl<8, 4, 3>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      case 7: return sf::launch_power_cl<4, 2, 3>(dK, du, n, 1e-6, 500, dL, dc, dd, 0, 0);
      default: return SF_EINVAL;
    }
  };
  s = run();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) s = (sf_status)(s | run());
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  double diag[4];
  cudaMemcpy(diag, dd, 32, cudaMemcpyDeviceToHost);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("n %d variant %d status %d cuda %s diag %.15g %g %g %g  us/launch %.1f us/iter %.3f\n", n,
         variant, (int)s, cudaGetErrorString(e), diag[0], diag[1], diag[2], diag[3], ms * 50.0,
         ms * 50.0 / diag[1]);
  return 0;
}
