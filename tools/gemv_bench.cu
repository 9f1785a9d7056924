// gemv_bench.cu -- standalone timing of the pixel-space FISTA matvec (k_gemv_sym's
// tile code) against a plain streaming read of the same packed store, warm (L2)
// and cold (after a 512 MB write), at several grid sizes.  Not part of the engine.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2603_08582_b200/csrc tools/gemv_bench.cu -o /tmp/gemv_bench
#include <cstdio>
#include <vector>

#include "sf_gemv_tile.cuh"

using namespace sf;

__global__ void __launch_bounds__(256, 2)
k_gemv_clone(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
             const float *__restrict__ z32, float *__restrict__ P, int nt) {
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int2 ij = tiles[t];
    const int64_t store = tri_index(ij.x, ij.y, nt);
    const float4 *T = reinterpret_cast<const float4 *>(A + store * (int64_t)kTileElems);
    float4 a[4][4];
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = __ldg(T + (int64_t)(warp + 8 * s4) * kTile + lane + 32 * i);
    gemv_tile_compute<0>(a, ij.x, ij.y, z32, P, nt, 1, s_row, s_col);
  }
}

template <int U>
__global__ void __launch_bounds__(256) k_stream(const float4 *__restrict__ A, int64_t n4,
                                                float *__restrict__ out) {
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(A + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) {
    float4 v = __ldg(A + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 123.456f) out[0] = s;
}

__global__ void k_thrash(float4 *buf, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                 \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(int argc, char **argv) {
  int n = argc > 1 ? atoi(argv[1]) : 4096;
  int nt = (n + kTile - 1) / kTile;
  int64_t T = (int64_t)nt * (nt + 1) / 2;
  int64_t elems = T * kTileElems;
  printf("N=%d nt=%d tiles=%lld store=%.1f MB\n", n, nt, (long long)T, elems * 4e-6);
  float *A, *z, *P, *out;
  float4 *thr;
  int2 *tiles;
  CK(cudaMalloc(&A, elems * 4));
  CK(cudaMalloc(&z, (int64_t)nt * kTile * 4));
  CK(cudaMalloc(&P, (int64_t)nt * nt * kTile * 4));
  CK(cudaMalloc(&out, 16));
  const int64_t thr4 = (512ll << 20) / 16;
  CK(cudaMalloc(&thr, thr4 * 16));
  std::vector<int2> ht;
  for (int i = 0; i < nt; ++i)
    for (int j = i; j < nt; ++j) ht.push_back(make_int2(i, j));
  CK(cudaMalloc(&tiles, ht.size() * sizeof(int2)));
  CK(cudaMemcpy(tiles, ht.data(), ht.size() * sizeof(int2), cudaMemcpyHostToDevice));
  CK(cudaMemset(A, 0, elems * 4));
  CK(cudaMemset(z, 0, (int64_t)nt * kTile * 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  auto time_it = [&](const char *name, auto launch, bool cold) {
    const int reps = 200;
    float tot = 0.f;
    for (int w = 0; w < 5; ++w) launch();
    if (!cold) {
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&tot, e0, e1);
    } else {
      for (int r = 0; r < 50; ++r) {
        k_thrash<<<sms * 4, 256>>>(thr, thr4);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      tot *= (float)reps / 50.f;
    }
    float us = tot * 1e3f / reps;
    printf("%-34s %s %8.2f us  %7.0f GB/s\n", name, cold ? "cold" : "warm", us,
           elems * 4.0 / (us * 1e3));
  };

  for (int cold = 0; cold < 2; ++cold) {
    for (int g : {sms, 2 * sms, (int)T}) {
      char nm[64];
      snprintf(nm, sizeof nm, "gemv_sym grid=%d", g);
      time_it(nm, [&] { k_gemv_clone<<<g, 256>>>(A, tiles, T, z, P, nt); }, cold);
    }
    for (int g : {sms, 2 * sms, 4 * sms, 8 * sms}) {
      char nm[64];
      snprintf(nm, sizeof nm, "stream U=4 grid=%d", g);
      time_it(nm, [&] { k_stream<4><<<g, 256>>>((const float4 *)A, elems / 4, out); }, cold);
      snprintf(nm, sizeof nm, "stream U=8 grid=%d", g);
      time_it(nm, [&] { k_stream<8><<<g, 256>>>((const float4 *)A, elems / 4, out); }, cold);
    }
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
