// Microbenchmark: read pattern of the T_x epilogue (Ld planes x scattered
// source rows x 128 states per block) from the plane-major Y layout
// [t][r][P] against a state-tiled layout [tile][t][r][128].  Answers whether
// DRAM page locality limits the epilogue.  nvcc -O3 -arch=sm_100a ylayout.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int LD = 12;
__global__ void rd_plane(const int* __restrict__ Y, const int* __restrict__ rows, int nrows, size_t P, size_t nLp,
                         int* out) {
  // block: 128 states (32 lanes x 4 B), warps over rows
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t sb = (size_t)blockIdx.x * 128;
  const int r0 = blockIdx.y * 256;
  int acc = 0;
  for (int i = r0 + warp; i < min(nrows, r0 + 256); i += 8) {
    const int r = rows[i];
    uint32_t w[LD];
#pragma unroll
    for (int t = 0; t < LD; ++t) w[t] = __ldg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(Y) + ((size_t)t * nLp + r) * P + sb) + lane);
#pragma unroll
    for (int t = 0; t < LD; ++t) acc += (int)w[t];
  }
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void rd_tiled(const int* __restrict__ Y, const int* __restrict__ rows, int nrows, size_t P, size_t nLp,
                         int* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t tile = blockIdx.x;
  const int r0 = blockIdx.y * 256;
  const char* base = reinterpret_cast<const char*>(Y) + tile * (size_t)LD * nLp * 128;
  int acc = 0;
  for (int i = r0 + warp; i < min(nrows, r0 + 256); i += 8) {
    const int r = rows[i];
    uint32_t w[LD];
#pragma unroll
    for (int t = 0; t < LD; ++t) w[t] = __ldg(reinterpret_cast<const uint32_t*>(base + ((size_t)t * nLp + r) * 128) + lane);
#pragma unroll
    for (int t = 0; t < LD; ++t) acc += (int)w[t];
  }
  if (acc == 0x12345678) out[0] = acc;
}
// rows interleaved: [tile][r][t][128] (the 12 planes of a row adjacent)
__global__ void rd_rowmajor(const int* __restrict__ Y, const int* __restrict__ rows, int nrows, size_t P, size_t nLp,
                            int* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t tile = blockIdx.x;
  const int r0 = blockIdx.y * 256;
  const char* base = reinterpret_cast<const char*>(Y) + tile * (size_t)LD * nLp * 128;
  int acc = 0;
  for (int i = r0 + warp; i < min(nrows, r0 + 256); i += 8) {
    const int r = rows[i];
    uint32_t w[LD];
#pragma unroll
    for (int t = 0; t < LD; ++t) w[t] = __ldg(reinterpret_cast<const uint32_t*>(base + ((size_t)r * LD + t) * 128) + lane);
#pragma unroll
    for (int t = 0; t < LD; ++t) acc += (int)w[t];
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t nLp = 3072, nL = 3003, P = 30720;  // 240 tiles of 128 states
  const size_t bytes = LD * nLp * P;
  int *Y, *rows, *out;
  cudaMalloc(&Y, bytes);
  cudaMemset(Y, 1, bytes);
  cudaMalloc(&out, 4);
  std::vector<int> seq(nL), rnd(nL);
  for (size_t i = 0; i < nL; ++i) seq[i] = rnd[i] = (int)i;
  std::mt19937 g(1);
  std::shuffle(rnd.begin(), rnd.end(), g);
  cudaMalloc(&rows, nL * 4);
  dim3 grid(P / 128, (nL + 255) / 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double useful = (double)LD * nL * P;
  for (int order = 0; order < 2; ++order) {
    cudaMemcpy(rows, order ? rnd.data() : seq.data(), nL * 4, cudaMemcpyHostToDevice);
    for (int kind = 0; kind < 3; ++kind) {
      float best = 1e9;
      for (int it = 0; it < 6; ++it) {
        cudaEventRecord(a);
        if (kind == 0) rd_plane<<<grid, 256>>>(Y, rows, nL, P, nLp, out);
        else if (kind == 1) rd_tiled<<<grid, 256>>>(Y, rows, nL, P, nLp, out);
        else rd_rowmajor<<<grid, 256>>>(Y, rows, nL, P, nLp, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it) best = std::min(best, ms);
      }
      printf("rows %s layout %s: %.3f ms, %.0f GB/s\n", order ? "random" : "sequential",
             kind == 0 ? "plane-major [t][r][P]" : kind == 1 ? "tiled [tile][t][r][128]" : "row-major [tile][r][t][128]",
             best, useful / best / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
