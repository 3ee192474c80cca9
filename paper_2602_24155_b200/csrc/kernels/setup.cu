// Setup-time eliminations on the device (RuvContext /
// FinalReducer solves).  Same results as host/elim.hpp:
//   pivot_scan_device: forward elimination over F_p, rows in order, pivot =
//     first nonzero column of the reduced row (the reference's first-unit rule,
//     linalg.hpp:551-578 / 752-791);
//   inverse_mod_q_device: Gauss-Jordan inverse over Z/q (unique, so any unit
//     pivot order gives the reference's U).
// Entries are kept lazily in int32 (each pivot adds < q^2 to an entry; the
// bound is checked on the host), so only the pivot row and the pivot column
// are reduced per step and the n^2 (or n x cols) update is a plain multiply-add.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../host/common.hpp"
#include "setup.cuh"

namespace drzg {
cudaStream_t device_stream(int device);  // pipeline.cu
namespace dev {

// first column c in [0, cols) with row[c] % p != 0, or -1; one block
__global__ void first_nonzero_kernel(const int* row, int cols, int p, int* out) {
  __shared__ int best;
  if (threadIdx.x == 0) best = cols;
  __syncthreads();
  for (int c = threadIdx.x; c < cols; c += blockDim.x)
    if (row[c] % p != 0) {
      atomicMin(&best, c);
      break;
    }
  __syncthreads();
  if (threadIdx.x == 0) *out = best < cols ? best : -1;
}

// inverse of the pivot entry, taken once before any block rescales the row
__global__ void pivot_inverse_kernel(const int* row, int m, const int* cptr, const int* inv_tab, int* iv_out) {
  const int c = *cptr;
  if (c >= 0) *iv_out = inv_tab[((row[c] % m) + m) % m];
}

// normalise row r by the pivot inverse *ivp (and reduce it fully); skipped
// when c < 0
__global__ void normalise_row_kernel(int* row, int cols, int m, const int* cptr, const int* ivp) {
  const int c = *cptr;
  if (c < 0) return;
  const int iv = *ivp;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    int v = ((row[j] % m) + m) % m;
    row[j] = (v * iv) % m;
  }
}

// f[r] = a[r][c] mod m for rows [r_lo, r_hi): snapshot of the pivot column
// taken before any block of the update can zero it
__global__ void factors_kernel(const int* a, int ld, int r_lo, int r_hi, const int* cptr, int m, int* f) {
  const int c = *cptr;
  const int r = r_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r_hi) return;
  f[r] = c < 0 ? 0 : ((a[(size_t)r * ld + c] % m) + m) % m;
}

// rows [r_lo, r_hi) (except `skip`) += (m - f_r) * pivot_row
__global__ void eliminate_kernel(int* a, int ld, int cols, int r_lo, int r_hi, int skip, const int* pivot_row,
                                 const int* cptr, int m, const int* fac) {
  const int c = *cptr;
  if (c < 0) return;
  const int r = r_lo + blockIdx.y;
  if (r >= r_hi || r == skip) return;
  int* row = a + (size_t)r * ld;
  const int f = fac[r];
  if (f == 0) return;
  const int g = m - f;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) row[j] += g * pivot_row[j];
}

// Gauss-Jordan: pick the first row >= c with a unit (mod p) in column c
__global__ void pivot_row_kernel(const int* a, int ld, int n, int c, int p, int* out) {
  __shared__ int best;
  if (threadIdx.x == 0) best = n;
  __syncthreads();
  for (int r = c + threadIdx.x; r < n; r += blockDim.x)
    if (a[(size_t)r * ld + c] % p != 0) atomicMin(&best, r);
  __syncthreads();
  if (threadIdx.x == 0) out[0] = best < n ? best : -1;
}

__global__ void swap_rows_kernel(int* a, int ld, int cols, int c, const int* rptr) {
  const int r = *rptr;
  if (r < 0 || r == c) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    int t = a[(size_t)r * ld + j];
    a[(size_t)r * ld + j] = a[(size_t)c * ld + j];
    a[(size_t)c * ld + j] = t;
  }
}

__global__ void set_const_kernel(int* out, int v) { *out = v; }

__global__ void reduce_all_kernel(int* a, size_t count, int m) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    a[i] = ((a[i] % m) + m) % m;
}

}  // namespace dev

namespace {
void ck(cudaError_t e, const char* w) {
  if (e != cudaSuccess) throw contract_error(std::string(w) + ": " + cudaGetErrorString(e), __FILE__, __LINE__);
}
std::vector<int> inverse_table(int m, int p) {
  std::vector<int> t(m, 0);
  for (int x = 1; x < m; ++x)
    if (x % p) t[x] = (int)invm((u64)x, (u64)m);
  return t;
}
}  // namespace

std::vector<int> pivot_scan_device(u64 p, int rows, int cols, const std::vector<u32>& m) {
  DRZG_REQUIRE((int64_t)rows * ((int64_t)(p - 1) * (p - 1) + p) < (1ll << 31), "pivot_scan_device: lazy bound");
  cudaStream_t st;
  {
    int dev = 0;
    ck(cudaGetDevice(&dev), "device");
    st = device_stream(dev);  // the thread's stream: retained allocations, no pool regrowth
  }
  int *da = nullptr, *dpiv = nullptr, *dinv = nullptr, *dfac = nullptr;
  size_t nn = (size_t)rows * cols;
  ck(cudaMallocAsync(&dfac, (rows + 1) * sizeof(int), st), "alloc");
  ck(cudaMallocAsync(&da, nn * sizeof(int), st), "alloc");
  ck(cudaMallocAsync(&dpiv, rows * sizeof(int), st), "alloc");
  auto itab = inverse_table((int)p, (int)p);
  ck(cudaMallocAsync(&dinv, itab.size() * sizeof(int), st), "alloc");
  std::vector<int> h(m.begin(), m.end());
  ck(cudaMemcpyAsync(da, h.data(), nn * sizeof(int), cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(dinv, itab.data(), itab.size() * sizeof(int), cudaMemcpyHostToDevice, st), "copy");
  const int threads = 256;
  const int cblocks = std::min(64, (cols + threads - 1) / threads);
  for (int r = 0; r < rows; ++r) {
    int* row = da + (size_t)r * cols;
    dev::first_nonzero_kernel<<<1, 1024, 0, st>>>(row, cols, (int)p, dpiv + r);
    dev::pivot_inverse_kernel<<<1, 1, 0, st>>>(row, (int)p, dpiv + r, dinv, dfac + rows);
    dev::normalise_row_kernel<<<cblocks, threads, 0, st>>>(row, cols, (int)p, dpiv + r, dfac + rows);
    if (r + 1 < rows) {
      // rows below, in slabs of 65535 (grid.y limit)
      dev::factors_kernel<<<(rows - r - 1 + 255) / 256, 256, 0, st>>>(da, cols, r + 1, rows, dpiv + r, (int)p, dfac);
      for (int lo = r + 1; lo < rows; lo += 65535) {
        int hi = std::min(rows, lo + 65535);
        dim3 g(cblocks, hi - lo);
        dev::eliminate_kernel<<<g, threads, 0, st>>>(da, cols, cols, lo, hi, -1, row, dpiv + r, (int)p, dfac);
      }
    }
  }
  std::vector<int> piv(rows);
  ck(cudaMemcpyAsync(piv.data(), dpiv, rows * sizeof(int), cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "sync");
  ck(cudaGetLastError(), "pivot scan");
  cudaFreeAsync(da, st);
  cudaFreeAsync(dpiv, st);
  cudaFreeAsync(dinv, st);
  cudaFreeAsync(dfac, st);
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(st);
  return piv;
}

std::vector<u32> inverse_mod_q_device(u64 p, u64 q, int n, const std::vector<u32>& a) {
  DRZG_REQUIRE(q < 256 && (int64_t)n * (int64_t)(q * q) < (1ll << 31), "inverse_mod_q_device: lazy bound");
  cudaStream_t st;
  {
    int dev = 0;
    ck(cudaGetDevice(&dev), "device");
    st = device_stream(dev);  // the thread's stream: retained allocations, no pool regrowth
  }
  const int w = 2 * n;
  std::vector<int> h((size_t)n * w, 0);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) h[(size_t)i * w + j] = (int)(a[(size_t)i * n + j] % q);
    h[(size_t)i * w + n + i] = 1;
  }
  int *da = nullptr, *dr = nullptr, *dc = nullptr, *dinv = nullptr, *dfac = nullptr;
  ck(cudaMallocAsync(&dfac, (n + 1) * sizeof(int), st), "alloc");
  ck(cudaMallocAsync(&da, h.size() * sizeof(int), st), "alloc");
  ck(cudaMallocAsync(&dr, sizeof(int), st), "alloc");
  ck(cudaMallocAsync(&dc, sizeof(int), st), "alloc");
  auto itab = inverse_table((int)q, (int)p);
  ck(cudaMallocAsync(&dinv, itab.size() * sizeof(int), st), "alloc");
  ck(cudaMemcpyAsync(da, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(dinv, itab.data(), itab.size() * sizeof(int), cudaMemcpyHostToDevice, st), "copy");
  const int threads = 256;
  const int cblocks = std::min(64, (w + threads - 1) / threads);
  for (int c = 0; c < n; ++c) {
    dev::pivot_row_kernel<<<1, 1024, 0, st>>>(da, w, n, c, (int)p, dr);
    dev::swap_rows_kernel<<<cblocks, threads, 0, st>>>(da, w, w, c, dr);
    dev::set_const_kernel<<<1, 1, 0, st>>>(dc, c);
    int* prow = da + (size_t)c * w;
    dev::pivot_inverse_kernel<<<1, 1, 0, st>>>(prow, (int)q, dc, dinv, dfac + n);
    dev::normalise_row_kernel<<<cblocks, threads, 0, st>>>(prow, w, (int)q, dc, dfac + n);
    dev::factors_kernel<<<(n + 255) / 256, 256, 0, st>>>(da, w, 0, n, dc, (int)q, dfac);
    for (int lo = 0; lo < n; lo += 65535) {
      int hi = std::min(n, lo + 65535);
      dim3 g(cblocks, hi - lo);
      dev::eliminate_kernel<<<g, threads, 0, st>>>(da, w, w, lo, hi, c, prow, dc, (int)q, dfac);
    }
  }
  dev::reduce_all_kernel<<<1024, 256, 0, st>>>(da, h.size(), (int)q);
  ck(cudaMemcpyAsync(h.data(), da, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st), "copy");
  int pr = 0;
  ck(cudaMemcpyAsync(&pr, dr, sizeof(int), cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "sync");
  ck(cudaGetLastError(), "inverse");
  cudaFreeAsync(da, st);
  cudaFreeAsync(dr, st);
  cudaFreeAsync(dc, st);
  cudaFreeAsync(dinv, st);
  cudaFreeAsync(dfac, st);
  cudaStreamSynchronize(st);
  cudaStreamSynchronize(st);
  std::vector<u32> inv((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[(size_t)i * n + j] = (u32)h[(size_t)i * w + n + j];
  return inv;
}

}  // namespace drzg
