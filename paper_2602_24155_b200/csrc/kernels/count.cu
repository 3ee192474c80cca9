// Brute-force point count #X(F_{p^r}) on the device: the
// same enumeration as the reference count_points (oracle.hpp:190-245) —
// points of P^n normalised so the first nonzero coordinate is 1, stratum by
// stratum — one thread per point, field arithmetic through the add / mul
// tables of F_{p^r} (host/post.hpp ExtField), reduced per block.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../host/post.hpp"
#include "count.cuh"

namespace drzg {
cudaStream_t device_stream(int device);  // pipeline.cu

namespace dev {

struct CountArgs {
  const unsigned short* add;  // q x q
  const unsigned short* mul;  // q x q
  const unsigned short* powt; // q x (d+1)
  const int* tc;              // live terms: coefficient (field element)
  const int* te;              // live terms: exponents, nv each
  int nterms, nv, n, lead, q, d;
  long long npts;             // q^(n - lead)
};

__global__ void count_kernel(CountArgs a, unsigned long long* out) {
  __shared__ unsigned long long blk;
  if (threadIdx.x == 0) blk = 0;
  __syncthreads();
  unsigned long long local = 0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < a.npts;
       idx += (long long)gridDim.x * blockDim.x) {
    // coordinates x[lead+1..n] from idx (x[n] fastest, as the reference's odometer)
    int x[6] = {0, 0, 0, 0, 0, 0};
    long long t = idx;
    for (int i = a.n; i > a.lead; --i) {
      x[i] = (int)(t % a.q);
      t /= a.q;
    }
    x[a.lead] = 1;
    unsigned acc = 0;
    for (int k = 0; k < a.nterms; ++k) {
      unsigned v = (unsigned)a.tc[k];
      const int* e = a.te + k * a.nv;
      for (int i = a.lead + 1; i <= a.n && v; ++i)
        if (e[i]) v = a.mul[v * a.q + a.powt[x[i] * (a.d + 1) + e[i]]];
      acc = a.add[acc * a.q + v];
    }
    local += acc == 0;
  }
  atomicAdd(&blk, local);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, blk);
}

}  // namespace dev

namespace {
void ck(cudaError_t e, const char* w) {
  if (e != cudaSuccess) throw contract_error(std::string(w) + ": " + cudaGetErrorString(e), __FILE__, __LINE__);
}
}  // namespace

i64 count_points_device(const Hypersurface& X, int r, i64 budget) {
  ExtField F = ExtField::make(X.p, r);
  const u64 q = F.q;
  const int nv = X.nv(), n = X.n;
  Z work(0);
  for (int m = 0; m <= n; ++m) work += Z::pow(q, (u64)m);
  DRZG_REQUIRE(work <= Z((long)budget), "count_points: budget exceeded");
  DRZG_REQUIRE(q <= 65535, "count_points_device: field too large");
  std::vector<unsigned short> addt(q * q), mult(q * q), powt(q * (X.d + 1));
  for (u64 x = 0; x < q; ++x)
    for (u64 y = 0; y < q; ++y) {
      addt[x * q + y] = (unsigned short)F.add(x, y);
      mult[x * q + y] = (unsigned short)F.mul[x * q + y];
    }
  for (u64 v = 0; v < q; ++v) {
    powt[v * (X.d + 1)] = 1;
    for (int e = 1; e <= X.d; ++e) powt[v * (X.d + 1) + e] = (unsigned short)F.mul[powt[v * (X.d + 1) + e - 1] * q + v];
  }
  // the calling thread's stream on this device (pipeline.cu): its retained
  // stream-ordered allocations serve these buffers without regrowing the pool
  int dev = 0;
  ck(cudaGetDevice(&dev), "device");
  cudaStream_t st = device_stream(dev);
  unsigned short *da, *dm, *dp;
  int *dtc, *dte;
  unsigned long long* dout;
  ck(cudaMallocAsync(&da, addt.size() * 2, st), "alloc");
  ck(cudaMallocAsync(&dm, mult.size() * 2, st), "alloc");
  ck(cudaMallocAsync(&dp, powt.size() * 2, st), "alloc");
  ck(cudaMallocAsync(&dout, 8, st), "alloc");
  ck(cudaMemcpyAsync(da, addt.data(), addt.size() * 2, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(dm, mult.data(), mult.size() * 2, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemcpyAsync(dp, powt.data(), powt.size() * 2, cudaMemcpyHostToDevice, st), "copy");
  ck(cudaMemsetAsync(dout, 0, 8, st), "memset");
  auto terms = X.f.terms();
  std::vector<int> tcv, tev;
  ck(cudaMallocAsync(&dtc, std::max<size_t>(terms.size(), 1) * 4, st), "alloc");
  ck(cudaMallocAsync(&dte, std::max<size_t>(terms.size(), 1) * nv * 4, st), "alloc");
  for (int lead = 0; lead <= n; ++lead) {
    tcv.clear();
    tev.clear();
    for (auto& t : terms) {
      bool dead = false;
      for (int i = 0; i < lead; ++i) dead |= t.e[i] != 0;
      u32 c = (u32)(t.c % X.p);
      if (dead || !c) continue;
      tcv.push_back((int)c);
      for (int i = 0; i < nv; ++i) tev.push_back(t.e[i]);
    }
    long long npts = 1;
    for (int i = lead + 1; i <= n; ++i) npts *= (long long)q;
    if (!tcv.empty()) {
      ck(cudaMemcpyAsync(dtc, tcv.data(), tcv.size() * 4, cudaMemcpyHostToDevice, st), "copy");
      ck(cudaMemcpyAsync(dte, tev.data(), tev.size() * 4, cudaMemcpyHostToDevice, st), "copy");
    }
    dev::CountArgs a{da, dm, dp, dtc, dte, (int)tcv.size(), nv, n, lead, (int)q, X.d, npts};
    int blocks = (int)std::min<long long>((npts + 255) / 256, 148 * 16);
    dev::count_kernel<<<std::max(blocks, 1), 256, 0, st>>>(a, dout);
    ck(cudaStreamSynchronize(st), "count");  // tcv/tev are reused next stratum
  }
  unsigned long long cnt = 0;
  ck(cudaMemcpyAsync(&cnt, dout, 8, cudaMemcpyDeviceToHost, st), "copy");
  ck(cudaStreamSynchronize(st), "sync");
  ck(cudaGetLastError(), "count kernel");
  cudaFreeAsync(da, st);
  cudaFreeAsync(dm, st);
  cudaFreeAsync(dp, st);
  cudaFreeAsync(dtc, st);
  cudaFreeAsync(dte, st);
  cudaFreeAsync(dout, st);
  cudaStreamSynchronize(st);
  return (i64)cnt;
}

}  // namespace drzg
