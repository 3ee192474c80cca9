// Multi-GPU gather of the Frobenius matrix behind the C ABI.
//
// Columns of F are independent (reference zeta.hpp:109-133 threads over
// them), so one process per GPU reduces its own columns; this file assembles
// F on every rank with ONE ncclAllGather.  Entries travel as fixed-width
// 62-bit limbs (NCCL's integer Sum would wrap mod 2^64 and every entry has
// exactly one owner, so no reduction is needed), with each rank's column
// ownership mask in the same buffer.  NCCL is taken from the process (torch
// loads it) or from the system libnccl.so.2, resolved at run time so that the
// library loads on hosts without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/drzg.h"
#include "pipeline.cuh"

namespace drzg {
void set_last_error(const std::string& s);
cudaStream_t device_stream(int device);  // pipeline.cu

namespace {
struct Nccl {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  static const Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's own (torch's)
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
      if (!h) return;
      n.get_id = (decltype(n.get_id))dlsym(h, "ncclGetUniqueId");
      n.init = (decltype(n.init))dlsym(h, "ncclCommInitRank");
      n.destroy = (decltype(n.destroy))dlsym(h, "ncclCommDestroy");
      n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
      n.err = (decltype(n.err))dlsym(h, "ncclGetErrorString");
    });
    DRZG_REQUIRE(n.get_id && n.init && n.destroy && n.all_gather && n.err, "NCCL (libnccl.so.2) unavailable");
    return n;
  }
};
#define DRZG_NCCL(x)                                                                                \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess) throw ::drzg::contract_error(std::string("NCCL: ") + Nccl::get().err(r_), \
                                                        __FILE__, __LINE__);                        \
  } while (0)

struct Comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0, device = 0;
};

constexpr int kLimbBits = 62;

template <class F>
int nguard(F&& f) {
  try {
    f();
    set_last_error("");
    return 0;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1;
  } catch (...) {
    set_last_error("unknown error");
    return 1;
  }
}
}  // namespace

// entries of the owned columns as `width` 62-bit limbs each (zeros elsewhere)
// followed by the b-entry ownership mask
std::vector<int64_t> encode_columns(int b, const std::vector<Z>& F, const std::vector<int>& cols, int width) {
  std::vector<int64_t> out((size_t)b * b * width + b, 0);
  const Z base = Z(1) << kLimbBits;
  for (int j : cols) {
    DRZG_REQUIRE(j >= 0 && j < b, "gather_F: column out of range");
    out[(size_t)b * b * width + j] = 1;
    for (int i = 0; i < b; ++i) {
      Z v = F[(size_t)i * b + j];
      DRZG_REQUIRE(!(v < Z(0)), "gather_F: Frobenius entries are non-negative residues");
      for (int t = 0; t < width; ++t) {
        Z r = v.mod(base);
        out[((size_t)i * b + j) * width + t] = (int64_t)r.to_u64();
        v = (v - r).divexact(base);
      }
      DRZG_REQUIRE(v == Z(0), "gather_F: entry exceeds the limb width");
    }
  }
  return out;
}

// every rank's block -> full F (each column from its owner)
std::vector<Z> decode_blocks(int b, const std::vector<int64_t>& all, int nranks, int width) {
  const size_t per = (size_t)b * b * width + b;
  std::vector<Z> F((size_t)b * b, Z(0));
  std::vector<int> owner(b, -1);
  const Z base = Z(1) << kLimbBits;
  for (int r = 0; r < nranks; ++r) {
    const int64_t* blk = all.data() + per * r;
    for (int j = 0; j < b; ++j) {
      if (!blk[(size_t)b * b * width + j]) continue;
      DRZG_REQUIRE(owner[j] < 0, "gather_F: column " + std::to_string(j) + " owned by two ranks");
      owner[j] = r;
      for (int i = 0; i < b; ++i) {
        Z v(0);
        for (int t = width - 1; t >= 0; --t) v = v * base + Z::from_u64((u64)blk[((size_t)i * b + j) * width + t]);
        F[(size_t)i * b + j] = v;
      }
    }
  }
  for (int j = 0; j < b; ++j) DRZG_REQUIRE(owner[j] >= 0, "gather_F: column " + std::to_string(j) + " has no owner");
  return F;
}

}  // namespace drzg

using namespace drzg;

extern "C" {

int drzg_nccl_unique_id(uint8_t* id_out) {
  return nguard([&] {
    ncclUniqueId id;
    DRZG_NCCL(Nccl::get().get_id(&id));
    static_assert(sizeof(id) == DRZG_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

drzg_comm* drzg_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, int32_t device) {
  Comm* out = nullptr;
  nguard([&] {
    auto c = std::make_unique<Comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    DRZG_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    DRZG_NCCL(Nccl::get().init(&c->comm, nranks, uid, rank));
    out = c.release();
  });
  return reinterpret_cast<drzg_comm*>(out);
}

void drzg_comm_free(drzg_comm* c) {
  Comm* cm = reinterpret_cast<Comm*>(c);
  if (!cm) return;
  if (cm->comm) Nccl::get().destroy(cm->comm);
  delete cm;
}

char* drzg_gather_F(drzg_comm* c, int32_t b, const char* const* F_local, const int32_t* cols, int32_t ncols,
                    int32_t width) {
  char* out = nullptr;
  nguard([&] {
    Comm& cm = *reinterpret_cast<Comm*>(c);
    DRZG_REQUIRE(width >= 1 && width <= 16, "gather_F: limb width");
    DRZG_CUDA(cudaSetDevice(cm.device));
    std::vector<Z> F((size_t)b * b);
    for (size_t i = 0; i < F.size(); ++i) F[i] = Z::from_str(F_local[i]);
    std::vector<int> own(cols, cols + ncols);
    std::vector<int64_t> mine = encode_columns(b, F, own, width);
    const size_t per = mine.size();
    cudaStream_t st = device_stream(cm.device);  // the thread's stream (retained allocations)
    int64_t *dsend = nullptr, *drecv = nullptr;
    DRZG_CUDA(cudaMallocAsync(&dsend, per * 8, st));
    DRZG_CUDA(cudaMallocAsync(&drecv, per * 8 * cm.nranks, st));
    DRZG_CUDA(cudaMemcpyAsync(dsend, mine.data(), per * 8, cudaMemcpyHostToDevice, st));
    DRZG_NCCL(Nccl::get().all_gather(dsend, drecv, per, ncclInt64, cm.comm, st));
    std::vector<int64_t> all(per * cm.nranks);
    DRZG_CUDA(cudaMemcpyAsync(all.data(), drecv, all.size() * 8, cudaMemcpyDeviceToHost, st));
    DRZG_CUDA(cudaFreeAsync(dsend, st));
    DRZG_CUDA(cudaFreeAsync(drecv, st));
    DRZG_CUDA(cudaStreamSynchronize(st));
    std::vector<Z> full = decode_blocks(b, all, cm.nranks, width);
    std::ostringstream os;
    os << "{\"F\":[";
    for (size_t i = 0; i < full.size(); ++i) os << (i ? "," : "") << "\"" << full[i].str() << "\"";
    os << "]}";
    const std::string s = os.str();
    out = (char*)std::malloc(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
  return out;
}

// host halves of the gather (no NCCL, no device): the limb encoding and the
// owner-by-column decoding, for the CPU tests
char* drzg_gather_F_host(int32_t nranks, int32_t b, const char* const* F_blocks, const int32_t* cols,
                         const int32_t* col_ptr, int32_t width) {
  char* out = nullptr;
  nguard([&] {
    std::vector<int64_t> all;
    for (int r = 0; r < nranks; ++r) {
      std::vector<Z> F((size_t)b * b);
      for (size_t i = 0; i < F.size(); ++i) F[i] = Z::from_str(F_blocks[(size_t)r * b * b + i]);
      std::vector<int> own(cols + col_ptr[r], cols + col_ptr[r + 1]);
      std::vector<int64_t> blk = encode_columns(b, F, own, width);
      all.insert(all.end(), blk.begin(), blk.end());
    }
    std::vector<Z> full = decode_blocks(b, all, nranks, width);
    std::ostringstream os;
    os << "{\"F\":[";
    for (size_t i = 0; i < full.size(); ++i) os << (i ? "," : "") << "\"" << full[i].str() << "\"";
    os << "]}";
    const std::string s = os.str();
    out = (char*)std::malloc(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
  return out;
}

}  // extern "C"
