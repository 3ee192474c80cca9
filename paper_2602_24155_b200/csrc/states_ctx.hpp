// The device context behind drzg_ctx (states.cu) and the PEP store (pep.cu).
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "../../include/drzg.h"
#include "pipeline.cuh"

namespace drzg {

struct StatesCtx {
  Hypersurface X;
  int M = 0;
  Policy policy = Policy::p_chunk;
  RuvTables T;
  drzg_stripe_plan sp{};
  HostMod hm;
  cudaStream_t st = nullptr;
  int device = 0;
  std::unique_ptr<ReductionEngine> eng;
  std::vector<ReductionEngine::Live> states;  // id -> state
  std::vector<char> alive;
  std::mutex mu;  // one call at a time per context
  ~StatesCtx() {
    if (eng) {
      cudaSetDevice(device);
      eng.reset();
    }
    if (st) cudaStreamDestroy(st);
  }
};

}  // namespace drzg
