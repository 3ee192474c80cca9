// Frobenius-matrix assembly and the zeta driver on top of the device engine.
// Same contract as reference frobenius_matrix (zeta.hpp:36-136) and run_zeta
// (zeta.hpp:438-549): identical F mod p^M, charpoly residues, Q, Newton
// polygon and counts on the same input and plan.
#pragma once

#include <set>
#include <string>
#include <vector>

#include "engine.cuh"
#include "host/post.hpp"

namespace drzg {

struct FrobOptions {
  Policy policy = Policy::p_chunk;
  PlanOverrides overrides;
  int only_pole = 0;
  std::vector<int> columns;  // empty = all (subject to only_pole)
  bool profile = false;      // per-kernel CUDA-event timing
};

struct StageTimes {
  double tables = 0, seeds = 0, device = 0, final = 0, total = 0;
};

struct FrobResult {
  i64 b = 0;
  std::vector<Z> F;          // b x b row-major; columns not computed are 0
  std::vector<int> computed; // column indices computed
  Ledger led;
  StageTimes t;
  KernelClock clk;
  int M = 0, Ld = 0, q = 0, nL = 0, side = 0;
  i64 terms = 0;
  int groups = 0;            // device passes (memory-bounded column groups)
};

FrobResult frobenius_matrix(const Hypersurface& X, const Basis& B, const PrecisionPlan& plan, const std::set<int>& S,
                            const FrobOptions& opt, int device);

struct CountCheck {
  int r = 0;
  Z from_zeta, from_count;
  bool ok = false;
};

struct ZetaOptions {
  Policy policy = Policy::p_chunk;
  PlanOverrides overrides;
  bool verify_counts = true;
  i64 count_budget = 200000000;
  bool profile = false;
};

struct ZetaOut {
  std::vector<Z> Q, Q_alt;
  bool ambiguous = false;
  PrecisionPlan plan;
  NewtonPolygon np;
  std::vector<i64> hodge;
  Invariants inv;
  std::string domino;
  std::vector<CountCheck> counts;
  Ledger led;
  FrobResult last;
  double wall = 0;
  std::vector<std::string> reasons;  // escalation ladder steps taken
};

ZetaOut run_zeta(const Hypersurface& X, const ZetaOptions& opt, int device);

// run_zeta's battery on a given F (zeta.hpp:456-535): charpoly, Q recovery,
// sign tie-break by point counts, Newton >= Hodge, point-count checks.
// Returns "" (res filled) or the reason the plan must escalate.  Used by the
// multi-GPU path on the gathered F.
// (fsplit_known: Fedder's F-split test already computed, 0 / 1, or null)
std::string finish_zeta(const Hypersurface& X, const PrecisionPlan& plan, const std::vector<Z>& F, i64 b,
                        const ZetaOptions& opt, ZetaOut& res, const int* fsplit_known = nullptr);

std::set<int> working_set_for(const Hypersurface& X, Policy pol);

}  // namespace drzg
