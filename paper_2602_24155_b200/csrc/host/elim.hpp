// Elimination kernels used at setup time.
//
// pivot_scan_fp: forward elimination over F_p with the reference's pivot
//   rule — rows in order, pivot = first column (not yet a pivot column)
//   holding a unit.  The reference applies that rule inside UnitEchelon over
//   Z/p^M (linalg.hpp:551-578) and inside FpEchelon over F_p
//   (linalg.hpp:752-791).  A row's state when its turn comes is the same
//   under full and forward-only elimination, and "unit mod p^M" means
//   "nonzero mod p", so the F_p scan reproduces the reference's pivot set.
// inverse_mod_q: Gauss-Jordan inverse of a square matrix over Z/q, q = p^e
//   small; any unit pivot order gives the unique inverse.
#pragma once

#include <algorithm>
#include <vector>

#include "common.hpp"

namespace drzg {

struct PivotScan {
  std::vector<int> pivot_col_of_row;  // -1 for rows without a unit pivot
  int rank = 0;
};

// rows x cols matrix over F_p, row-major entries in [0, p)
inline PivotScan pivot_scan_fp(u64 p, int rows, int cols, std::vector<u32> m) {
  DRZG_REQUIRE((int64_t)m.size() == (int64_t)rows * cols, "pivot_scan_fp: bad size");
  PivotScan out;
  out.pivot_col_of_row.assign(rows, -1);
  std::vector<char> used(cols, 0);
  // lazy reduction: entries grow by < p*p per update, reduce a row before overflow
  const u32 P = (u32)p;
  const u64 step = (u64)(P - 1) * (P - 1) + P;
  const u64 cap = 0xFFFFFFFFull - step;
  std::vector<u64> bound(rows, P);
  for (int r = 0; r < rows; ++r) {
    u32* row = m.data() + (size_t)r * cols;
    for (int c = 0; c < cols; ++c) row[c] %= P;
    bound[r] = P;
    int pc = -1;
    for (int c = 0; c < cols; ++c)
      if (row[c] && !used[c]) {
        pc = c;
        break;
      }
    if (pc < 0) continue;
    u32 inv = (u32)invm(row[pc], p);
    for (int c = 0; c < cols; ++c) row[c] = (u32)((u64)row[c] * inv % P);
    used[pc] = 1;
    out.pivot_col_of_row[r] = pc;
    ++out.rank;
    for (int r2 = r + 1; r2 < rows; ++r2) {
      u32* dst = m.data() + (size_t)r2 * cols;
      u32 lead = dst[pc] % P;
      if (!lead) continue;
      if (bound[r2] > cap) {
        for (int c = 0; c < cols; ++c) dst[c] %= P;
        bound[r2] = P;
      }
      u32 f = P - lead;
      for (int c = 0; c < cols; ++c) dst[c] += f * row[c];
      bound[r2] += step;
    }
  }
  return out;
}

// inverse of an n x n matrix over Z/q (entries in [0, q)), q < 2^16; throws
// when the matrix is singular mod p
inline std::vector<u32> inverse_mod_q(u64 p, u64 q, int n, std::vector<u32> a) {
  DRZG_REQUIRE(q < 256, "inverse_mod_q: modulus too large");
  const int w = 2 * n;
  std::vector<u32> m((size_t)n * w, 0);
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) m[(size_t)i * w + j] = a[(size_t)i * n + j] % (u32)q;
    m[(size_t)i * w + n + i] = 1;
  }
  const u32 Q = (u32)q;
  // lazy accumulation: each pivot adds < Q^2 to an entry, so n pivots stay
  // below 2^32 whenever n * Q^2 < 2^32 - Q
  DRZG_REQUIRE((u64)n * Q * Q < 0xFFFFFFFFull - Q, "inverse_mod_q: order too large for lazy u32");
  for (int c = 0; c < n; ++c) {
    int pr = -1;
    for (int r = c; r < n; ++r)
      if ((m[(size_t)r * w + c] % Q) % p) {
        pr = r;
        break;
      }
    DRZG_REQUIRE(pr >= 0, "inverse_mod_q: singular mod p");
    if (pr != c)
      std::swap_ranges(m.begin() + (size_t)pr * w, m.begin() + (size_t)(pr + 1) * w, m.begin() + (size_t)c * w);
    u32* prow = m.data() + (size_t)c * w;
    u32 inv = (u32)invm(prow[c] % Q, q);
    for (int j = 0; j < w; ++j) prow[j] = (prow[j] % Q) * inv % Q;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      u32* row = m.data() + (size_t)r * w;
      u32 f = row[c] % Q;
      if (!f) continue;
      u32 g = Q - f;
      for (int j = 0; j < w; ++j) row[j] += g * prow[j];
    }
  }
  std::vector<u32> inv((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[(size_t)i * n + j] = m[(size_t)i * w + n + j] % Q;
  return inv;
}

}  // namespace drzg
