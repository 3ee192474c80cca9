// The reduction game's move rules, shared by host and device code.  Each
// function is a restatement of the reference rule it cites; S is a bitmask
// over the nv variables (bit i set <=> i in S).
#pragma once

#include "mono.hpp"

namespace drzg {

DRZG_HD bool in_mask(unsigned mask, int i) { return (mask >> i) & 1u; }

// reduction.hpp:18-32: remove `amount` units, repeatedly decrementing the
// first positive entry
DRZG_HD Expo tweak(const Expo& I, int amount) {
  Expo r = I;
  int left = amount;
  if (left > I.total()) return r;
  while (left > 0) {
    for (int i = 0; i < r.nv && left > 0; ++i)
      if (r.e[i] > 0) {
        --r.e[i];
        --left;
        break;
      }
  }
  return r;
}

// reduction.hpp:46-56
DRZG_HD bool legal(int d, const Expo& u, const Expo& v, i64 k, unsigned S) {
  if (v.total() != d || k < 0) return false;
  for (int i = 0; i < u.nv; ++i) {
    bool inS = in_mask(S, i);
    if (inS && v.e[i] == 0 && u.e[i] != 0) return false;
    i64 left = (i64)u.e[i] - k * v.e[i];
    if (left < (inS ? 0 : 1)) return false;
  }
  return true;
}

// reduction.hpp:59-67
DRZG_HD i64 k_max_legal(const Expo& u, const Expo& v, unsigned S) {
  i64 k = (i64)1 << 62;
  bool any = false;
  for (int i = 0; i < u.nv; ++i) {
    if (v.e[i] == 0) continue;
    i64 room = in_mask(S, i) ? (i64)u.e[i] : (i64)u.e[i] - 1;
    i64 q = room / v.e[i];
    if (!any || q < k) k = q;
    any = true;
  }
  if (!any) return 0;
  return k < 0 ? 0 : k;
}

// reduction.hpp:71-91
DRZG_HD Expo choose_v_greedy(int d, const Expo& u, unsigned S) {
  Expo v(u.nv);
  int placed = 0;
  for (int s = 0; s < u.nv; ++s)
    if (in_mask(S, s) && u.e[s] != 0 && placed < d) {
      v.e[s] = 1;
      ++placed;
    }
  int m = 0, idle = 0;
  while (placed < d && idle < u.nv) {
    if (v.e[m] < u.e[m]) {
      ++v.e[m];
      ++placed;
      idle = 0;
    } else {
      ++idle;
    }
    m = (m + 1) % u.nv;
  }
  return v;
}

// reduction.hpp:96-111
DRZG_HD void repair_v(const Expo& u, Expo& v, unsigned S) {
  for (int i = 0; i < u.nv; ++i) {
    if (in_mask(S, i) || v.e[i] < u.e[i]) continue;
    while (v.e[i] > 0 && v.e[i] >= u.e[i]) {
      int j = -1;
      for (int c = 0; c < u.nv && j < 0; ++c) {
        if (c == i) continue;
        i64 cap = in_mask(S, c) ? (i64)u.e[c] : (i64)u.e[c] - 1;
        if (v.e[c] < cap) j = c;
      }
      if (j < 0) return;
      --v.e[i];
      ++v.e[j];
    }
  }
}

// reduction.hpp:538-563: seed exponent u = tweak(E+1, D) made honest for S
DRZG_HD bool seed_u(const Expo& full, int D, unsigned S, Expo* out) {
  Expo u = tweak(full, D);
  for (int i = 0; i < u.nv; ++i) {
    if (in_mask(S, i) || u.e[i] >= 1) continue;
    int j = -1;
    for (int c = 0; c < u.nv; ++c) {
      bool ok = in_mask(S, c) ? u.e[c] >= 1 : u.e[c] >= 2;
      if (ok && (j < 0 || u.e[c] > u.e[j])) j = c;
    }
    if (j < 0) return false;
    --u.e[j];
    ++u.e[i];
  }
  *out = u;
  return true;
}

// p-chunk move for a state at the sweep top (reduction.hpp:486-496)
DRZG_HD void pchunk_move(int d, int n, i64 p, const Expo& u, int pole, unsigned S, Expo* v_out, i64* k_out) {
  Expo v = choose_v_greedy(d, u, S);
  repair_v(u, v, S);
  i64 kt = p < (i64)(pole - n) ? p : (i64)(pole - n);
  i64 km = k_max_legal(u, v, S);
  *v_out = v;
  *k_out = kt < km ? kt : km;
}

}  // namespace drzg
