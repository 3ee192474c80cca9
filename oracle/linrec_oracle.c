/* TEST INFRASTRUCTURE ONLY — the plain-C restatement of the reference's
 * recurrence evaluator, used by tests/ as an independent CPU checker (never
 * linked into the product).
 *
 *   oracle_linrec_eval   reference linrec_eval, linalg.hpp:337-410:
 *       w <- M(0) M(1) ... M(tmax) w,  M(t) = t A + B  (factor t = tmax first)
 *       on ModMatrix / ModVec layout (linalg.hpp:94-141): `limbs` planes of
 *       base-beta digits, plane-major then row-major.  The reference's three
 *       internal paths (dense 1-limb :366-397, sparse CSC :257-331, generic
 *       multi-plane :398-409) all return the canonical residue of the exact
 *       product mod p^M; this restatement computes that product directly:
 *       per output row and digit-plane sum s = t1 + t2 < limbs (planes at or
 *       beyond `limbs` vanish, linalg.hpp:284, because p^M | beta^limbs), a
 *       192-bit exact accumulator, then base-beta normalisation with the top
 *       digit reduced mod p^(M - limb_exp*(limbs-1)).
 *   oracle_matvec        reference matvec, linalg.hpp:144-192.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef struct {
  uint64_t w[3];
} u192;

static void add_prod(u192* a, uint64_t x, uint64_t y) {
  u128 pr = (u128)x * y;
  u128 lo = (u128)a->w[0] + (uint64_t)pr;
  a->w[0] = (uint64_t)lo;
  u128 mid = (u128)a->w[1] + (uint64_t)(pr >> 64) + (uint64_t)(lo >> 64);
  a->w[1] = (uint64_t)mid;
  a->w[2] += (uint64_t)(mid >> 64);
}

static void add192(u192* a, const u192* b) {
  u128 lo = (u128)a->w[0] + b->w[0];
  a->w[0] = (uint64_t)lo;
  u128 mid = (u128)a->w[1] + b->w[1] + (uint64_t)(lo >> 64);
  a->w[1] = (uint64_t)mid;
  a->w[2] += b->w[2] + (uint64_t)(mid >> 64);
}

static uint64_t divmod(u192* v, uint64_t beta) {
  u128 cur = v->w[2];
  uint64_t q2 = (uint64_t)(cur / beta);
  cur = ((cur % beta) << 64) | v->w[1];
  uint64_t q1 = (uint64_t)(cur / beta);
  cur = ((cur % beta) << 64) | v->w[0];
  uint64_t q0 = (uint64_t)(cur / beta);
  uint64_t r = (uint64_t)(cur % beta);
  v->w[0] = q0;
  v->w[1] = q1;
  v->w[2] = q2;
  return r;
}

static void normalise(u192* acc, int limbs, uint64_t beta, uint64_t top_mod, uint64_t* out) {
  u192 carry = {{0, 0, 0}};
  for (int s = 0; s < limbs; ++s) {
    u192 v = acc[s];
    add192(&v, &carry);
    out[s] = divmod(&v, beta);
    carry = v;
  }
  out[limbs - 1] %= top_mod;
}

static uint64_t ipow(uint64_t p, int e) {
  uint64_t r = 1;
  for (int i = 0; i < e; ++i) r *= p;
  return r;
}

/* y = (t A + B) x, or A x when B == NULL */
static void factor(int limbs, uint64_t beta, uint64_t top_mod, int side, const uint64_t* A, const uint64_t* B,
                   uint64_t t, const uint64_t* x, uint64_t* y) {
  size_t nn = (size_t)side * side;
  u192 accA[8], accB[8], comb[8];
  uint64_t da[8], db[8], out[8];
  for (int i = 0; i < side; ++i) {
    memset(accA, 0, sizeof accA);
    memset(accB, 0, sizeof accB);
    for (int j = 0; j < side; ++j)
      for (int t1 = 0; t1 < limbs; ++t1) {
        uint64_t a = A[t1 * nn + (size_t)i * side + j];
        uint64_t b = B ? B[t1 * nn + (size_t)i * side + j] : 0;
        for (int t2 = 0; t1 + t2 < limbs; ++t2) {
          uint64_t xv = x[(size_t)t2 * side + j];
          add_prod(&accA[t1 + t2], a, xv);
          if (B) add_prod(&accB[t1 + t2], b, xv);
        }
      }
    normalise(accA, limbs, beta, top_mod, da);
    if (!B) {
      for (int s = 0; s < limbs; ++s) y[(size_t)s * side + i] = da[s];
      continue;
    }
    normalise(accB, limbs, beta, top_mod, db);
    for (int s = 0; s < limbs; ++s) {
      comb[s].w[0] = db[s];
      comb[s].w[1] = comb[s].w[2] = 0;
      add_prod(&comb[s], t, da[s]);
    }
    normalise(comb, limbs, beta, top_mod, out);
    for (int s = 0; s < limbs; ++s) y[(size_t)s * side + i] = out[s];
  }
}

int oracle_linrec_eval(uint64_t p, int M, int limbs, int limb_exp, uint64_t beta, int side, const uint64_t* A,
                       const uint64_t* B, int64_t tmax, uint64_t* w) {
  if (limbs < 1 || limbs > 8 || tmax < 0) return 1;
  uint64_t top_mod = ipow(p, M - limb_exp * (limbs - 1));
  size_t vn = (size_t)limbs * side;
  uint64_t* nxt = (uint64_t*)malloc(vn * sizeof(uint64_t));
  uint64_t* cur = (uint64_t*)malloc(vn * sizeof(uint64_t));
  memcpy(cur, w, vn * sizeof(uint64_t));
  for (int64_t t = tmax; t >= 0; --t) {
    factor(limbs, beta, top_mod, side, A, B, (uint64_t)t, cur, nxt);
    uint64_t* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  memcpy(w, cur, vn * sizeof(uint64_t));
  free(cur);
  free(nxt);
  return 0;
}

int oracle_matvec(uint64_t p, int M, int limbs, int limb_exp, uint64_t beta, int side, const uint64_t* A,
                  const uint64_t* x, uint64_t* y) {
  if (limbs < 1 || limbs > 8) return 1;
  factor(limbs, beta, ipow(p, M - limb_exp * (limbs - 1)), side, A, NULL, 0, x, y);
  return 0;
}
