/* drzg — B200-native controlled-reduction engine (arXiv 2602.24155).
 *
 * The drop-in boundary: a plain C ABI (no C++ or torch types) over the
 * device kernels and the device-resident reduction engine.  Each entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj/include/drzeta/).  All functions return 0 on success;
 * on failure they return nonzero and drzg_last_error() holds the message
 * (the reference's contract_error text, file:line included).  Functions that
 * return char* hand back a malloc'd JSON document (free with drzg_free); on
 * failure they return NULL.
 *
 * Residue layouts at this boundary are the reference's:
 *   ModMatrix / ModVec (linalg.hpp:94-141): `limbs` planes of base-beta
 *   digits, plane-major then row-major, beta = p^limb_exp from StripePlan.
 *   Hypersurface coefficients: one per degree-d monomial in the reference's
 *   grevlex-descending order (monomial.hpp:84-149).
 */
#ifndef DRZG_H
#define DRZG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* StripePlan (linalg.hpp:20-58) */
typedef struct drzg_stripe_plan {
  uint64_t p;
  int32_t M;
  int32_t limbs;
  int32_t limb_exp;
  int32_t pad_;
  uint64_t beta;
  int64_t stripe;
} drzg_stripe_plan;

const char* drzg_last_error(void);
void drzg_free(char* s);
int drzg_device_count(void);

/* StripePlan::make(p, M)  — linalg.hpp:35-58 */
int drzg_stripe_plan_make(uint64_t p, int32_t M, drzg_stripe_plan* out);

/* linrec_eval(A, B, tmax, w, ctr) — linalg.hpp:337-410.
 * w <- M(0) M(1) ... M(tmax) w with M(t) = t*A + B (factor t = tmax first),
 * side x side operands; host buffers (copied to and from the device inside
 * the call).  *matvecs += tmax + 1. */
int drzg_linrec_eval(const drzg_stripe_plan* plan, int32_t side, const uint64_t* A, const uint64_t* B, int64_t tmax,
                     uint64_t* w, int64_t* matvecs);

/* same, all pointers in device memory, launched on `stream`
 * (cudaStream_t or NULL); *kernel_ms receives the CUDA-event time of the
 * stepping kernels when non-NULL */
int drzg_linrec_eval_device(const drzg_stripe_plan* plan, int32_t side, const uint64_t* dA, const uint64_t* dB,
                            int64_t tmax, uint64_t* dw, int64_t* matvecs, void* stream, float* kernel_ms);

/* detail::sparse_steps(plan, A, B, tmax, w, ctr) — linalg.hpp:257-331.
 * A and B in SparseOp CSC form (linalg.hpp:219-252): col_ptr[side+1],
 * row_idx[nnz], digs[nnz*limbs] entry-major. */
int drzg_sparse_steps(const drzg_stripe_plan* plan, int32_t side, const int64_t* a_col_ptr, const int32_t* a_row_idx,
                      const uint64_t* a_digs, const int64_t* b_col_ptr, const int32_t* b_row_idx,
                      const uint64_t* b_digs, int64_t tmax, uint64_t* w, int64_t* matvecs);

/* reduce_chunk(C, store, st, v, k, ledger) — reduction.hpp:394-423, for one
 * state of the hypersurface (p, n, d, coeffs) at working precision M and the
 * default working set; w in ModVec layout, updated in place; u updated. */
char* drzg_reduce_chunk(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int32_t* u,
                        int32_t pole, const int32_t* v, int64_t k, uint64_t* w, int32_t device);

/* frobenius_matrix(X, B, plan, policy, pep, S, only_pole, threads) —
 * zeta.hpp:36-136.  policy: 0 p-chunk.  columns: optional subset (NULL = all)
 * for partitioning across GPUs.  JSON: F (b*b decimal strings, row-major),
 * charpoly residues mod p^(M+n) (all columns only), plan, ledger
 * (matvecs/startups/combines), stage and kernel timings. */
char* drzg_frobenius(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t policy, int32_t r_uniform,
                     int32_t nm_override, int32_t only_pole, const int32_t* columns, int32_t ncolumns,
                     int32_t device, int32_t profile);

/* run_zeta(X, opts) — zeta.hpp:438-549.  JSON: Q, ambiguity, plan, slopes,
 * invariants (p-rank, height, domino, newton height), count checks, ledger,
 * wall time.  count_budget: ZetaOptions::count_budget (zeta.hpp:406), the
 * largest #P^n(F_{p^r}) the brute-force checks enumerate; <= 0 keeps the
 * reference default 2e8 (the GPU counter makes larger budgets cheap: the
 * cubic fourfold's r = 2 check enumerates 2.9e8 points of P^5(F_49)). */
char* drzg_zeta(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t policy, int32_t r_uniform,
                int32_t nm_override, int32_t verify_counts, int64_t count_budget, int32_t device, int32_t profile);

/* the rest of run_zeta on a given Frobenius matrix (zeta.hpp:456-535): the
 * charpoly, recover_Q, the sign tie-break, Newton >= Hodge and the point-count
 * checks, for the plan choose_precision(overrides) after `escalations` steps
 * of escalate_plan.  F: b*b decimal strings, row-major (e.g. gathered from
 * several GPUs).  JSON {"status": "ok", Q, ...} or {"status": "escalate",
 * "reason": ...} when the reference would escalate the plan. */
char* drzg_zeta_from_F(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r_uniform,
                       int32_t nm_override, int32_t escalations, int32_t b, const char* const* F,
                       int32_t verify_counts, int64_t count_budget);

/* synthetic input by the reference CLI's generator rule (drzeta_main.cpp:112-122):
 * std::mt19937_64(seed), coefficient rng() % p per grevlex monomial, redrawn
 * until smooth for the full set and the policy's working set (run_zeta's two
 * checks, zeta.hpp:440-445).  fermat != 0 returns sum x_i^d.  coeffs_out
 * holds C(n+d, n) entries. */
int drzg_random_hypersurface(uint64_t p, int32_t n, int32_t d, uint64_t seed, int32_t policy, int32_t fermat,
                             uint64_t* coeffs_out, int32_t* tries_out);

/* brute-force #X(F_{p^r}) — oracle.hpp:190-245 (the driver's count checks) */
int drzg_count_points(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r, int64_t budget,
                      int64_t* out);

/* the same count enumerated on the GPU (one thread per point) */
int drzg_count_points_device(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r, int64_t budget,
                             int64_t* out);

/* charpoly + recover_Q on a given F (zeta.hpp:456-470); F as b*b decimal strings */
char* drzg_charpoly(uint64_t p, int32_t n, int32_t d, int32_t r_uniform, int32_t nm_override, int32_t b,
                    const char* const* F);

/* ---- reduction-policy interface on device-resident GameStates ----------
 *
 * drzg_ctx stands in for the reference's (RuvContext, PepStoreBase) pair of
 * one (f, S, p^M) run (reduction.hpp:150-242, 143-147): the shared Dixon
 * tables (Jp, Jp^-1 mod q, the gather/scatter tables) and the HBM slot pool
 * the states live in.  A state id names one GameState{u, pole, w}
 * (reduction.hpp:113-117); w crosses the boundary in ModVec layout (limbs
 * planes of base-beta digits over Homog_{dn-n}, linalg.hpp:94-117).  The
 * working set is default_S(n, d), or {n} for policy 2 (var-by-var),
 * zeta.hpp:433-436.  A context serves one call at a time (internal lock). */
typedef struct drzg_ctx drzg_ctx;

/* RuvContext(X, StripePlan::make(p, M), S) — reduction.hpp:150-195; NULL on error */
drzg_ctx* drzg_ctx_create(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int32_t policy,
                          int32_t device);
void drzg_ctx_free(drzg_ctx* ctx);
/* side = |Homog_{dn-n}| (RuvContext::side), floor_len = |Homog_{dn-n-1}|,
 * the StripePlan of the ModVec layout, and the device digit plan q^Ld */
int drzg_ctx_info(drzg_ctx* ctx, int32_t* side, int32_t* floor_len, drzg_stripe_plan* plan, int32_t* digit_base,
                  int32_t* digit_planes);
/* upload GameStates (e.g. seed_reduction_input's, reduction.hpp:538-563):
 * u: count x (n+1), pole: count, w: count x (limbs x side) */
int drzg_states_seed(drzg_ctx* ctx, int32_t count, const int32_t* u, const int32_t* pole, const uint64_t* w,
                     int32_t* ids_out);
/* download states; any output pointer may be NULL */
int drzg_states_read(drzg_ctx* ctx, int32_t count, const int32_t* ids, int32_t* u_out, int32_t* pole_out,
                     uint64_t* w_out);
int drzg_states_free(drzg_ctx* ctx, int32_t count, const int32_t* ids);
/* reduce_chunk(C, store, st, v, k, ledger) for every listed state at once —
 * reduction.hpp:394-423: k pole drops along v (count x (n+1)); u <- u - k v,
 * pole <- pole - k.  ledger (matvecs, startups, combines) is added to. */
int drzg_step_batch(drzg_ctx* ctx, int32_t count, const int32_t* ids, const int32_t* v, const int64_t* k,
                    int64_t* ledger);
/* combine_states(states, ledger) — reduction.hpp:426-451: states with equal
 * (u, pole) are summed into the first; ids_out receives the survivors in
 * order (the others are freed) */
int drzg_states_combine(drzg_ctx* ctx, int32_t count, const int32_t* ids, int32_t* ids_out, int32_t* count_out,
                        int64_t* ledger);
/* run_policy(C, store, states, policy, ledger) — reduction.hpp:464-533:
 * drives every state to pole n (0 p-chunk, 1 depth-first, 2 var-by-var);
 * ids_out receives the floor states the reference returns */
int drzg_run_policy(drzg_ctx* ctx, int32_t count, const int32_t* ids, int32_t policy, int32_t* ids_out,
                    int32_t* count_out, int64_t* ledger);
/* floor_to_numerator(C, st, g) for every listed floor state — reduction.hpp:
 * 566-581: g (ModVec layout over Homog_{dn-n-1}, floor_len entries) += x^{u-1} w */
int drzg_floor_accumulate(drzg_ctx* ctx, int32_t count, const int32_t* ids, uint64_t* g);

/* ---- the linear-recurrence data structure (PEP) ------------------------
 *
 * PepStoreBase::get(v) / stats() (reduction.hpp:143-147) over a context, with
 * make_pep_store's backings "eager", "lazy", "lru:N", "lfuda:N" (pep.hpp:
 * 15-209): exactly-once builds under concurrency, shared entries (an eviction
 * never invalidates a held one).  An entry is build_ruv(C, v) (reduction.hpp:
 * 253-297): the n+2 matrices A_0..A_n, A_{n+1}, computed from the device's
 * unit-vector solves Jp^-1 e_j.  NULL on error (drzg_last_error). */
typedef struct drzg_pep_store drzg_pep_store;
drzg_pep_store* drzg_pep_store_create(drzg_ctx* ctx, const char* spec);
void drzg_pep_store_free(drzg_pep_store* store);
/* entry for move vector v (n+1 exponents, |v| = d): planes_out (may be NULL)
 * receives (n+2) x limbs x side x side u64 (ModMatrix plane layout per
 * matrix, linalg.hpp:119-141), nnz_out the PepEntry::nnz count */
int drzg_pep_get(drzg_pep_store* store, const int32_t* v, uint64_t* planes_out, int64_t* nnz_out);
/* PepStats: hits, misses, evictions */
int drzg_pep_stats(drzg_pep_store* store, int64_t* hits, int64_t* misses, int64_t* evictions);
/* eval_to_linear(E, x, v, plan) — reduction.hpp:300-339: A = sum_i v_i A_i,
 * B = sum_i x_i A_i + A_{n+1} (ModMatrix layout), the operands drzg_linrec_eval takes */
int drzg_pep_eval_to_linear(drzg_pep_store* store, const int32_t* v, const int32_t* x, uint64_t* A, uint64_t* B);
/* test hook: a store over stub entries (no device), for the backings' bookkeeping */
drzg_pep_store* drzg_pep_store_create_stub(int32_t nv, int32_t d, const char* spec);

/* ---- multi-GPU: the Frobenius gather over NCCL -------------
 *
 * One process per GPU reduces a subset of the columns (drzg_frobenius with
 * `columns`); the columns are independent (zeta.hpp:109-133).  drzg_gather_F
 * assembles F on every rank with one ncclAllGather of 62-bit limbs plus each
 * rank's column-ownership mask (no reduction: every entry has one owner, and
 * NCCL's integer Sum would wrap mod 2^64).  The communicator is NCCL's:
 * rank 0 makes the id, the caller ships it to the other ranks (e.g. over
 * torch.distributed), every rank calls drzg_comm_init.  NCCL is resolved at
 * run time (the process's libnccl.so.2, else the system one). */
#define DRZG_NCCL_ID_BYTES 128
typedef struct drzg_comm drzg_comm;
int drzg_nccl_unique_id(uint8_t* id_out);
drzg_comm* drzg_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, int32_t device);
void drzg_comm_free(drzg_comm* comm);
/* F_local: b*b decimal strings (this rank's columns filled); cols: the ncols
 * columns this rank owns; width: 62-bit limbs per entry.  JSON {"F": [...]}
 * (the full matrix, on every rank); NULL on error */
char* drzg_gather_F(drzg_comm* comm, int32_t b, const char* const* F_local, const int32_t* cols, int32_t ncols,
                    int32_t width);
/* test hook: the same encode/decode without NCCL for nranks blocks at once
 * (F_blocks: nranks x b*b strings; rank r owns cols[col_ptr[r] .. col_ptr[r+1])) */
char* drzg_gather_F_host(int32_t nranks, int32_t b, const char* const* F_blocks, const int32_t* cols,
                         const int32_t* col_ptr, int32_t width);

/* Fedder's F-splitting criterion, one of run_zeta's invariants (zeta.hpp:
 * 336-350): *out = 1 / 0, or -1 where run_zeta leaves it undefined (d > n+1).
 * Host only.  0 on success. */
int drzg_fsplit(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* DRZG_H */
