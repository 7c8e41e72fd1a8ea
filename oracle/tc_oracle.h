/*
 * tc_oracle.h -- CPU restatement of the reference triangle-pair kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * Restates /root/reference/pkg/src/tricontact/kernels.py (RK below) per pair,
 * in the exact IEEE operation order numpy uses there (no FMA contraction; the
 * 3-term einsum reduction order pinned in oracle/README.md), so that its
 * outputs are bit-identical to the reference run in place.  Pinned against
 * the tests/golden fixtures generated from the reference itself
 * (tests/golden/make_golden.py).
 */
#ifndef TC_ORACLE_H
#define TC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as tc_params in include/tricontact_b200.h (RK/kernels.py:42-72). */
typedef struct {
    double epsilon, c_factor, alpha_iterative, alpha_regulariser, move_factor, start_coord;
    int32_t n_iterative;
    int32_t flags;
} tco_params;

#define TCO_N_MARGINS 10

/* Result columns (RK/kernels.py:96-105): any pointer may be NULL.
 * ids: 4 bytes per pair (see oracle/README.md); NULL to skip. */
#define TCO_DECL(SFX, REAL)                                                              \
    int tco_comparison_##SFX(const REAL* A, const REAL* B, int64_t n, const REAL* eps,   \
                             REAL* distance, REAL* point_a, REAL* point_b, REAL* bary_a, \
                             REAL* bary_b, int8_t* kind, uint8_t* ids, int threads);     \
    int tco_iterative_##SFX(const REAL* A, const REAL* B, int64_t n, const REAL* eps,    \
                            const tco_params* p, REAL* distance, REAL* point_a,          \
                            REAL* point_b, REAL* bary_a, REAL* bary_b, int8_t* kind,     \
                            uint8_t* ids, int threads);                                  \
    int tco_hybrid_##SFX(const REAL* A, const REAL* B, int64_t n, const REAL* eps,       \
                         const uint8_t* allow_fb, const tco_params* p, REAL* distance,   \
                         REAL* point_a, REAL* point_b, REAL* bary_a, REAL* bary_b,       \
                         int8_t* kind, uint8_t* ids, int64_t* counts, int threads);      \
    int tco_closest_point_triangle_##SFX(const REAL* P, const REAL* T, int64_t n,        \
                                         REAL* closest, REAL* bary, int threads);        \
    int tco_degenerate_##SFX(const REAL* T, int64_t n, double rel_tol, uint8_t* mask, int threads);              \
    int tco_apply_motion_##SFX(const REAL* points, int64_t n, const double* quat, const REAL* t, \
                               REAL* out);                                                    \
    int tco_margins_##SFX(const REAL* A, const REAL* B, int64_t n, const REAL* eps,              \
                          const tco_params* p, double* margins, int threads);

TCO_DECL(f64, double)
TCO_DECL(f32, float)

#ifdef __cplusplus
}
#endif
#endif
