/*
 * tc_oracle.c -- instantiates the CPU restatement of RK/kernels.py for
 * float64 and float32.  TEST INFRASTRUCTURE ONLY (see tc_oracle.h).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).  The 3-term
 * dot-product reduction order is the one numpy 2.3's einsum("ij,ij->i")
 * uses on this container's AVX-512 dispatch, pinned by
 * tests/test_oracle_golden.py against vectors made by the reference itself:
 *   float64: (p0 + p2) + p1     float32: (p0 + p1) + p2
 */
#include <math.h>
#include <stdint.h>

#include "tc_oracle.h"

#include <pthread.h>

#define TCO_MAX_THREADS 256

typedef void (*tco_body_fn)(int64_t lo, int64_t hi, int tid, void* arg);

typedef struct {
    tco_body_fn fn;
    void* arg;
    int64_t lo, hi;
    int tid;
} tco_job;

static void* tco_run_job(void* p) {
    tco_job* j = (tco_job*)p;
    j->fn(j->lo, j->hi, j->tid, j->arg);
    return NULL;
}

/* Static contiguous split of [0, n) over `threads` POSIX threads. */
static void tco_parallel_for(int64_t n, int threads, tco_body_fn fn, void* arg) {
    if (threads < 1) threads = 1;
    if (threads > TCO_MAX_THREADS) threads = TCO_MAX_THREADS;
    if (n < 4096 || threads == 1) {
        fn(0, n, 0, arg);
        return;
    }
    pthread_t th[TCO_MAX_THREADS];
    tco_job jobs[TCO_MAX_THREADS];
    int started[TCO_MAX_THREADS];
    for (int t = 0; t < threads; ++t) {
        jobs[t].fn = fn;
        jobs[t].arg = arg;
        jobs[t].lo = n * t / threads;
        jobs[t].hi = n * (t + 1) / threads;
        jobs[t].tid = t;
        started[t] = (t > 0) && pthread_create(&th[t], NULL, tco_run_job, &jobs[t]) == 0;
        if (t > 0 && !started[t]) tco_run_job(&jobs[t]);
    }
    tco_run_job(&jobs[0]);
    for (int t = 1; t < threads; ++t)
        if (started[t]) pthread_join(th[t], NULL);
}

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)

#define REAL double
#define SFX f64
#define SQRT sqrt
#define FMA fma
#define DOT3_ORDER_02_1 1
#include "tc_oracle_impl.h"
#undef REAL
#undef SFX
#undef SQRT
#undef FMA
#undef DOT3_ORDER_02_1

#define REAL float
#define SFX f32
#define SQRT sqrtf
#define FMA fmaf
#define DOT3_ORDER_02_1 0
#include "tc_oracle_impl.h"
#undef REAL
#undef SFX
#undef SQRT
#undef FMA
#undef DOT3_ORDER_02_1
