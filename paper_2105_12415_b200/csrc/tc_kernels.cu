// tc_kernels.cu -- sm_100a kernels and the C ABI of include/tricontact_b200.h.
//
// Kernels (one triangle pair per thread, grid-stride / persistent over the
// pair range, grid sized to the SM count x resident CTAs per SM; CTA sizes
// per kernel, see BS_* below):
//   comparison_kernel  RK/kernels.py:301-401
//   iterative_kernel   RK/kernels.py:447-565 (pairs double-buffered in
//       shared memory by cp.async one tile ahead)
//   hybrid_kernel      RK/kernels.py:568-605 -- iterative for a tile of one
//       pair per thread, NOT_TERMINATED lanes (with allow_fb) are appended to
//       a shared-memory queue by warp ballot; whenever the queue holds a full
//       CTA of pairs, all threads screen them for degenerate triangles and
//       run the comparison phases on them, so the divergent fallback executes
//       on full warps.  The fallback never leaves the kernel.
//   blocks_hybrid_kernel  all-pairs particle blocks (RK/stepping.py:285-308,
//       RK/contact.py:97-140): both meshes staged in shared memory, optional
//       fused rigid motions (RK/geometry.py:162-176)
//   frontier_hybrid_kernel + frontier_count/write_kernel  the multiscale
//       traversal's rounds (RK/stepping.py:311-368)
//   cpt_kernel / ptd_kernel / degenerate_kernel: RK/kernels.py:157,
//       RK/surrogate.py:237-257, RK/geometry.py:68.
// Every kernel reduces its tallies per CTA (warp shuffles) and folds them
// into a device tc_stats with one set of atomics per CTA.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cub/device/device_scan.cuh>
#include <vector>
#include <mutex>
#include <condition_variable>
#include <memory>
#include <thread>
#include <dlfcn.h>
#if __has_include(<nccl.h>)
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed on first use (tc_allreduce_stats)
#else
// the few NCCL types tc_allreduce_stats uses (ABI-stable values of nccl.h)
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclSum = 0, ncclMin = 3 } ncclRedOp_t;
typedef enum { ncclInt64 = 4, ncclFloat64 = 8 } ncclDataType_t;
#endif

#include "tc_pair.cuh"
#include "../../include/tricontact_b200.h"

namespace tc {

// CTA sizes.  BLOCK (256) serves the one-pair-per-thread helpers and is the
// largest CTA; the batched kernels pick their own size (measured on cfg1):
// the iterative and all-pairs block kernels run 256-thread CTAs, the hybrid
// and multiscale-frontier kernels 128-thread CTAs, whose queue batches and
// per-tile barriers span half as many warps (+3 % hybrid; 64 and 96 are
// slower), the comparison kernel 64-thread CTAs (+7 % over 256); the
// iterative kernel loses 3 % at 128.  Device helpers
// read the CTA size from blockDim.x.
constexpr int BLOCK = 256;
#ifndef TC_BS_ITER
#define TC_BS_ITER 256
#endif
#ifndef TC_BS_HYB
#define TC_BS_HYB 128
#endif
#ifndef TC_BS_CMP
#define TC_BS_CMP 64
#endif
#ifndef TC_BS_BLK
#define TC_BS_BLK 256
#endif
#ifndef TC_BS_FRONT
#define TC_BS_FRONT 128
#endif
constexpr int BS_ITER = TC_BS_ITER, BS_HYB = TC_BS_HYB, BS_CMP = TC_BS_CMP, BS_BLK = TC_BS_BLK,
              BS_FRONT = TC_BS_FRONT;
// resident CTAs per SM of a bs-thread kernel for a register budget given as
// CTAs of 256 threads (launch bounds)
#define TC_MINB(bs, n256) ((n256) * 256 / (bs))
// L2 bulk prefetch of the next tile's inputs at the start of each tile: +0.7 %
// with the round-1 kernels, -0.5 % (fp64) / -1.6 % (fp32) with the round-2
// fallback phases (tools/varbench.py, 2^24 cfg1 pairs): off
#ifndef TC_PREFETCH
#define TC_PREFETCH 0
#endif
// dynamic shared memory of the comparison phases, per thread (stride BLOCK):
// [crossing points: SCR values (at most 4 points, see comparison_phase1);
//  in phase 2 the hoisted edge lengths and reciprocals]
// [pair slot: SLOT values]
constexpr int SCR = 12;
constexpr int SLOT = 18;
// resident CTAs per SM the register allocator targets (launch bounds)
#ifndef TC_ITER_MINB
#define TC_ITER_MINB 2
#endif
#ifndef TC_HYBRID_MINB
#define TC_HYBRID_MINB 2
#endif

static std::atomic<int64_t> g_launches{0};
static std::atomic<int64_t> g_max_ctas{0};  // test knob: tc_debug_set_max_ctas
static thread_local char g_err[512] = "";

static int set_err(const char* what, cudaError_t e) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return TC_ECUDA;
}

template <typename T>
struct Args {
    const T* tri_a;
    const T* tri_b;
    int64_t n;
    const T* eps;
    T eps_scalar;
    const uint8_t* allow;
    T* distance;
    T* pa;
    T* pb;
    T* ba;
    T* bb;
    int8_t* kind;
    uint8_t* ids;
    tc_stats* stats;
    double c_factor, alpha_it, alpha_reg, move_factor, start_coord;
    int n_iterative;
    // library-owned cumulative counters {pairs, fallbacks} of the warp-specialised hybrid's
    // launches on this device (fallback_history): device memory, and the host-mapped
    // copy CTA 0 refreshes; or NULL
    unsigned long long* hist = nullptr;
    unsigned long long* hist_host = nullptr;
};

template <class R, class A>
__device__ __forceinline__ KP<R> make_kp(const A& a) {
    using T = typename Store<R>::type;
    KP<R> k;
    k.c_factor = R(T(a.c_factor));
    k.alpha_it = R(T(a.alpha_it));
    k.alpha_reg = R(T(a.alpha_reg));
    k.move_factor = R(T(a.move_factor));
    k.start_coord = R(T(a.start_coord));
    k.n_iterative = a.n_iterative;
    return k;
}

// ---- loads / stores ---------------------------------------------------------
template <bool SOA, class R, typename T>
__device__ __forceinline__ void load_tri(const T* __restrict__ src, int64_t i, int64_t n, R* t) {
    if (SOA) {
#pragma unroll
        for (int k = 0; k < 9; ++k) t[k] = R(__ldg(src + k * n + i));
    } else {
        const T* p = src + 9 * i;
#pragma unroll
        for (int k = 0; k < 9; ++k) t[k] = R(__ldg(p + k));
    }
}

// The calling thread's planar shared-memory slot of 18 pair coordinates
// (stride BLOCK, conflict-free), `offset` elements into the dynamic smem.
template <typename T>
__device__ __forceinline__ T* thread_slot(int offset) {
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    return reinterpret_cast<T*>(tc_dyn_smem) + offset + threadIdx.x;
}

// Asynchronous copy of one pair (18 values) from global memory into the
// calling thread's slot (cp.async, LDGSTS: no registers, the copy lands while
// the thread computes); pairs j >= n copy nothing.  One commit group per call.
#ifndef TC_SMEM_PREFETCH
#define TC_SMEM_PREFETCH 1
#endif
// (Tried and measured slower for the hybrid kernel: a second pair slot filled
// by cp.async (the shared-memory growth shrinks L1, which holds the queued
// pairs' re-reads and the spills), 96-thread CTAs with a double-buffered
// slot, and a two-pass variant that runs the iterative over all of a CTA's
// tiles before its fallback.)
template <typename T>
__device__ __forceinline__ void cp_async_val(T* dst, const T* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Keep the register-resident pair in the thread's slot so the iterative
// epilogue re-reads it from shared memory instead of global memory.
template <int BS, class R, typename T>
__device__ __forceinline__ void stash_pair(T* slot, const R* A, const R* B) {
    constexpr int bs = BS;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        slot[k * bs] = val(A[k]);
        slot[(9 + k) * bs] = val(B[k]);
    }
}

// Two-value shared-memory words of a planar pair slot (TC_WS_PAIRED_F64 / _F32).
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <class R, typename T2>
__device__ __forceinline__ void stash_pair2(T2* slot2, const R* A, const R* B) {
    auto c = [&](int k) { return val(k < 9 ? A[k] : B[k - 9]); };
#pragma unroll
    for (int kk = 0; kk < 9; ++kk) {
        T2 v;
        v.x = c(2 * kk);
        v.y = c(2 * kk + 1);
        slot2[kk * 32] = v;
    }
}
// Coordinate k of the triangle starting at coordinate `first` (0: A, 9: B) of a paired slot.
template <class R>
struct PairTri {
    const typename Vec2<typename Store<R>::type>::type* p;
    int first;
    __device__ __forceinline__ R operator[](int k) const {
        const int c = first + k;
        const auto v = p[(c >> 1) * 32];
        return R((c & 1) ? v.y : v.x);
    }
    __device__ __forceinline__ void vertex(int k, R* v) const {
#pragma unroll
        for (int i = 0; i < 3; ++i) v[i] = (*this)[3 * k + i];
    }
};

// Iterative kernel for one pair: the reference's operation order in strict
// mode, the Gram-matrix form in the fast build (tc_pair.cuh).  SA / SB give
// the epilogue's re-reads of the pair (a shared-memory copy).
template <class R, class TA, class TB, class EpsFn>
__device__ __forceinline__ void run_iterative(const TA& SA, const TB& SB, const R* A, const R* B, EpsFn eps_fn,
                                              const KP<R>& kp, Rec<R>& r) {
    if constexpr (IsStrict<R>::value) {
        auto reload = [&](R* A0, R* B0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                A0[k] = SA[k];
                B0[k] = SB[k];
            }
        };
        if (kp.start_coord >= R(0) && kp.start_coord <= R(1)) iterative_pair<true>(A, B, eps_fn(), kp, r, reload);
        else iterative_pair<false>(A, B, eps_fn(), kp, r, reload);
    } else {
        auto reload = [&](R* A9, R* B9) {
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                A9[k] = SA[k];
                B9[k] = SB[k];
            }
        };
        if (kp.start_coord >= R(0) && kp.start_coord <= R(1)) iterative_pair_gram<true>(A, B, kp, r, reload, eps_fn);
        else iterative_pair_gram<false>(A, B, kp, r, reload, eps_fn);
    }
}
template <int BS, class R, typename T, class EpsFn>
__device__ __forceinline__ void run_iterative(const T* slot, const R* A, const R* B, EpsFn eps_fn, const KP<R>& kp,
                                              Rec<R>& r) {
    constexpr int bs = BS;
    run_iterative(SmemTri<R>{slot, bs}, SmemTri<R>{slot + 9 * bs, bs}, A, B, eps_fn, kp, r);
}

// L2 eviction-priority hints for the result stores (TC_OUT_HINT): the hybrid
// writes every lane's tile result at once and rewrites the open pairs' rows
// after their fallback, several tiles later.  Tile stores of open pairs can
// carry evict_last (their sectors stay in L2 until the rewrite, which then
// needs no DRAM read-modify-write), the fallback's final stores evict_first.
#ifndef TC_OUT_HINT
#define TC_OUT_HINT 0
#endif
__device__ __forceinline__ uint64_t l2_policy(bool last) {
    uint64_t p;
    if (last) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(int8_t* p, int8_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b8 [%0], %1, %2;" ::"l"(p), "h"((short)v), "l"(pol) : "memory");
}
template <typename T>
__device__ __forceinline__ void st_col(T* p, T v, bool hint, uint64_t pol) {
    if (hint) st_hint(p, v, pol);
    else *p = v;
}

// FULL: the caller checked at launch that every result column is requested
// and no feature ids are (the common drop-in / bench record): no per-column
// null tests in the kernel.
template <bool SOA, bool FULL, class R, typename T>
__device__ __forceinline__ void store_rec_full(const Args<T>& a, int64_t i, const Rec<R>& r) {
    static_assert(FULL, "");
    const int64_t n = a.n;
    a.distance[i] = val(r.distance);
    a.kind[i] = (int8_t)r.kind;
    if (SOA) {
        T* const pa = a.pa + i;
        T* const pb = a.pb + i;
        T* const ba = a.ba + i;
        T* const bb = a.bb + i;
        pa[0] = val(r.pa[0]); pa[n] = val(r.pa[1]); pa[2 * n] = val(r.pa[2]);
        pb[0] = val(r.pb[0]); pb[n] = val(r.pb[1]); pb[2 * n] = val(r.pb[2]);
        ba[0] = val(r.ba[0]); ba[n] = val(r.ba[1]);
        bb[0] = val(r.bb[0]); bb[n] = val(r.bb[1]);
    } else {
        T* const pa = a.pa + 3 * i;
        T* const pb = a.pb + 3 * i;
        pa[0] = val(r.pa[0]); pa[1] = val(r.pa[1]); pa[2] = val(r.pa[2]);
        pb[0] = val(r.pb[0]); pb[1] = val(r.pb[1]); pb[2] = val(r.pb[2]);
        a.ba[2 * i] = val(r.ba[0]); a.ba[2 * i + 1] = val(r.ba[1]);
        a.bb[2 * i] = val(r.bb[0]); a.bb[2 * i + 1] = val(r.bb[1]);
    }
}
template <typename T>
static bool full_record(const Args<T>& a) {
    return a.distance && a.kind && a.pa && a.pb && a.ba && a.bb && !a.ids;
}

template <bool SOA, class R, typename T>
__device__ __forceinline__ void store_rec(const Args<T>& a, int64_t i, const Rec<R>& r, bool hint = false,
                                          uint64_t pol = 0) {
    const int64_t n = a.n;
    if (a.distance) st_col(a.distance + i, val(r.distance), hint, pol);
    if (a.kind) st_col(a.kind + i, (int8_t)r.kind, hint, pol);
    if (SOA) {
        if (a.pa) { st_col(a.pa + i, val(r.pa[0]), hint, pol); st_col(a.pa + n + i, val(r.pa[1]), hint, pol);
                    st_col(a.pa + 2 * n + i, val(r.pa[2]), hint, pol); }
        if (a.pb) { st_col(a.pb + i, val(r.pb[0]), hint, pol); st_col(a.pb + n + i, val(r.pb[1]), hint, pol);
                    st_col(a.pb + 2 * n + i, val(r.pb[2]), hint, pol); }
        if (a.ba) { st_col(a.ba + i, val(r.ba[0]), hint, pol); st_col(a.ba + n + i, val(r.ba[1]), hint, pol); }
        if (a.bb) { st_col(a.bb + i, val(r.bb[0]), hint, pol); st_col(a.bb + n + i, val(r.bb[1]), hint, pol); }
    } else {
        if (a.pa) { st_col(a.pa + 3 * i, val(r.pa[0]), hint, pol); st_col(a.pa + 3 * i + 1, val(r.pa[1]), hint, pol);
                    st_col(a.pa + 3 * i + 2, val(r.pa[2]), hint, pol); }
        if (a.pb) { st_col(a.pb + 3 * i, val(r.pb[0]), hint, pol); st_col(a.pb + 3 * i + 1, val(r.pb[1]), hint, pol);
                    st_col(a.pb + 3 * i + 2, val(r.pb[2]), hint, pol); }
        if (a.ba) { st_col(a.ba + 2 * i, val(r.ba[0]), hint, pol); st_col(a.ba + 2 * i + 1, val(r.ba[1]), hint, pol); }
        if (a.bb) { st_col(a.bb + 2 * i, val(r.bb[0]), hint, pol); st_col(a.bb + 2 * i + 1, val(r.bb[1]), hint, pol); }
    }
    if (a.ids) {
        uint8_t* p = a.ids + 4 * i;
        if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(p) = r.ids;
        } else {
            p[0] = r.ids & 0xFF; p[1] = (r.ids >> 8) & 0xFF; p[2] = (r.ids >> 16) & 0xFF; p[3] = r.ids >> 24;
        }
    }
}

// ---- per-CTA tallies -> tc_stats ----------------------------------------------
struct Tally {
    // per-thread counts fit 32 bits (a thread sees at most n / (grid * BLOCK)
    // pairs); widened to 64 bits in the CTA reduction
    unsigned iterative = 0, comparison = 0, degenerate = 0, contacts = 0, intersecting = 0;
    double min_d = __builtin_huge_val();
    float min_f = __builtin_huge_valf();  // fp32 kernels keep the running minimum in float (exact; no FP64 pipe)

    template <class R>
    __device__ __forceinline__ void result(const Rec<R>& r) {
        if (r.kind == KIND_DEGENERATE) return;
        contacts += (r.kind == KIND_CONTACT);
        intersecting += (r.ids >> 24) & FLAG_INTERSECT ? 1 : 0;
        if constexpr (sizeof(typename Store<R>::type) == 4) {
            const float d = (float)val(r.distance) + 0.0f;  // -0 -> +0
            min_f = (d < min_f) ? d : min_f;
        } else {
            const double d = (double)val(r.distance) + 0.0;  // -0 -> +0
            min_d = (d < min_d) ? d : min_d;
        }
    }

    // COMPARISON_IS_FALLBACK: hybrid comparisons also count as fallbacks
    template <bool COMPARISON_IS_FALLBACK, int NWARPS = BLOCK / 32>
    __device__ void flush(tc_stats* s, unsigned long long* hist = nullptr, unsigned long long* hist_host = nullptr,
                          unsigned ring_waits = 0, unsigned self_tiles = 0) {  // (the CTA's, read by thread 0)
        if (!s && !hist) return;
        __shared__ unsigned long long red[5][NWARPS];  // iterative, comparison, degenerate, contacts, intersecting
        __shared__ double redm[NWARPS];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if ((double)min_f < min_d) min_d = (double)min_f;
        unsigned long long it64 = iterative, cm64 = comparison, dg64 = degenerate, ct64 = contacts,
                           ix64 = intersecting;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            it64 += __shfl_xor_sync(0xffffffffu, it64, off);
            cm64 += __shfl_xor_sync(0xffffffffu, cm64, off);
            dg64 += __shfl_xor_sync(0xffffffffu, dg64, off);
            ct64 += __shfl_xor_sync(0xffffffffu, ct64, off);
            ix64 += __shfl_xor_sync(0xffffffffu, ix64, off);
            const double o = __shfl_xor_sync(0xffffffffu, min_d, off);
            min_d = (o < min_d) ? o : min_d;
        }
        if (lane == 0) {
            red[0][wid] = it64; red[1][wid] = cm64; red[2][wid] = dg64; red[3][wid] = ct64;
            red[4][wid] = ix64;
            redm[wid] = min_d;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long v[5] = {0, 0, 0, 0, 0};
            double m = __builtin_huge_val();
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
                for (int k = 0; k < 5; ++k) v[k] += red[k][w];
                m = (redm[w] < m) ? redm[w] : m;
            }
            if (hist) {
                atomicAdd(hist, v[0]);
                atomicAdd(hist + 1, v[1] + v[2]);
                if (ring_waits) atomicAdd(hist + 2, (unsigned long long)ring_waits);
                if (self_tiles) atomicAdd(hist + 3, (unsigned long long)self_tiles);
                if (blockIdx.x == 0) {
                    // a few posted writes to host memory per launch (per-CTA system-scope
                    // reductions over PCIe cost 0.2 ms per launch); the totals of CTAs
                    // still running reach the host with the next launch.  The snapshot is
                    // bracketed by a sequence number (words 0 and 5) so the host never
                    // uses a torn one (a launch once read the new pair count with the old
                    // fallback count, took the rate for 0 and switched kernels).
                    __threadfence();
                    volatile unsigned long long* hh = hist_host;
                    const unsigned long long seq = atomicAdd(hist + 4, 1ull) + 1ull;
                    hh[0] = seq;
                    __threadfence_system();
                    for (int k = 0; k < 4; ++k) hh[1 + k] = ((volatile unsigned long long*)hist)[k];
                    __threadfence_system();
                    hh[5] = seq;
                }
            }
            if (!s) return;
            auto* c = reinterpret_cast<unsigned long long*>(s);
            if (v[0]) atomicAdd(c + 0, v[0]);
            if (v[1]) {
                atomicAdd(c + 1, v[1]);
                if (COMPARISON_IS_FALLBACK) atomicAdd(c + 2, v[1]);
            }
            if (v[2]) atomicAdd(c + 3, v[2]);
            if (v[3]) atomicAdd(c + 4, v[3]);
            if (v[4]) atomicAdd(c + 5, v[4]);
            // distances are >= 0 (or NaN, skipped): IEEE order == unsigned bit order
            if (m == m && m < __builtin_huge_val())
                atomicMin(reinterpret_cast<unsigned long long*>(&s->min_distance),
                          (unsigned long long)__double_as_longlong(m));
        }
    }
};

template <typename T, bool STRICT>
struct Pol { using R = T; };
template <typename T>
struct Pol<T, true> { using R = Strict<T>; };

// ---- kernels ---------------------------------------------------------------------

// Block-shared work queues of pair indices for the compacted comparison
// phases: q1 holds pairs awaiting phase 1 (crossings), q2 pairs awaiting
// phase 2 (features).  Bit 62 of a q2 entry marks "ids only".
template <int QB>  // the CTA size: one batch
struct Queues {
    int64_t q1[2 * QB];
    int64_t q2[2 * QB];
    int n1, n2;
};

// Shared-memory crossing-point scratch of the calling thread (4 x 3 values).
template <class R, int BS>
__device__ __forceinline__ Scratch<R> thread_scratch() {
    using T = typename Store<R>::type;
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    Scratch<R> s;
    s.p = reinterpret_cast<T*>(tc_dyn_smem) + threadIdx.x;
    s.stride = BS;
    return s;
}
// The calling thread's planar shared-memory slot for the pair under
// comparison (18 coordinates, stride BLOCK), after the crossing scratch.
// Timing-only experiment knobs (wrong results): TC_X_STAGE_HOT re-reads queued
// pairs from a small hot region, TC_X_TILE_HOT loads every tile from one, to
// bound what hiding those loads' latency could gain.
#ifndef TC_X_STAGE_HOT
#define TC_X_STAGE_HOT 0
#endif
#ifndef TC_X_TILE_HOT
#define TC_X_TILE_HOT 0
#endif
#ifndef TC_X_NOSTORE
#define TC_X_NOSTORE 0
#endif
template <bool SOA, int BS, class R, typename T>
__device__ __forceinline__ void stage_pair(const Args<T>& a, int64_t j, SmemTri<R>& A, SmemTri<R>& B, R& eps,
                                           T* slot) {
    constexpr int bs = BS;
    if (TC_X_STAGE_HOT) j &= 1023;
#ifndef TC_X_STAGE_NONE
#define TC_X_STAGE_NONE 0
#endif
#pragma unroll
    for (int k = 0; k < 9 * (1 - TC_X_STAGE_NONE); ++k) {
        slot[k * bs] = __ldg(SOA ? a.tri_a + k * a.n + j : a.tri_a + 9 * j + k);
        slot[(9 + k) * bs] = __ldg(SOA ? a.tri_b + k * a.n + j : a.tri_b + 9 * j + k);
    }
    A.p = slot;
    A.stride = bs;
    B.p = slot + 9 * bs;
    B.stride = bs;
    eps = R(a.eps ? a.eps[j] : a.eps_scalar);
}
template <typename T>
constexpr size_t scratch_bytes(int bs) { return sizeof(T) * (SCR + SLOT) * bs; }
constexpr int64_t IDS_ONLY = int64_t(1) << 62;

// Warp-aggregated append (all 32 lanes of the warp must call it).
// TC_DEBUG builds (libtricontact_b200_debug.so, tests/test_gpu_stress.py)
// trap on any queue overflow, out-of-range queued index or leftover queue
// entry -- the checks compute-sanitizer would otherwise provide, which this
// pool does not allow.
#ifndef TC_DEBUG
#define TC_DEBUG 0
#endif
#define TC_CHECK(cond)                  \
    do {                                \
        if (TC_DEBUG && !(cond)) __trap(); \
    } while (0)

__device__ __forceinline__ void push(int64_t* q, int* n, bool pred, int64_t v, int cap) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    TC_CHECK(base >= 0 && base + __popc(m) <= cap);
    if (pred) q[base + __popc(m & ((1u << lane) - 1u))] = v;
}

template <bool SOA, int BS, typename T>
__device__ __forceinline__ void async_pair(const Args<T>& a, int64_t j, T* slot) {
    if (j < a.n) {
        constexpr int bs = BS;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            cp_async_val(slot + k * bs, SOA ? a.tri_a + k * a.n + j : a.tri_a + 9 * j + k);
            cp_async_val(slot + (9 + k) * bs, SOA ? a.tri_b + k * a.n + j : a.tri_b + 9 * j + k);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <bool SOA, class R, typename T>
__device__ __forceinline__ void load_pair(const Args<T>& a, int64_t j, R* A, R* B, R& eps) {
    load_tri<SOA>(a.tri_a, j, a.n, A);
    load_tri<SOA>(a.tri_b, j, a.n, B);
    eps = R(a.eps ? a.eps[j] : a.eps_scalar);
}

// One elected thread asks the TMA unit to pull the CTA's next tile of inputs
// into L2 (cp.async.bulk.prefetch.L2: no registers, no shared memory), so the
// next tile's loads hit L2 instead of HBM.
template <bool SOA, int BS, typename T>
__device__ __forceinline__ void prefetch_tile(const Args<T>& a, int64_t tile) {
    if (!TC_PREFETCH || threadIdx.x != 0) return;
    constexpr int bs = BS;
    const int64_t start = tile * bs;
    if (start >= a.n) return;
    const int64_t cnt = (a.n - start) < bs ? (a.n - start) : bs;
    auto pf = [](const void* p, int64_t bytes) {
        bytes &= ~int64_t(15);
        if (bytes > 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)bytes) : "memory");
    };
    if (SOA) {
#pragma unroll 1
        for (int k = 0; k < 9; ++k) {
            pf(a.tri_a + k * a.n + start, cnt * (int64_t)sizeof(T));
            pf(a.tri_b + k * a.n + start, cnt * (int64_t)sizeof(T));
        }
    } else {
        pf(a.tri_a + 9 * start, 9 * cnt * (int64_t)sizeof(T));
        pf(a.tri_b + 9 * start, 9 * cnt * (int64_t)sizeof(T));
    }
}

// Where the comparison phases read a queued pair from and write its result
// to.  FlatSource: pair j of the flat (n,3,3)/SoA batch, staged into the
// thread's shared-memory slot; results into the BatchResult columns.
template <bool SOA, class R, typename T, int BS, bool FULL = false>
struct FlatSource {
    const Args<T>& a;
    T* slot;  // the calling thread's pair slot
    __device__ __forceinline__ bool want_ids() const { return !FULL && a.ids != nullptr; }
    __device__ __forceinline__ void stage(int64_t j, SmemTri<R>& A, SmemTri<R>& B, R& eps) const {
        TC_CHECK(j >= 0 && j < a.n);
        stage_pair<SOA, BS>(a, j, A, B, eps, slot);
    }
    __device__ __forceinline__ void store(int64_t j, const Rec<R>& r) const {
        if constexpr (FULL) store_rec_full<SOA, FULL>(a, j, r);
        else if (TC_OUT_HINT) store_rec<SOA>(a, j, r, true, l2_policy(false));
        else store_rec<SOA>(a, j, r);
    }
    __device__ __forceinline__ void store_ids01(int64_t j, uint32_t ids) const {
        if (FULL) return;
        a.ids[4 * j] = (uint8_t)(ids & 0xFF);
        a.ids[4 * j + 1] = (uint8_t)((ids >> 8) & 0xFF);
    }
    // row j keeps its (open: flags 0) iterative result; kind and flags say DEGENERATE
    __device__ __forceinline__ void mark_degenerate(int64_t j) const {
        if (FULL || a.kind) a.kind[j] = (int8_t)KIND_DEGENERATE;
        if (!FULL && a.ids) a.ids[4 * j + 3] = (uint8_t)FLAG_DEGENERATE;
    }
};

// Run whole batches (QB pairs -- the CTA size --, or the remainder when
// `final_`) from the queues until neither holds a full batch.  Block-uniform;
// every batch runs on full warps.  `fallback_flag`: hybrid results carry
// FLAG_FALLBACK.
// SCREEN: the batch's pairs are screened for degenerate triangles before
// phase 1 (RK/kernels.py:596-600) -- on full warps of open pairs instead of
// divergently in the producing tile; a degenerate pair keeps its iterative
// result and is marked DEGENERATE (src.mark_degenerate).
template <bool SCREEN = false, class R, class Src, int QB>
__device__ __forceinline__ void drain(const Src& src, Queues<QB>& Q, Tally& tl, bool final_, uint32_t fallback_flag) {
    const bool want_ids = src.want_ids();
    while (true) {
        const int c1 = Q.n1, c2 = Q.n2;
        TC_CHECK(c1 >= 0 && c1 <= 2 * QB && c2 >= 0 && c2 <= 2 * QB);
        __syncthreads();  // everyone has read the counts before they change
        int which = 0;
        if (c1 >= QB || (final_ && c1 > 0)) which = 1;
        else if (c2 >= QB || (final_ && c2 > 0)) which = 2;
        if (!which) break;
        const int c = which == 1 ? c1 : c2;
        const int m = c < QB ? c : QB;
        int64_t e = -1;
        if ((int)threadIdx.x < m) e = (which == 1 ? Q.q1 : Q.q2)[c - m + threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {
            if (which == 1) Q.n1 = c - m;
            else Q.n2 = c - m;
        }
        bool push2 = false;
        int64_t e2 = 0;
        if (e >= 0) {
            const int64_t j = e & (IDS_ONLY - 1);
            SmemTri<R> A, B;
            R eps;
            src.stage(j, A, B, eps);
            Rec<R> r;
            bool screened = false;
            if constexpr (SCREEN) {
                if (which == 1 && (degenerate_tri_t<R>(A) || degenerate_tri_t<R>(B))) {
                    src.mark_degenerate(j);
                    tl.degenerate++;
                    screened = true;
                }
            }
            if (screened) {
            } else if (which == 1) {
                tl.comparison++;
                if (comparison_phase1(A, B, eps, thread_scratch<R, QB>(), r)) {
                    r.ids |= fallback_flag << 24;
                    src.store(j, r);
                    tl.result(r);
                    push2 = want_ids;
                    e2 = j | IDS_ONLY;
                } else {
                    push2 = true;
                    e2 = j;
                }
            } else {
                const bool ids_only = (e & IDS_ONLY) != 0;
                comparison_phase2(A, B, eps, ids_only, r, thread_scratch<R, QB>());
                if (ids_only) {
                    src.store_ids01(j, r.ids);
                } else {
                    r.ids |= fallback_flag << 24;
                    src.store(j, r);
                    tl.result(r);
                }
            }
        }
        if (which == 1) push(Q.q2, &Q.n2, push2, e2, 2 * QB);
        __syncthreads();
    }
    TC_CHECK(!final_ || (Q.n1 == 0 && Q.n2 == 0));
}

template <typename T, bool STRICT, bool SOA>
__global__ void __launch_bounds__(BS_CMP, TC_MINB(BS_CMP, 2)) comparison_kernel(Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    __shared__ Queues<BS_CMP> Q;
    Tally tl;
    if (threadIdx.x == 0) Q.n1 = Q.n2 = 0;
    __syncthreads();
    const int64_t ntiles = (a.n + BS_CMP - 1) / BS_CMP;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t i = tile * BS_CMP + threadIdx.x;
        bool need2 = false;
        int64_t e2 = 0;
        if (i < a.n) {
            SmemTri<R> A, B;
            R eps;
            stage_pair<SOA, BS_CMP>(a, i, A, B, eps, thread_slot<T>(SCR * BS_CMP));
            Rec<R> r;
            tl.comparison++;
            if (comparison_phase1(A, B, eps, thread_scratch<R, BS_CMP>(), r)) {
                store_rec<SOA>(a, i, r);
                tl.result(r);
                need2 = a.ids != nullptr;
                e2 = i | IDS_ONLY;
            } else {
                need2 = true;
                e2 = i;
            }
        }
        push(Q.q2, &Q.n2, need2, e2, 2 * BS_CMP);
        __syncthreads();
        drain<false, R>(FlatSource<SOA, R, T, BS_CMP>{a, thread_slot<T>(SCR * BS_CMP)}, Q, tl, false, 0u);
    }
    drain<false, R>(FlatSource<SOA, R, T, BS_CMP>{a, thread_slot<T>(SCR * BS_CMP)}, Q, tl, true, 0u);
    // comparison_batch alone counts as comparison work but not as a fallback
    tl.flush<false>(a.stats);
}

template <typename T, bool STRICT, bool SOA>
__global__ void __launch_bounds__(BS_ITER, TC_MINB(BS_ITER, TC_ITER_MINB)) iterative_kernel(Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    const KP<R> kp = make_kp<R>(a);
    Tally tl;
    // double-buffered pair slots filled by cp.async one tile ahead (see hybrid_kernel)
    T* const slot0 = thread_slot<T>(0);
    int cur = 0;
    const int64_t stride = (int64_t)gridDim.x * BS_ITER;
    const int64_t first = (int64_t)blockIdx.x * BS_ITER + threadIdx.x;
    if (TC_SMEM_PREFETCH) async_pair<SOA, BS_ITER>(a, first, slot0);
    for (int64_t i = first; i - threadIdx.x < a.n; i += stride) {
        T* slot = slot0 + cur * (SLOT * BS_ITER);
        cur ^= 1;
        R A[9], B[9];
        if (TC_SMEM_PREFETCH) {
            cp_async_wait_all();
            async_pair<SOA, BS_ITER>(a, i + stride, slot0 + cur * (SLOT * BS_ITER));
            if (i >= a.n) continue;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                A[k] = R(slot[k * BS_ITER]);
                B[k] = R(slot[(9 + k) * BS_ITER]);
            }
        } else {
            if (i >= a.n) continue;
            R eps_unused;
            load_pair<SOA>(a, i, A, B, eps_unused);
            stash_pair<BS_ITER>(slot, A, B);
        }
        Rec<R> r;
        run_iterative<BS_ITER>(slot, A, B, [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
        store_rec<SOA>(a, i, r);
        tl.iterative++;
        tl.result(r);
    }
    tl.flush<false>(a.stats);
}

// (Tried: two pairs per thread interleaved, 384 threads per CTA -- twice the
// independent FP64 chains per warp but one CTA per SM at the register cap;
// measured slower than two 256-thread CTAs.)

// RK/kernels.py:568-605.  Per tile of BLOCK pairs: the iterative kernel on
// every lane; open (NOT_TERMINATED, fallback allowed) pairs are appended to
// q1; full batches of q1 are screened for degenerate triangles and run phase
// 1 of the comparison kernel, and non-intersecting ones move on to q2 for
// phase 2 -- so the screen and both fallback phases execute on full warps,
// inside this kernel.  (Running
// phase 1 in-tile on the compacted open lanes, straight from the owners'
// shared-memory slots, saves the re-read of queued pairs but idles half the
// warps: measured 8% slower on cfg1.)
// TC_TILE_CPASYNC: the next tile's pair is copied into a second per-thread
// shared-memory slot by cp.async while the current tile computes, so a tile
// starts from shared memory instead of waiting for its global loads.
#ifndef TC_TILE_CPASYNC
#define TC_TILE_CPASYNC 0
#endif
template <typename T, bool STRICT, bool SOA>
#ifndef TC_HYB_CTAS  // resident hybrid CTAs per SM the register budget targets
#define TC_HYB_CTAS TC_MINB(BS_HYB, TC_HYBRID_MINB)
#endif
#ifndef TC_HYB_CTAS_F32  // fp32: half the registers per value, 6 CTAs (80 registers) measured 2.3 % faster
#define TC_HYB_CTAS_F32 6
#endif
__global__ void __launch_bounds__(BS_HYB, sizeof(T) == 4 ? TC_HYB_CTAS_F32 : TC_HYB_CTAS) hybrid_kernel(Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    __shared__ Queues<BS_HYB> Q;
    const KP<R> kp = make_kp<R>(a);
    Tally tl;
    if (threadIdx.x == 0) Q.n1 = Q.n2 = 0;
    __syncthreads();
    const int64_t ntiles = (a.n + BS_HYB - 1) / BS_HYB;
    T* const slot = thread_slot<T>(SCR * BS_HYB);  // the comparison phases' pair slot, free here
    T* const nslot = thread_slot<T>((SCR + SLOT) * BS_HYB);  // TC_TILE_CPASYNC: the next tile's pair
    if (TC_TILE_CPASYNC) async_pair<SOA, BS_HYB>(a, (int64_t)blockIdx.x * BS_HYB + threadIdx.x, nslot);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (!TC_TILE_CPASYNC) prefetch_tile<SOA, BS_HYB>(a, tile + gridDim.x);
        const int64_t i = tile * BS_HYB + threadIdx.x;
        bool enq = false;
        if (TC_TILE_CPASYNC) cp_async_wait_all();
        if (i < a.n) {
            R A[9], B[9], eps;
            if (TC_TILE_CPASYNC) {
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    A[k] = R(nslot[k * BS_HYB]);
                    B[k] = R(nslot[(9 + k) * BS_HYB]);
                }
                eps = R(a.eps ? a.eps[i] : a.eps_scalar);
            } else {
                load_pair<SOA>(a, TC_X_TILE_HOT ? (i & 4095) : i, A, B, eps);
            }
            stash_pair<BS_HYB>(slot, A, B);
            // (the stash consumed the slot's values: the next copy may land)
            if (TC_TILE_CPASYNC) async_pair<SOA, BS_HYB>(a, i + (int64_t)gridDim.x * BS_HYB, nslot);
            Rec<R> r;
#ifndef TC_X_RELOAD_GLOBAL
#define TC_X_RELOAD_GLOBAL 0
#endif
            if (TC_X_RELOAD_GLOBAL && SOA)
                run_iterative(GlobalTri<R>{a.tri_a + i, a.n}, GlobalTri<R>{a.tri_b + i, a.n}, A, B,
                              [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
            else
                run_iterative<BS_HYB>(slot, A, B, [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
            tl.iterative++;
            // open pairs are queued; the phase-1 batches screen them for
            // degenerate triangles (drain<SCREEN>)
            enq = r.kind == KIND_NOT_TERMINATED && (a.allow == nullptr || a.allow[i]);
            // every lane stores its tile result now (open pairs a placeholder
            // the fallback overwrites), so output sectors are written whole
            if (!TC_X_NOSTORE) {
                if (TC_OUT_HINT) store_rec<SOA>(a, i, r, TC_OUT_HINT == 2 || enq, l2_policy(true));
                else store_rec<SOA>(a, i, r);
            }
            if (!enq) tl.result(r);
        } else if (TC_TILE_CPASYNC) {
            asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count uniform
        }
        push(Q.q1, &Q.n1, enq, i, 2 * BS_HYB);
        __syncthreads();
        drain<true, R>(FlatSource<SOA, R, T, BS_HYB>{a, slot}, Q, tl, false, (uint32_t)FLAG_FALLBACK);
    }
    if (TC_TILE_CPASYNC) cp_async_wait_all();
    drain<true, R>(FlatSource<SOA, R, T, BS_HYB>{a, slot}, Q, tl, true, (uint32_t)FLAG_FALLBACK);
    tl.flush<true, BS_HYB / 32>(a.stats, a.hist, a.hist_host);  // (the history: pairs and fallbacks)
}


// ---- warp-specialised hybrid (the fast fp64 hybrid) ----------------------------------
// One CTA per SM.  WS_IW iterative warps stream their own 32-pair warp tiles
// like iterative_kernel (no CTA barrier) and hand each open pair -- its index
// AND its 18 coordinates, copied from the warp's stash -- to a shared-memory
// ring; WS_FWG fallback warpgroups take batches of 128 from the ring and run
// the degenerate screen and phase 1 on the ring slots in place, then move the
// non-intersecting pairs (with their coordinates) to the warpgroup's phase-2
// stack.  No queued pair is re-read from global memory, and the sweeps never
// wait at a CTA barrier for the fallback.
// TC_HYBRID_WS: 1 = this kernel for the fast hybrids, 0 = the fused kernel
// everywhere.  fp64: 12 iterative warps + 1 fallback warpgroup at 128
// registers (cfg1 2.245 -> 2.081 ms; 10 + 4 and 8 + 8 measured slower);
// fp32 (80 registers): 16 + 8 warps (1.375 -> 1.290 ms; 12 + 8 1.390, 18 + 8
// 1.325, 16 + 12 1.312).  Strict builds keep the fused kernel (with this one:
// fp64 +3.3 %, fp32 +8.3 %; TC_WS_STRICT).
// Template flags: FULL (every result column requested, no ids: no per-column
// null tests), SELF (iterative warps serve their own open pairs when the ring
// is nearly full: TC_WS_SELF, ws_self_serve).  Which of {this kernel, its SELF
// instance, the fused kernel} a fast hybrid launch gets follows the device's
// FallbackHistory (launch3); all three give the same bits.
#ifndef TC_HYBRID_WS
#define TC_HYBRID_WS 1
#endif
#ifndef TC_WS_IW_F64
#define TC_WS_IW_F64 12
#endif
#ifndef TC_WS_IW_F32
#define TC_WS_IW_F32 16
#endif
#ifndef TC_WS_FWG_F64
#define TC_WS_FWG_F64 1
#endif
#ifndef TC_WS_FWG_F32
#define TC_WS_FWG_F32 2
#endif
#ifndef TC_WS_STRICT
#define TC_WS_STRICT 0
#endif
#ifndef TC_WS_RING
#define TC_WS_RING 512
#endif
// TC_WS_ASYNC: each iterative warp double-buffers its 32-pair stash and pulls
// its next tile into the spare buffer with 16-byte cp.async.cg copies (no
// registers, L1 bypassed) while the current tile computes.
#ifndef TC_WS_IT_REGS
#define TC_WS_IT_REGS 0
#endif
#ifndef TC_WS_FB_REGS
#define TC_WS_FB_REGS 0
#endif
#ifndef TC_WS_ASYNC
#define TC_WS_ASYNC 0
#endif
#ifndef TC_WS_Q2
#define TC_WS_Q2 256
#endif
constexpr int WS_RING = TC_WS_RING;  // ring slots (256: 2.347 ms -- producers wait; 512-768: 2.08)
#ifndef TC_WS_FB
#define TC_WS_FB 128
#endif
constexpr int WS_FB = TC_WS_FB;      // threads of one fallback warpgroup (= one batch)
constexpr int WS_Q2 = TC_WS_Q2 < 2 * WS_FB ? TC_WS_Q2 : 2 * WS_FB;      // phase-2 stack entries per warpgroup (< 2 WS_FB: phase-1 batches shrink to fit)
// TC_WS_ASYNC_LANE_F32 / _F64: the same double buffering with every lane copying its own pair
// (18 element-sized cp.async into its stash slots, any layout, alignment or tile tail; no warp
// synchronisation: a lane only ever reads its own slots).  With the paired fp32 stash the fp32
// hybrid gains 2.8 % (1.235 -> 1.200 ms, bitwise equal); fp64 does not have the shared memory for
// a second stash next to the full ring, and loses with a smaller one: on for float only.
#ifndef TC_WS_ASYNC_LANE_F32
#define TC_WS_ASYNC_LANE_F32 1
#endif
#ifndef TC_WS_ASYNC_LANE_F64
#define TC_WS_ASYNC_LANE_F64 0
#endif
template <typename T>
__host__ __device__ constexpr bool ws_async_lane() { return sizeof(T) == 8 ? TC_WS_ASYNC_LANE_F64 : TC_WS_ASYNC_LANE_F32; }
template <typename T>
__host__ __device__ constexpr int ws_nbuf() { return (TC_WS_ASYNC || ws_async_lane<T>()) ? 2 : 1; }  // stash buffers per iterative warp
static_assert(WS_Q2 >= WS_FB + 32 && WS_Q2 <= 2 * WS_FB, "phase-2 stack size");

constexpr int64_t WS_FREE = -1;
struct WsGroup {
    int64_t q2[WS_Q2];  // pair index (| IDS_ONLY) of each phase-2 stack entry
    int n2, m, pos;
};
template <int FWG>
struct WsShared {
    int64_t ring[WS_RING];  // pair index of each ring slot (one consumer group: WS_FREE = free)
    // Slot sequence numbers (bounded multi-producer / multi-consumer queue; used with FWG > 1):
    // slot q starts at q; the producer holding position p waits for seq == p,
    // fills the slot and sets p + 1; the consumer holding p waits for p + 1,
    // reads and sets p + WS_RING (free for the next lap).  With two fallback
    // warpgroups a claim a whole lap ahead of the other group's unfinished
    // batch can therefore never take the previous lap's entry for its own.
    int seq[WS_RING];
    WsGroup g[FWG];
    int tail, head, done;
    unsigned ring_waits, self_tiles;  // polls of producers on a full ring; tiles served by their own warp
};
// TC_WS_SELF: when the ring is nearly full (the fallback warps are behind: a
// batch with many open pairs, e.g. BASELINE config 3's near-parallel class at
// 84 % fallbacks), an iterative warp runs the comparison phases for its own
// tile's open pairs, straight from its stash, instead of sleeping on a full
// ring -- the static 12 + 4 split of the warps then degrades towards the fused
// kernel's behaviour instead of towards four warps' throughput.
// TC_WS_SELF_MARGIN: serve locally when fewer than this many ring positions are unclaimed.
// TC_WS_SELF: 0 never, 1 chosen per launch from the device's fallback history, 2 always.
#ifndef TC_WS_SELF
#define TC_WS_SELF 1
#endif
#ifndef TC_WS_SELF_MARGIN
#define TC_WS_SELF_MARGIN 192
#endif
// dynamic shared memory (T elements): [ring coordinates 18 x WS_RING]
// [per warpgroup: phase-2 coordinates 18 x WS_Q2, crossing scratch SCR x WS_FB]
// [iterative stash 18 x 32 IW]
template <typename T, int IW, int FWG>
constexpr size_t ws_smem_bytes(bool self) {
    return sizeof(T) * (18 * WS_RING + FWG * (18 * WS_Q2 + SCR * WS_FB) + ws_nbuf<T>() * 18 * 32 * IW +
                        (self ? SCR * 32 * IW : 0));
}
// Producer / consumer ordering inside the CTA.  TC_WS_FENCE 1: fence.acq_rel.cta
// instead of __threadfence_block() (fence.sc.cta, MEMBAR.SC): release /
// acquire around the slot words is all the hand-over needs.
// The iterative warps' stash as two-value words (16-byte stash stores,
// epilogue re-reads and ring copies): fp32 hybrid -2.7 %, fp64 +1 % (the fp64
// kernel is bound by its FP64 chains, not by issue slots): on for float only.
#ifndef TC_WS_PAIRED_F64
#define TC_WS_PAIRED_F64 0
#endif
#ifndef TC_WS_PAIRED_F32
#define TC_WS_PAIRED_F32 1
#endif
// Full-record kernel instance without per-column null tests (fp32 -2.1 %, fp64 +-0)
#ifndef TC_WS_FULL
#define TC_WS_FULL 1
#endif
#ifndef TC_WS_FENCE
#define TC_WS_FENCE 0
#endif
__device__ __forceinline__ void ws_fence() {
#if TC_WS_FENCE
    asm volatile("fence.acq_rel.cta;" ::: "memory");
#else
    __threadfence_block();
#endif
}
// named barrier of fallback warpgroup g (ids 1..FWG; 0 is __syncthreads)
__device__ __forceinline__ void fb_sync(int g) { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(WS_FB) : "memory"); }

// TC_WS_SELF cold path: the degenerate screen and both comparison phases for
// one open pair read from an iterative warp's stash (planar [18][32] or paired
// words), results stored like the fallback warpgroup's; returns the tally
// contributions (1 degenerate, 2 compared, 4 contact, 8 intersecting) and the distance.
struct ServeOut {
    unsigned flags;
    double dist;
};
template <typename T, bool STRICT, bool SOA, bool FULL, bool PAIRED>
__device__ __noinline__ ServeOut ws_self_serve(const Args<T>* ap, int64_t i, const T* stash, T* scr_p) {
    using R = typename Pol<T, STRICT>::R;
    const Args<T>& a = *ap;
    Scratch<R> scr;
    scr.p = scr_p;
    scr.stride = 32;
    const FlatSource<SOA, R, T, 32, FULL> src{a, nullptr};  // (stores only)
    const R eps = R(a.eps ? a.eps[i] : a.eps_scalar);
    ServeOut out{0u, 0.0};
    auto serve = [&](const auto& TA, const auto& TB) {
        Rec<R> r;
        if (degenerate_tri_t<R>(TA) || degenerate_tri_t<R>(TB)) {
            src.mark_degenerate(i);
            out.flags = 1u;
            return;
        }
        if (comparison_phase1(TA, TB, eps, scr, r)) {
            r.ids |= (uint32_t)FLAG_FALLBACK << 24;
            src.store(i, r);
            if (!FULL && a.ids != nullptr) {
                Rec<R> r2;
                comparison_phase2(TA, TB, eps, true, r2, scr);
                src.store_ids01(i, r2.ids);
            }
        } else {
            comparison_phase2(TA, TB, eps, false, r, scr);
            r.ids |= (uint32_t)FLAG_FALLBACK << 24;
            src.store(i, r);
        }
        out.flags = 2u | (r.kind == KIND_CONTACT ? 4u : 0u) | (((r.ids >> 24) & FLAG_INTERSECT) ? 8u : 0u);
        out.dist = (double)val(r.distance);
    };
    if constexpr (PAIRED) {
        using T2 = typename Vec2<T>::type;
        const T2* s2 = reinterpret_cast<const T2*>(stash);
        serve(PairTri<R>{s2, 0}, PairTri<R>{s2, 9});
    } else {
        serve(SmemTri<R>{stash, 32}, SmemTri<R>{stash + 9 * 32, 32});
    }
    return out;
}

template <typename T, bool STRICT, bool SOA, int WS_IW, int WS_FWG, bool FULL, bool SELF>
__global__ void __launch_bounds__(32 * WS_IW + WS_FWG * WS_FB, 1) hybrid_ws_kernel(const __grid_constant__ Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    constexpr bool PAIRED = sizeof(T) == 8 ? TC_WS_PAIRED_F64 : TC_WS_PAIRED_F32;
    static_assert(!(TC_WS_ASYNC && PAIRED), "the 16-byte cp.async tiles land in planar layout");
    constexpr bool LANE_ASYNC = ws_async_lane<T>() && !TC_WS_ASYNC;
    constexpr int WS_NBUF = ws_nbuf<T>();
    constexpr int WS_IT = 32 * WS_IW;  // iterative threads
    constexpr int WS_BS = WS_IT + WS_FWG * WS_FB;
    __shared__ WsShared<WS_FWG> S;
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    T* const ringd = reinterpret_cast<T*>(tc_dyn_smem);
    Tally tl;
    constexpr bool SEQ = WS_FWG > 1;  // several consumers: sequence-numbered slots (WsShared)
    for (int k = threadIdx.x; k < WS_RING; k += WS_BS) {
        S.seq[k] = k;
        S.ring[k] = WS_FREE;
    }
    if (threadIdx.x == 0) {
        S.tail = S.head = S.done = 0;
        S.ring_waits = S.self_tiles = 0;
        for (int g = 0; g < WS_FWG; ++g) S.g[g].n2 = S.g[g].m = S.g[g].pos = 0;
    }
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid < WS_IW) {
        // ---- iterative warps ----
        if constexpr (TC_WS_FB_REGS > 0 && TC_WS_IT_REGS > 0 && sizeof(T) == 8)
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TC_WS_IT_REGS));
        const KP<R> kp = make_kp<R>(a);
        // the warp's stash: WS_NBUF buffers of [18][32] values
        T* const wstash = ringd + 18 * WS_RING + WS_FWG * (18 * WS_Q2 + SCR * WS_FB) + wid * (WS_NBUF * 18 * 32);
        const int64_t nwt = (a.n + 31) / 32;
        const int64_t wstep = (int64_t)gridDim.x * WS_IW;
        // 16-byte copies need every SoA plane row 16-byte aligned
        constexpr int CH = 16 / (int)sizeof(T);  // values per copy
        const bool can_async = TC_WS_ASYNC && SOA && a.n % CH == 0 &&
                               ((reinterpret_cast<uintptr_t>(a.tri_a) | reinterpret_cast<uintptr_t>(a.tri_b)) & 15) == 0;
        auto pre = [&](int64_t wt) { return can_async && wt < nwt && (wt + 1) * 32 <= a.n; };  // full tiles only
        auto issue = [&](int64_t wt, T* buf) {
            constexpr int LPP = 32 / CH;   // lanes per plane row
            constexpr int PPI = 32 / LPP;  // plane rows per instruction
            const int pl = lane / LPP, off = (lane % LPP) * CH;
#pragma unroll
            for (int j = 0; j < (18 + PPI - 1) / PPI; ++j) {
                const int k = j * PPI + pl;
                if (k < 18) {
                    const T* src = (k < 9 ? a.tri_a + (int64_t)k * a.n : a.tri_b + (int64_t)(k - 9) * a.n) + wt * 32 + off;
                    const unsigned d = (unsigned)__cvta_generic_to_shared(buf + k * 32 + off);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        // LANE_ASYNC: lane-wise copy of pair wt * 32 + lane into the lane's slots of `buf`
        auto issue_lane = [&](int64_t wt, T* buf) {
            const int64_t j = wt * 32 + lane;
            if (wt < nwt && j < a.n) {
#pragma unroll
                for (int c = 0; c < 18; ++c) {
                    const T* src = SOA ? (c < 9 ? a.tri_a + (int64_t)c * a.n : a.tri_b + (int64_t)(c - 9) * a.n) + j
                                       : (c < 9 ? a.tri_a + 9 * j + c : a.tri_b + 9 * j + (c - 9));
                    // coordinate c of this lane: planar slot[c * 32], paired word (c >> 1) * 32, half c & 1
                    T* dst = PAIRED ? buf + ((c >> 1) * 32 + lane) * 2 + (c & 1) : buf + c * 32 + lane;
                    cp_async_val(dst, src);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        int cur = 0;
        const int64_t wt0 = (int64_t)blockIdx.x * WS_IW + wid;
        if (LANE_ASYNC) issue_lane(wt0, wstash);
        else if (pre(wt0)) issue(wt0, wstash);
        for (int64_t wt = wt0; wt < nwt; wt += wstep) {
            const int64_t i = wt * 32 + lane;
            T* const slot = wstash + cur * (18 * 32) + lane;
            // TC_WS_PAIRED: the same buffer as 9 x 32 two-value words (coordinates 2kk, 2kk + 1 of lane l at
            // word kk * 32 + l): the stash, the epilogue's re-read and the ring copy move 16 bytes at a time
            using T2 = typename Vec2<T>::type;
            T2* const slot2 = reinterpret_cast<T2*>(wstash + cur * (18 * 32)) + lane;
            const bool staged = LANE_ASYNC || pre(wt);
            if (LANE_ASYNC) {
                cp_async_wait_all();  // (a lane reads only the slots it copied itself: no warp barrier)
                cur ^= 1;
                issue_lane(wt + wstep, wstash + cur * (18 * 32));
            } else if (TC_WS_ASYNC) {
                if (staged) cp_async_wait_all();
                __syncwarp();  // the tile is visible to every lane; the previous tile's reads of the spare buffer are done
                cur ^= 1;
                if (pre(wt + wstep)) issue(wt + wstep, wstash + cur * (18 * 32));
            }
            bool enq = false;
            if (i < a.n) {
                R A[9], B[9], eps;
                if (staged && PAIRED) {
#pragma unroll
                    for (int kk = 0; kk < 9; ++kk) {
                        const T2 v = slot2[kk * 32];
                        const int c = 2 * kk;
                        (c < 9 ? A[c] : B[c - 9]) = R(v.x);
                        (c + 1 < 9 ? A[c + 1] : B[c + 1 - 9]) = R(v.y);
                    }
                } else if (staged) {
#pragma unroll
                    for (int k = 0; k < 9; ++k) {
                        A[k] = R(slot[k * 32]);
                        B[k] = R(slot[(9 + k) * 32]);
                    }
                } else {
                    load_pair<SOA>(a, i, A, B, eps);
                    if (PAIRED) stash_pair2(slot2, A, B);
                    else stash_pair<32>(slot, A, B);
                }
                Rec<R> r;
                if (PAIRED)
                    run_iterative(PairTri<R>{slot2, 0}, PairTri<R>{slot2, 9}, A, B,
                                  [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
                else
                    run_iterative<32>(slot, A, B, [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
                tl.iterative++;
                enq = r.kind == KIND_NOT_TERMINATED && (a.allow == nullptr || a.allow[i]);
                // open pairs: a placeholder the fallback overwrites
                if constexpr (FULL) store_rec_full<SOA, FULL>(a, i, r);
                else store_rec<SOA>(a, i, r);
                if (!enq) tl.result(r);
            }
            const unsigned m = __ballot_sync(0xffffffffu, enq);
            bool self = false;
            if (SELF && m) {
                int occ = 0;
                if (lane == 0) occ = *(volatile int*)&S.tail - *(volatile int*)&S.head;
                self = __shfl_sync(0xffffffffu, occ, 0) > WS_RING - TC_WS_SELF_MARGIN;
            }
            if (self) {
                if (lane == 0) atomicAdd(&S.self_tiles, 1u);
                if (enq) {
                    // the comparison phases for this lane's open pair, read from the warp's stash
                    // (a separate function: the cold path stays out of the sweep's register allocation)
                    T* const scr_p = ringd + 18 * WS_RING + WS_FWG * (18 * WS_Q2 + SCR * WS_FB) +
                                     WS_NBUF * 18 * 32 * WS_IW + wid * (SCR * 32) + lane;  // (allocated with SELF)
#ifndef TC_X_SELF_NOCALL  // timing-only
#define TC_X_SELF_NOCALL 0
#endif
                    const ServeOut so = TC_X_SELF_NOCALL ? ServeOut{0u, (double)(scr_p - slot)} :
                        ws_self_serve<T, STRICT, SOA, FULL, PAIRED>(
                        &a, i, PAIRED ? reinterpret_cast<const T*>(slot2) : slot, scr_p);
                    tl.degenerate += so.flags & 1u;
                    if (so.flags & 2u) {
                        tl.comparison++;
                        tl.contacts += (so.flags >> 2) & 1u;
                        tl.intersecting += (so.flags >> 3) & 1u;
                        const double d = so.dist + 0.0;
                        tl.min_d = (d < tl.min_d) ? d : tl.min_d;
                    }
                }
                __syncwarp();
            } else if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&S.tail, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (enq) {
                    const int pos = base + __popc(m & ((1u << lane) - 1u));
                    const int q = (unsigned)pos % (unsigned)WS_RING;
                    volatile int* sq = &S.seq[q];
                    volatile int64_t* idx = &S.ring[q];
                    // ring full: the fallback frees slots
                    unsigned polls = 0;
                    if (SEQ) while (*sq != pos) { __nanosleep(64); ++polls; }
                    else while (*idx != WS_FREE) { __nanosleep(64); ++polls; }
                    if (polls) atomicAdd(&S.ring_waits, polls);  // (rare: the fallback-history signal)
                    ws_fence();  // the slot's previous reader is done before we overwrite it
                    if (PAIRED) {
#pragma unroll
                        for (int kk = 0; kk < 9; ++kk) {
                            const auto v = slot2[kk * 32];
                            ringd[(2 * kk) * WS_RING + q] = v.x;
                            ringd[(2 * kk + 1) * WS_RING + q] = v.y;
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 18; ++k) ringd[k * WS_RING + q] = slot[k * 32];
                    }
                    if (SEQ) *idx = i;
                    // the slot and the placeholder row before the sequence number / index
                    ws_fence();
                    if (SEQ) *sq = pos + 1;
                    else *idx = i;
                }
            }
        }
        ws_fence();
        __syncwarp();
        if (lane == 0) atomicAdd(&S.done, 1);
    } else {
        // ---- fallback warpgroups ----
        // TC_WS_FB_REGS: the launch allocates 65536 / threads registers per
        // thread (96 at 640 threads); the fallback warpgroups take the spare
        // ones (setmaxnreg needs warpgroup-aligned roles: WS_IW % 4 == 0)
        if constexpr (TC_WS_FB_REGS > 0 && sizeof(T) == 8) {
            static_assert(WS_IW % 4 == 0, "setmaxnreg is per warpgroup");
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TC_WS_FB_REGS));
        }
        const int gi = (threadIdx.x - WS_IT) / WS_FB, ft = (threadIdx.x - WS_IT) % WS_FB;
        WsGroup& G = S.g[gi];
        T* const q2d = ringd + 18 * WS_RING + gi * (18 * WS_Q2 + SCR * WS_FB);
        Scratch<R> scr;
        scr.p = q2d + 18 * WS_Q2 + ft;
        scr.stride = WS_FB;
        const bool want_ids = !FULL && a.ids != nullptr;
        const FlatSource<SOA, R, T, WS_FB, FULL> src{a, nullptr};  // (stores only)
        auto phase2_batches = [&](bool final_) {
            while (true) {
                const int c2 = *(volatile int*)&G.n2;
                fb_sync(gi);  // everyone has read the count before it changes
                if (!(c2 >= WS_FB || (final_ && c2 > 0))) break;
                const int m2 = c2 < WS_FB ? c2 : WS_FB;
                const int sl = c2 - m2 + ft;
                const int64_t e = ft < m2 ? G.q2[sl] : -1;
                fb_sync(gi);
                if (ft == 0) G.n2 = c2 - m2;
                if (e >= 0) {
                    const int64_t j = e & (IDS_ONLY - 1);
                    const SmemTri<R> A{q2d + sl, WS_Q2}, B{q2d + 9 * WS_Q2 + sl, WS_Q2};
                    const R eps = R(a.eps ? a.eps[j] : a.eps_scalar);
                    Rec<R> r;
                    const bool ids_only = (e & IDS_ONLY) != 0;
                    comparison_phase2(A, B, eps, ids_only, r, scr);
                    if (ids_only) {
                        src.store_ids01(j, r.ids);
                    } else {
                        r.ids |= (uint32_t)FLAG_FALLBACK << 24;
                        src.store(j, r);
                        tl.result(r);
                    }
                }
                fb_sync(gi);  // the stack slots are free again
            }
        };
        while (true) {
            if (ft == 0) {
                // claim a batch of ring positions [h, h + m) for this warpgroup
                int m = 0, h = 0;
                while (true) {
                    const int d = *(volatile int*)&S.done;
                    ws_fence();
                    h = *(volatile int*)&S.head;
                    const int avail = *(volatile int*)&S.tail - h;
                    // a batch must fit the phase-2 stack (n2 < WS_FB here)
                    const int want = WS_Q2 < 2 * WS_FB ? min(WS_FB, WS_Q2 - *(volatile int*)&G.n2) : WS_FB;
                    m = avail >= want ? want : (d == WS_IW ? avail : 0);
                    if (m > 0) {
                        if (atomicCAS(&S.head, h, h + m) == h) break;
                        continue;
                    }
                    if (d == WS_IW) break;  // all produced and claimed
                    __nanosleep(256);
#ifdef TC_X_COUNT_FB_IDLE  // experiment: the leader's idle polls in place of the self-served tiles
                    atomicAdd(&S.self_tiles, 1u);
#endif
                }
                G.m = m;
                G.pos = h;
            }
            fb_sync(gi);
            const int m = *(volatile int*)&G.m, pos = *(volatile int*)&G.pos;
            if (m == 0) break;
            const int q = (unsigned)(pos + ft) % (unsigned)WS_RING;
            int64_t j = -1;
            if (ft < m) {
                volatile int* sq = &S.seq[q];
                volatile int64_t* idx = &S.ring[q];
                // claimed by a producer, not yet written
                if (SEQ) while (*sq != pos + ft + 1) __nanosleep(32);
                else while ((j = *idx) == WS_FREE) __nanosleep(32);
                ws_fence();
                if (SEQ) j = *idx;
            }
            bool push2 = false;
            int64_t e2 = 0;
            if (j >= 0) {
                const SmemTri<R> A{ringd + q, WS_RING}, B{ringd + 9 * WS_RING + q, WS_RING};
                const R eps = R(a.eps ? a.eps[j] : a.eps_scalar);
                Rec<R> r;
                // RK/kernels.py:596-600: a degenerate open pair keeps its
                // iterative result and is marked DEGENERATE
                if (degenerate_tri_t<R>(A) || degenerate_tri_t<R>(B)) {
                    src.mark_degenerate(j);
                    tl.degenerate++;
                } else {
                    tl.comparison++;
                    if (comparison_phase1(A, B, eps, scr, r)) {
                        r.ids |= (uint32_t)FLAG_FALLBACK << 24;
                        src.store(j, r);
                        tl.result(r);
                        push2 = want_ids;
                        e2 = j | IDS_ONLY;
                    } else {
                        push2 = true;
                        e2 = j;
                    }
                }
            }
            // move phase-2 pairs (index and coordinates) to the stack, then free the ring slots
            {
                const unsigned mm = __ballot_sync(0xffffffffu, push2);
                int base = 0;
                if (mm) {
                    if ((ft & 31) == 0) base = atomicAdd(&G.n2, __popc(mm));
                    base = __shfl_sync(0xffffffffu, base, 0);
                }
                if (push2) {
                    const int sl = base + __popc(mm & ((1u << (ft & 31)) - 1u));
                    TC_CHECK(sl < WS_Q2);
                    G.q2[sl] = e2;
#pragma unroll
                    for (int k = 0; k < 18; ++k) q2d[k * WS_Q2 + sl] = ringd[k * WS_RING + q];
                }
            }
            // every read of the ring slot (phase 1, the copy) before it is freed
            ws_fence();
            if (ft < m) {  // free for the next lap
                if (SEQ) *(volatile int*)&S.seq[q] = pos + ft + WS_RING;
                else *(volatile int64_t*)&S.ring[q] = WS_FREE;
            }
            fb_sync(gi);  // q2 entries visible, G.m / G.pos read by everyone
            phase2_batches(false);
        }
        phase2_batches(true);
    }
    if (TC_DEBUG) {  // every pushed pair was claimed, both phase-2 stacks are empty
        __syncthreads();
        if (threadIdx.x == 0) {
            TC_CHECK(S.head == S.tail && S.done == WS_IW);
            for (int g = 0; g < WS_FWG; ++g) TC_CHECK(S.g[g].n2 == 0);
        }
    }
    __syncthreads();  // the history counters are final
    tl.flush<true, WS_BS / 32>(a.stats, a.hist, a.hist_host, S.ring_waits, S.self_tiles);
}

// ---- hybrid for batches with few fallbacks (TC_WQ) ---------------------------------------
// All 16 warps of the one CTA per SM iterate (lane-wise cp.async prefetch of the
// next tile into a second stash buffer, as in hybrid_ws_kernel); a warp keeps the
// indices of its open pairs in a private 64-entry queue and, once 32 have
// gathered, serves them itself: every lane re-reads one queued pair from global
// memory (L2) into its free stash slot and runs ws_self_serve on it.  No warp
// waits for another, nobody idles while fallbacks are rare -- the regime the
// fallback history sends here (under TC_WS_FUSED_BELOW fallbacks per pair).
// At cfg1's 41 % the gathers and the divergence of warp-private batches lose
// (round 1 measured -10 % for warp-private queues); results are the same bits.
#ifndef TC_WQ
#define TC_WQ 1
#endif
constexpr int WQ_WARPS = 16;
constexpr int WQ_CAP = 64;
template <typename T>
constexpr size_t wq_smem_bytes() {
    return sizeof(T) * (2 * 18 * 32 * WQ_WARPS + SCR * 32 * WQ_WARPS);
}
template <typename T, bool STRICT, bool SOA, bool FULL>
__global__ void __launch_bounds__(32 * WQ_WARPS, 1) hybrid_wq_kernel(const __grid_constant__ Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    __shared__ int64_t queue[WQ_WARPS][WQ_CAP];
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    T* const base = reinterpret_cast<T*>(tc_dyn_smem);
    Tally tl;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const KP<R> kp = make_kp<R>(a);
    T* const wstash = base + wid * (2 * 18 * 32);
    T* const scr_p = base + 2 * 18 * 32 * WQ_WARPS + wid * (SCR * 32) + lane;
    int64_t* const q = queue[wid];
    int nq = 0;  // queued open pairs of this warp (warp-uniform)
    const int64_t nwt = (a.n + 31) / 32;
    const int64_t wstep = (int64_t)gridDim.x * WQ_WARPS;
    auto issue_lane = [&](int64_t wt, T* buf) {
        const int64_t j = wt * 32 + lane;
        if (wt < nwt && j < a.n) {
#pragma unroll
            for (int c = 0; c < 18; ++c) {
                const T* src = SOA ? (c < 9 ? a.tri_a + (int64_t)c * a.n : a.tri_b + (int64_t)(c - 9) * a.n) + j
                                   : (c < 9 ? a.tri_a + 9 * j + c : a.tri_b + 9 * j + (c - 9));
                cp_async_val(buf + c * 32 + lane, src);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // the comparison phases for up to 32 queued pairs, one per lane, staged in `slot`
    auto serve = [&](int cnt, T* slot) {
        const int64_t j = lane < cnt ? q[nq - cnt + lane] : -1;
        nq -= cnt;
        if (j >= 0) {
#pragma unroll
            for (int c = 0; c < 18; ++c)
                slot[c * 32] = __ldg(SOA ? (c < 9 ? a.tri_a + (int64_t)c * a.n : a.tri_b + (int64_t)(c - 9) * a.n) + j
                                         : (c < 9 ? a.tri_a + 9 * j + c : a.tri_b + 9 * j + (c - 9)));
            const ServeOut so = ws_self_serve<T, STRICT, SOA, FULL, false>(&a, j, slot, scr_p);
            tl.degenerate += so.flags & 1u;
            if (so.flags & 2u) {
                tl.comparison++;
                tl.contacts += (so.flags >> 2) & 1u;
                tl.intersecting += (so.flags >> 3) & 1u;
                const double d = so.dist + 0.0;
                tl.min_d = (d < tl.min_d) ? d : tl.min_d;
            }
        }
        __syncwarp();
    };
    int cur = 0;
    const int64_t wt0 = (int64_t)blockIdx.x * WQ_WARPS + wid;
    issue_lane(wt0, wstash);
    for (int64_t wt = wt0; wt < nwt; wt += wstep) {
        const int64_t i = wt * 32 + lane;
        T* const slot = wstash + cur * (18 * 32) + lane;
        cp_async_wait_all();  // (a lane reads only the slots it copied itself)
        cur ^= 1;
        issue_lane(wt + wstep, wstash + cur * (18 * 32));
        bool enq = false;
        if (i < a.n) {
            R A[9], B[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                A[k] = R(slot[k * 32]);
                B[k] = R(slot[(9 + k) * 32]);
            }
            Rec<R> r;
            run_iterative<32>(slot, A, B, [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
            tl.iterative++;
            enq = r.kind == KIND_NOT_TERMINATED && (a.allow == nullptr || a.allow[i]);
            // open pairs: a placeholder the warp overwrites when it serves its queue
            if constexpr (FULL) store_rec_full<SOA, FULL>(a, i, r);
            else store_rec<SOA>(a, i, r);
            if (!enq) tl.result(r);
        }
        const unsigned m = __ballot_sync(0xffffffffu, enq);
        if (m) {
            if (enq) q[nq + __popc(m & ((1u << lane) - 1u))] = i;
            nq += __popc(m);
            __syncwarp();  // the queue entries and the placeholder rows before any lane serves them
            if (nq >= 32) serve(32, slot);  // (the tile's slot is free now; nq < 32 before the push: nq <= 63)
        }
    }
    cp_async_wait_all();
    if (nq > 0) serve(nq, wstash + lane);
    tl.flush<true, WQ_WARPS>(a.stats, a.hist, a.hist_host);
}

// ---- warp-specialised hybrid, warp-granular fallback (TC_WSW) ---------------------------
// The same ring hand-over as hybrid_ws_kernel, but every fallback warp works
// on its own: it claims 32 ring slots at a time, runs the degenerate screen
// and phase 1 on them in place, moves the non-intersecting pairs to its own
// 64-entry phase-2 stack and runs phase-2 batches of 32 -- no named barriers,
// no shared batch state, and any number of fallback warps (WSW_FW), so the
// CTA need not be 16 warps: the ncu line counts of the 12 + 4 kernel showed
// its iterative warps asleep on a full ring ~17 x 64 ns per tile, i.e. four
// fallback warps (one per SM sub-partition, latency-bound at one instruction
// per ~7 cycles) set the pace.
#ifndef TC_WSW
#define TC_WSW 0
#endif
#ifndef TC_WSW_IW
#define TC_WSW_IW 12
#endif
#ifndef TC_WSW_FW
#define TC_WSW_FW 6
#endif
constexpr int WSW_Q2 = 64;  // phase-2 stack entries per fallback warp
template <typename T, int IW, int FW>
constexpr size_t wsw_smem_bytes() {
    return sizeof(T) * (18 * WS_RING + FW * (18 * WSW_Q2 + SCR * 32) + 18 * 32 * IW);
}
template <int FW>
struct WswShared {
    int64_t ring[WS_RING];  // pair index of each ring slot
    // Slot sequence numbers (bounded multi-producer / multi-consumer queue):
    // slot q starts at q; the producer holding position p waits for
    // seq == p, fills the slot and sets p + 1; the consumer holding p waits for
    // p + 1, reads and sets p + WS_RING (free for the next lap).  Several
    // consumers can therefore hold claims a lap apart without mistaking the
    // previous lap's entry for theirs.
    int seq[WS_RING];
    int64_t q2[FW][WSW_Q2];
    int tail, head, done;
};

template <typename T, bool STRICT, bool SOA, int IW, int FW>
__global__ void __launch_bounds__(32 * (IW + FW), 1) hybrid_wsw_kernel(Args<T> a) {
    using R = typename Pol<T, STRICT>::R;
    constexpr int NT = 32 * (IW + FW);
    __shared__ WswShared<FW> S;
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    T* const ringd = reinterpret_cast<T*>(tc_dyn_smem);
    Tally tl;
    for (int k = threadIdx.x; k < WS_RING; k += NT) S.seq[k] = k;
    if (threadIdx.x == 0) S.tail = S.head = S.done = 0;
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (wid < IW) {
        // ---- iterative warps (as in hybrid_ws_kernel) ----
        const KP<R> kp = make_kp<R>(a);
        T* const slot = ringd + 18 * WS_RING + FW * (18 * WSW_Q2 + SCR * 32) + wid * (18 * 32) + lane;
        const int64_t nwt = (a.n + 31) / 32;
        for (int64_t wt = (int64_t)blockIdx.x * IW + wid; wt < nwt; wt += (int64_t)gridDim.x * IW) {
            const int64_t i = wt * 32 + lane;
            bool enq = false;
            if (i < a.n) {
                R A[9], B[9], eps;
                load_pair<SOA>(a, i, A, B, eps);
                stash_pair<32>(slot, A, B);
                Rec<R> r;
                run_iterative<32>(slot, A, B, [&] { return R(a.eps ? a.eps[i] : a.eps_scalar); }, kp, r);
                tl.iterative++;
                enq = r.kind == KIND_NOT_TERMINATED && (a.allow == nullptr || a.allow[i]);
                store_rec<SOA>(a, i, r);  // open pairs: a placeholder the fallback overwrites
                if (!enq) tl.result(r);
            }
            const unsigned m = __ballot_sync(0xffffffffu, enq);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&S.tail, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (enq) {
                    const int pos = base + __popc(m & ((1u << lane) - 1u));
                    const int q = (unsigned)pos % (unsigned)WS_RING;
                    volatile int* sq = &S.seq[q];
                    while (*sq != pos) __nanosleep(64);  // ring full: the fallback frees slots
                    __threadfence_block();  // the slot's previous reader is done before we overwrite it
#pragma unroll
                    for (int k = 0; k < 18; ++k) ringd[k * WS_RING + q] = slot[k * 32];
                    S.ring[q] = i;
                    __threadfence_block();  // the slot and the placeholder row before the sequence number
                    *sq = pos + 1;
                }
            }
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) atomicAdd(&S.done, 1);
    } else {
        // ---- fallback warps ----
        const int fw = wid - IW;
        T* const q2d = ringd + 18 * WS_RING + fw * (18 * WSW_Q2 + SCR * 32);
        int64_t* const q2i = S.q2[fw];
        Scratch<R> scr;
        scr.p = q2d + 18 * WSW_Q2 + lane;
        scr.stride = 32;
        const bool want_ids = a.ids != nullptr;
        const FlatSource<SOA, R, T, 32> src{a, nullptr};  // (stores only)
        int n2 = 0;  // entries on this warp's phase-2 stack (warp-uniform)
        auto phase2_batches = [&](bool final_) {
            while (n2 >= 32 || (final_ && n2 > 0)) {
                const int m2 = n2 < 32 ? n2 : 32;
                const int sl = n2 - m2 + lane;
                n2 -= m2;
                if (lane < m2) {
                    const int64_t e = q2i[sl];
                    const int64_t j = e & (IDS_ONLY - 1);
                    const SmemTri<R> A{q2d + sl, WSW_Q2}, B{q2d + 9 * WSW_Q2 + sl, WSW_Q2};
                    const R eps = R(a.eps ? a.eps[j] : a.eps_scalar);
                    Rec<R> r;
                    const bool ids_only = (e & IDS_ONLY) != 0;
                    comparison_phase2(A, B, eps, ids_only, r, scr);
                    if (ids_only) {
                        src.store_ids01(j, r.ids);
                    } else {
                        r.ids |= (uint32_t)FLAG_FALLBACK << 24;
                        src.store(j, r);
                        tl.result(r);
                    }
                }
                __syncwarp();  // the stack slots are free again
            }
        };
        while (true) {
            int m = 0, h = 0;
            if (lane == 0) {
                // claim ring positions [h, h + m) for this warp
                while (true) {
                    const int d = *(volatile int*)&S.done;
                    __threadfence_block();
                    h = *(volatile int*)&S.head;
                    const int avail = *(volatile int*)&S.tail - h;
                    m = avail >= 32 ? 32 : (d == IW ? avail : 0);
                    if (m > 0) {
                        if (atomicCAS(&S.head, h, h + m) == h) break;
                        continue;
                    }
                    if (d == IW) break;  // all produced and claimed
                    __nanosleep(128);
                }
            }
            m = __shfl_sync(0xffffffffu, m, 0);
            h = __shfl_sync(0xffffffffu, h, 0);
            if (m == 0) break;
            const int q = (unsigned)(h + lane) % (unsigned)WS_RING;
            int64_t j = -1;
            if (lane < m) {
                volatile int* sq = &S.seq[q];
                while (*sq != h + lane + 1) __nanosleep(32);  // claimed by a producer, not yet written
                __threadfence_block();
                j = *(volatile int64_t*)&S.ring[q];
            }
            bool push2 = false;
            int64_t e2 = 0;
            if (j >= 0) {
                const SmemTri<R> A{ringd + q, WS_RING}, B{ringd + 9 * WS_RING + q, WS_RING};
                const R eps = R(a.eps ? a.eps[j] : a.eps_scalar);
                Rec<R> r;
                // RK/kernels.py:596-600: a degenerate open pair keeps its
                // iterative result and is marked DEGENERATE
                if (degenerate_tri_t<R>(A) || degenerate_tri_t<R>(B)) {
                    src.mark_degenerate(j);
                    tl.degenerate++;
                } else {
                    tl.comparison++;
                    if (comparison_phase1(A, B, eps, scr, r)) {
                        r.ids |= (uint32_t)FLAG_FALLBACK << 24;
                        src.store(j, r);
                        tl.result(r);
                        push2 = want_ids;
                        e2 = j | IDS_ONLY;
                    } else {
                        push2 = true;
                        e2 = j;
                    }
                }
            }
            // move phase-2 pairs (index and coordinates) to the warp's stack, then free the ring slots
            const unsigned mm = __ballot_sync(0xffffffffu, push2);
            if (push2) {
                const int sl = n2 + __popc(mm & ((1u << lane) - 1u));
                TC_CHECK(sl < WSW_Q2);
                q2i[sl] = e2;
#pragma unroll
                for (int k = 0; k < 18; ++k) q2d[k * WSW_Q2 + sl] = ringd[k * WS_RING + q];
            }
            n2 += __popc(mm);
            __threadfence_block();  // every read of the ring slot (phase 1, the copy) before it is freed
            if (lane < m) *(volatile int*)&S.seq[q] = h + lane + WS_RING;
            __syncwarp();
            phase2_batches(false);
        }
        phase2_batches(true);
    }
    tl.flush<true, NT / 32>(a.stats);
}

// ---- all-pairs particle-block kernel (BASELINE.json config 2) -----------------
// One CTA per particle-pair block at a time (grid-stride over blocks): both
// meshes are staged into shared memory in planar layout (coordinate c of
// triangle t at m[c * tris + t], conflict-free for consecutive triangles),
// then all tris x tris triangle pairs run the hybrid kernel from shared
// memory -- the flat/multiscale callers' all-pairs meshgrid
// (RK/stepping.py:285-308, RK/contact.py:97-140) without materialising the
// pair list.  CONTACT pairs are compacted to a global list; every pair is
// tallied in tc_stats.

template <typename T>
struct BlockArgs {
    const T* meshes;          // [n_meshes][tris][9]: world coordinates, or local ones with motions
    const T* motions;         // [n_meshes][7] (qw, qx, qy, qz, tx, ty, tz) or NULL
    int tris;                 // staging stride (the largest mesh)
    int64_t n_meshes;
    const int32_t* mesh_tris; // [n_meshes] triangles per mesh, or NULL (all `tris`)
    const int32_t* blocks;    // [nb][2] mesh indices (A, B)
    int64_t nb;
    const T* block_eps;       // [nb] or NULL
    T eps_scalar;
    int64_t max_contacts;
    int32_t* c_idx;           // [max][3] block, tri_a, tri_b
    T* c_dist;                // [max]
    T* c_pa;                  // [max][3]
    T* c_pb;                  // [max][3]
    unsigned long long* n_contacts;
    tc_stats* stats;
    double c_factor, alpha_it, alpha_reg, move_factor, start_coord;
    int n_iterative;
};

// RK/geometry.py:162-171 rotation_matrix of the unit quaternion (w, x, y, z),
// evaluated in double like the reference's Python floats, then rounded to T.
template <class R, typename T>
__device__ __forceinline__ void motion_matrix(const T* m, R* Rm, R* tr) {
    const double w = m[0], x = m[1], y = m[2], z = m[3];
    const double v[9] = {1.0 - 2.0 * (__dadd_rn(__dmul_rn(y, y), __dmul_rn(z, z))),
                         2.0 * __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, z)),
                         2.0 * __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)),
                         2.0 * __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, z)),
                         1.0 - 2.0 * (__dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z))),
                         2.0 * __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)),
                         2.0 * __dsub_rn(__dmul_rn(x, z), __dmul_rn(w, y)),
                         2.0 * __dadd_rn(__dmul_rn(y, z), __dmul_rn(w, x)),
                         1.0 - 2.0 * (__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)))};
#pragma unroll
    for (int k = 0; k < 9; ++k) Rm[k] = R(T(v[k]));
#pragma unroll
    for (int k = 0; k < 3; ++k) tr[k] = R(m[4 + k]);
}

// world = p @ R.T + t (RK/geometry.py:173-176) rounded like the reference's
// NumPy matmul: each row the FMA chain fma(R_i2, p2, fma(R_i1, p1, R_i0 p0)),
// then the translation (oracle tco_apply_motion_*, pinned to NumPy)
template <class R>
__device__ __forceinline__ void apply_motion(const R* Rm, const R* tr, const R* p, R* w) {
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = fmav(Rm[3 * i + 2], p[2], fmav(Rm[3 * i + 1], p[1], Rm[3 * i] * p[0])) + tr[i];
}

template <class R, typename T>
struct BlockSource {
    const BlockArgs<T>& a;
    const T* mA;
    const T* mB;
    int tris;                 // staging stride
    int cols;                 // triangles of mesh B: pair p = i * cols + k
    int64_t blk;
    R eps;
    __device__ __forceinline__ bool want_ids() const { return false; }
    __device__ __forceinline__ void stage(int64_t j, SmemTri<R>& A, SmemTri<R>& B, R& e) const {
        TC_CHECK(j >= 0 && j < (int64_t)tris * cols);
        const int i = (int)(j / cols), k = (int)(j % cols);
        A.p = mA + i;
        A.stride = tris;
        B.p = mB + k;
        B.stride = tris;
        e = eps;
    }
    __device__ __forceinline__ void store(int64_t j, const Rec<R>& r) const {
        if (r.kind != KIND_CONTACT) return;
        const unsigned long long slot = atomicAdd(a.n_contacts, 1ull);
        if ((long long)slot >= a.max_contacts) return;  // counted, not stored
        a.c_idx[3 * slot] = (int32_t)blk;
        a.c_idx[3 * slot + 1] = (int32_t)(j / cols);
        a.c_idx[3 * slot + 2] = (int32_t)(j % cols);
        if (a.c_dist) a.c_dist[slot] = val(r.distance);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (a.c_pa) a.c_pa[3 * slot + c] = val(r.pa[c]);
            if (a.c_pb) a.c_pb[3 * slot + c] = val(r.pb[c]);
        }
    }
    // degenerate pairs are counted, never emitted as contacts
    __device__ __forceinline__ void mark_degenerate(int64_t) const {}
    __device__ __forceinline__ void store_ids01(int64_t, uint32_t) const {}
};

template <typename T, bool STRICT>
__global__ void __launch_bounds__(BS_BLK, TC_MINB(BS_BLK, TC_HYBRID_MINB)) blocks_hybrid_kernel(BlockArgs<T> a) {
    using R = typename Pol<T, STRICT>::R;
    __shared__ Queues<BS_BLK> Q;
    extern __shared__ __align__(16) unsigned char tc_dyn_smem[];
    T* mA = reinterpret_cast<T*>(tc_dyn_smem) + SCR * BS_BLK;  // after the crossing scratch
    const int tris = a.tris;
    T* mB = mA + 9 * tris;
    const KP<R> kp = make_kp<R>(a);
    Tally tl;
    for (int64_t blk = blockIdx.x; blk < a.nb; blk += gridDim.x) {
        __syncthreads();  // the previous block is fully drained before its meshes are replaced
        const int64_t ia = a.blocks[2 * blk], ib = a.blocks[2 * blk + 1];
        const int na = a.mesh_tris ? a.mesh_tris[ia] : tris, nbt = a.mesh_tris ? a.mesh_tris[ib] : tris;
        // a mesh against itself skips the diagonal (RK/contact.py:119-124)
        const bool self = ia == ib;
        const int64_t P = (int64_t)na * nbt;
        const int64_t ntile = (P + BS_BLK - 1) / BS_BLK;
        const T* gA = a.meshes + ia * tris * 9;
        const T* gB = a.meshes + ib * tris * 9;
        if (a.motions) {
            // rigid motion fused into the staging (RK/stepping.py:157-159,
            // 290-291: Particle.world_tris = motion.apply_points(local))
            R RA[9], tA[3], RB[9], tB[3];
            motion_matrix(a.motions + 7 * ia, RA, tA);
            motion_matrix(a.motions + 7 * ib, RB, tB);
            for (int e = threadIdx.x; e < 3 * max(na, nbt); e += BS_BLK) {
                const int t = e / 3, v = e - 3 * (e / 3);
                R pa[3], pb[3], wa[3], wb[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    pa[c] = R(t < na ? __ldg(gA + 3 * e + c) : T(0));
                    pb[c] = R(t < nbt ? __ldg(gB + 3 * e + c) : T(0));
                }
                apply_motion(RA, tA, pa, wa);
                apply_motion(RB, tB, pb, wb);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (t < na) mA[(3 * v + c) * tris + t] = val(wa[c]);
                    if (t < nbt) mB[(3 * v + c) * tris + t] = val(wb[c]);
                }
            }
        } else {
            for (int e = threadIdx.x; e < 9 * max(na, nbt); e += BS_BLK) {
                const int t = e / 9, c = e - 9 * (e / 9);
                if (t < na) mA[c * tris + t] = __ldg(gA + e);
                if (t < nbt) mB[c * tris + t] = __ldg(gB + e);
            }
        }
        if (threadIdx.x == 0) Q.n1 = Q.n2 = 0;
        __syncthreads();
        const R eps = R(a.block_eps ? a.block_eps[blk] : a.eps_scalar);
        const BlockSource<R, T> src{a, mA, mB, tris, nbt, blk, eps};
        for (int64_t tile = 0; tile < ntile; ++tile) {
            const int64_t p = tile * BS_BLK + threadIdx.x;
            bool enq = false;
            const int i = (int)(p / nbt), k = (int)(p - (int64_t)i * nbt);
            if (p < P && !(self && i == k)) {
                const SmemTri<R> SA{mA + i, tris}, SB{mB + k, tris};
                R A[9], B[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) {
                    A[c] = SA[c];
                    B[c] = SB[c];
                }
                Rec<R> r;
                run_iterative(SA, SB, A, B, [&] { return eps; }, kp, r);
                tl.iterative++;
                enq = r.kind == KIND_NOT_TERMINATED;  // screened for degeneracy in the batches
                if (!enq) {
                    src.store(p, r);
                    tl.result(r);
                }
            }
            push(Q.q1, &Q.n1, enq, p, 2 * BS_BLK);
            __syncthreads();
            drain<true, R>(src, Q, tl, false, (uint32_t)FLAG_FALLBACK);
        }
        drain<true, R>(src, Q, tl, true, (uint32_t)FLAG_FALLBACK);
    }
    tl.flush<true>(a.stats);
}

// ---- multiscale frontier traversal ---------------------------
// RK/stepping.py:311-368 multiscale_contacts on the device, for a batch of
// particle pairs at once.  Trees are concatenated FlatTree arrays (surrogate
// nodes and mesh triangles, RK/stepping.py:78-129) with global ids.  One
// round = one hybrid launch over the frontier (per-pair halo 0.5 (eps_i +
// eps_j), fallback only where both sides are mesh triangles -- the
// reference's allow_fallback=both_fine), then the frontier is unfolded: a
// pairing that is in contact or unsettled and not at mesh level on both sides
// is replaced by the meshgrid of its children (a mesh-level side stays
// itself); mesh-level contacts are appended to the contact list.

template <typename T>
struct FrontierArgs {
    const T* tris;            // [n_total][9] world coordinates, or local ones with motions
    const int32_t* owner;     // [n_total] particle of each node (with motions)
    const T* motions;         // [n_particles][7] (qw, qx, qy, qz, tx, ty, tz) or NULL
    const T* node_eps;        // [n_total]
    const uint8_t* is_fine;   // [n_total]
    const int32_t* height;    // [n_total]
    const int32_t* fa;        // frontier: id on side i
    const int32_t* fb;        // id on side j
    const int32_t* ftag;      // particle-pair index
    int64_t n;
    int8_t* kind;             // [n] final kind per pairing
    int64_t max_contacts;
    int32_t* c_idx;           // [max][3] pair, id_i, id_j
    T* c_pa;
    T* c_pb;
    unsigned long long* n_contacts;
    unsigned long long* checks;  // [max_height + 1] pairings per max(height_i, height_j)
    int max_height;
    tc_stats* stats;
    double c_factor, alpha_it, alpha_reg, move_factor, start_coord;
    int n_iterative;
};

// One tree node's triangle; with motions the owner's rigid motion is applied
// on the fly (RK/stepping.py:157-159 world_tris, rounded like apply_points).
template <class R, typename T>
__device__ __forceinline__ void load_node(const FrontierArgs<T>& a, int64_t id, R* X) {
    if (a.motions) {
        R Rm[9], tr[3];
        motion_matrix(a.motions + 7 * (int64_t)a.owner[id], Rm, tr);
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            R p[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) p[c] = R(__ldg(a.tris + 9 * id + 3 * v + c));
            apply_motion(Rm, tr, p, X + 3 * v);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) X[k] = R(__ldg(a.tris + 9 * id + k));
    }
}

template <class R, typename T>
struct FrontierSource {
    const FrontierArgs<T>& a;
    __device__ __forceinline__ bool want_ids() const { return false; }
    __device__ __forceinline__ void stage(int64_t j, SmemTri<R>& A, SmemTri<R>& B, R& eps) const {
        T* slot = thread_slot<T>(SCR * BS_FRONT);
        TC_CHECK(j >= 0 && j < a.n);
        const int64_t ia = a.fa[j], ib = a.fb[j];
        R X[9], Y[9];
        load_node(a, ia, X);
        load_node(a, ib, Y);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            slot[k * BS_FRONT] = val(X[k]);
            slot[(9 + k) * BS_FRONT] = val(Y[k]);
        }
        A.p = slot;
        A.stride = BS_FRONT;
        B.p = slot + 9 * BS_FRONT;
        B.stride = BS_FRONT;
        eps = R(T(0.5)) * (R(a.node_eps[ia]) + R(a.node_eps[ib]));
    }
    __device__ __forceinline__ void store(int64_t j, const Rec<R>& r) const {
        a.kind[j] = (int8_t)r.kind;
        if (r.kind != KIND_CONTACT) return;
        const int64_t ia = a.fa[j], ib = a.fb[j];
        if (!(a.is_fine[ia] && a.is_fine[ib])) return;
        const unsigned long long slot = atomicAdd(a.n_contacts, 1ull);
        if ((long long)slot >= a.max_contacts) return;
        a.c_idx[3 * slot] = a.ftag[j];
        a.c_idx[3 * slot + 1] = (int32_t)ia;
        a.c_idx[3 * slot + 2] = (int32_t)ib;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            a.c_pa[3 * slot + c] = val(r.pa[c]);
            a.c_pb[3 * slot + c] = val(r.pb[c]);
        }
    }
    __device__ __forceinline__ void mark_degenerate(int64_t j) const { a.kind[j] = (int8_t)KIND_DEGENERATE; }
    __device__ __forceinline__ void store_ids01(int64_t, uint32_t) const {}
};

template <typename T, bool STRICT>
__global__ void __launch_bounds__(BS_FRONT, TC_MINB(BS_FRONT, TC_HYBRID_MINB)) frontier_hybrid_kernel(FrontierArgs<T> a) {
    using R = typename Pol<T, STRICT>::R;
    __shared__ Queues<BS_FRONT> Q;
    __shared__ unsigned long long hist[32];
    const KP<R> kp = make_kp<R>(a);
    const FrontierSource<R, T> src{a};
    Tally tl;
    if (threadIdx.x == 0) Q.n1 = Q.n2 = 0;
    if (threadIdx.x < 32) hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t ntiles = (a.n + BS_FRONT - 1) / BS_FRONT;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t i = tile * BS_FRONT + threadIdx.x;
        bool enq = false;
        if (i < a.n) {
            const int64_t ia = a.fa[i], ib = a.fb[i];
            R A[9], B[9];
            load_node(a, ia, A);
            load_node(a, ib, B);
            T* slot = thread_slot<T>(SCR * BS_FRONT);
            stash_pair<BS_FRONT>(slot, A, B);
            const bool both_fine = a.is_fine[ia] && a.is_fine[ib];
            const int h = max(a.height[ia], a.height[ib]);
            atomicAdd(&hist[h < 31 ? h : 31], 1ull);
            Rec<R> r;
            run_iterative<BS_FRONT>(slot, A, B,
                          [&] { return R(T(0.5)) * (R(a.node_eps[ia]) + R(a.node_eps[ib])); }, kp, r);
            tl.iterative++;
            enq = r.kind == KIND_NOT_TERMINATED && both_fine;  // screened for degeneracy in the batches
            if (!enq) {
                src.store(i, r);
                tl.result(r);
            }
        }
        push(Q.q1, &Q.n1, enq, i, 2 * BS_FRONT);
        __syncthreads();
        drain<true, R>(src, Q, tl, false, (uint32_t)FLAG_FALLBACK);
    }
    drain<true, R>(src, Q, tl, true, (uint32_t)FLAG_FALLBACK);
    __syncthreads();
    if (threadIdx.x <= (unsigned)a.max_height && threadIdx.x < 32 && hist[threadIdx.x])
        atomicAdd(a.checks + threadIdx.x, hist[threadIdx.x]);
    tl.flush<true>(a.stats);
}

// Unfolding: how many next-round pairings each pairing spawns.
__global__ void frontier_count_kernel(const int8_t* kind, const int32_t* fa, const int32_t* fb, int64_t n,
                                      const uint8_t* is_fine, const int32_t* child_off, int64_t* count) {
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < n; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t ia = fa[f], ib = fb[f];
        const bool fi = is_fine[ia], fj = is_fine[ib];
        const int k = kind[f];
        int64_t c = 0;
        if ((k == KIND_CONTACT || k == KIND_NOT_TERMINATED) && !(fi && fj)) {
            const int64_t ni = fi ? 1 : child_off[ia + 1] - child_off[ia];
            const int64_t nj = fj ? 1 : child_off[ib + 1] - child_off[ib];
            c = ni * nj;
        }
        count[f] = c;
    }
}

// Unfolding: write the children meshgrid (indexing "ij") of every spawning
// pairing at its exclusive-scan offset.
__global__ void frontier_write_kernel(const int32_t* fa, const int32_t* fb, const int32_t* ftag, int64_t n,
                                      const int64_t* count, const int64_t* offset, const uint8_t* is_fine,
                                      const int32_t* child_off, const int32_t* child_ids, int32_t* na, int32_t* nb,
                                      int32_t* ntag) {
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < n; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = count[f];
        if (!c) continue;
        const int32_t ia = fa[f], ib = fb[f];
        const bool fi = is_fine[ia], fj = is_fine[ib];
        const int64_t nj = fj ? 1 : child_off[ib + 1] - child_off[ib];
        const int64_t base = offset[f];
        for (int64_t r = 0; r < c; ++r) {
            const int64_t u = r / nj, v = r - u * nj;
            na[base + r] = fi ? ia : child_ids[child_off[ia] + u];
            nb[base + r] = fj ? ib : child_ids[child_off[ib] + v];
            ntag[base + r] = ftag[f];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(BLOCK) cpt_kernel(const T* P, const T* Tr, int64_t n, T* closest, T* bary) {
    using R = Strict<T>;
    for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        R p[3], t[9], c[3], u, w;
#pragma unroll
        for (int k = 0; k < 3; ++k) p[k] = R(P[3 * i + k]);
#pragma unroll
        for (int k = 0; k < 9; ++k) t[k] = R(Tr[9 * i + k]);
        closest_point_triangle(p, t, c, u, w);
        if (closest) { closest[3 * i] = c[0].v; closest[3 * i + 1] = c[1].v; closest[3 * i + 2] = c[2].v; }
        if (bary) { bary[2 * i] = u.v; bary[2 * i + 1] = w.v; }
    }
}

// Point-to-triangle distance with an indexed triangle per point (surrogate
// halo checks, RK/surrogate.py:237-257 conservative_epsilon and :463-505
// validate_conservative): closest point (RK/kernels.py:157), then
// np.linalg.norm(p - closest) in the reference's order, all in strict IEEE.
template <typename T>
__global__ void __launch_bounds__(BLOCK) ptd_kernel(const T* P, const T* Tr, const int32_t* tri_index, int64_t n,
                                                    T* distance, T* closest) {
    using R = Strict<T>;
    for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        const int64_t t_i = tri_index ? (int64_t)__ldg(tri_index + i) : i;
        R p[3], t[9], c[3], u, w, d[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) p[k] = R(__ldg(P + 3 * i + k));
#pragma unroll
        for (int k = 0; k < 9; ++k) t[k] = R(__ldg(Tr + 9 * t_i + k));
        closest_point_triangle(p, t, c, u, w);
#pragma unroll
        for (int k = 0; k < 3; ++k) d[k] = p[k] - c[k];
        distance[i] = sqrtv(norm3_sq_sum(d)).v;
        if (closest) { closest[3 * i] = c[0].v; closest[3 * i + 1] = c[1].v; closest[3 * i + 2] = c[2].v; }
    }
}

template <typename T>
__global__ void __launch_bounds__(BLOCK) degenerate_kernel(const T* Tr, int64_t n, double rel_tol, uint8_t* mask) {
    using R = Strict<T>;
    for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        R t[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) t[k] = R(Tr[9 * i + k]);
        mask[i] = degenerate_tri(t, rel_tol) ? 1 : 0;
    }
}

// FMA-pipe throughput probe: 8 independent FMA chains per thread, the
// denominator of the FP64/FP32 roofline (MEASURED_PEAKS.json has no FP64
// figure).  flops per launch = 2 * 8 * iters * blocks * BLOCK.
template <typename T>
__global__ void __launch_bounds__(BLOCK) fma_probe_kernel(T* sink, int iters) {
    T a[8];
    const T b = T(0.999999), c = T(1e-7);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = T(threadIdx.x + k) * T(1e-3);
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
        }
    }
    T s = T(0);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == T(-1)) sink[blockIdx.x] = s;  // never true; keeps the chains alive
}

// ---- device workload generator (benchmark / test helper) -------------------------
// The cfg0 distribution of BASELINE.json (A ~ U[0,1]^9; B = R(q)(A - c_A) + c_A
// + s u with q ~ N(0,1)^4 and u ~ N(0,1)^3 normalised, s ~ U[lo, hi]) drawn
// from a counter-based Philox4x32-10 stream keyed by (seed, pair index), so
// any pair range (a shard) is generated independently, in place, in HBM --
// the 2^28-pair cfg4 set costs milliseconds instead of minutes of host numpy.
// workloads.philox_pairs is the numpy mirror (tests/test_workloads.py).
struct Philox {
    uint32_t c[4];
};
__device__ __forceinline__ Philox philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                uint32_t k1) {
    Philox r{{c0, c1, c2, c3}};
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * r.c[0], hi0 = __umulhi(0xD2511F53u, r.c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * r.c[2], hi1 = __umulhi(0xCD9E8D57u, r.c[2]);
        r = Philox{{hi1 ^ r.c[1] ^ k0, lo1, hi0 ^ r.c[3] ^ k1, lo0}};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return r;
}
// 53-bit uniform in [0, 1) from two words (numpy's random_standard_uniform recipe)
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

__global__ void random_pairs_kernel(uint64_t seed, int64_t start, int64_t n, double lo, double hi, double* planes) {
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32) ^ 0x5EEDu;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t id = (uint64_t)(start + i);
        double u[18];
#pragma unroll
        for (int call = 0; call < 9; ++call) {
            const Philox r = philox4x32_10((uint32_t)id, (uint32_t)(id >> 32), (uint32_t)call, 0u, k0, k1);
            u[2 * call] = u53(r.c[0], r.c[1]);
            u[2 * call + 1] = u53(r.c[2], r.c[3]);
        }
        // u[0..8]: A; u[9]: s; u[10..17]: four Box-Muller pairs -> q (4), u (3)
        double z[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double rr = sqrt(-2.0 * log(1.0 - u[10 + 2 * k]));
            double sn, cs;
            sincospi(2.0 * u[11 + 2 * k], &sn, &cs);
            z[2 * k] = rr * cs;
            z[2 * k + 1] = rr * sn;
        }
        const double qn = rsqrt(z[0] * z[0] + z[1] * z[1] + z[2] * z[2] + z[3] * z[3]);
        const double w = z[0] * qn, x = z[1] * qn, y = z[2] * qn, zz = z[3] * qn;
        const double R[9] = {1 - 2 * (y * y + zz * zz), 2 * (x * y - w * zz), 2 * (x * zz + w * y),
                             2 * (x * y + w * zz), 1 - 2 * (x * x + zz * zz), 2 * (y * zz - w * x),
                             2 * (x * zz - w * y), 2 * (y * zz + w * x), 1 - 2 * (x * x + y * y)};
        const double un = rsqrt(z[4] * z[4] + z[5] * z[5] + z[6] * z[6]);
        const double s = lo + (hi - lo) * u[9];
        double c[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) c[d] = (u[d] + u[3 + d] + u[6 + d]) * (1.0 / 3.0);
#pragma unroll
        for (int v = 0; v < 3; ++v) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double b = R[3 * d] * (u[3 * v] - c[0]) + R[3 * d + 1] * (u[3 * v + 1] - c[1]) +
                                 R[3 * d + 2] * (u[3 * v + 2] - c[2]) + c[d] + s * z[4 + d] * un;
                planes[(int64_t)(3 * v + d) * n + i] = u[3 * v + d];
                planes[(int64_t)(9 + 3 * v + d) * n + i] = b;
            }
        }
    }
}

__global__ void stats_reset_kernel(tc_stats* s) {
    s->iterative = s->comparison = s->fallback = s->degenerate = s->contacts = s->intersecting = 0;
    s->min_distance = __builtin_huge_val();
}

// ---- launch helpers ------------------------------------------------------------------
// Per-device state is keyed by the calling thread's current device
// (cudaGetDevice), so one process can drive several GPUs through the same
// entry points.
constexpr int kMaxDevices = 64;

static int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    return dev;
}

static int sm_count() {
    static std::atomic<int> sms[kMaxDevices];
    const int dev = current_device();
    int v = sms[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// Per-device history of the warp-specialised hybrid: is its fallback warpgroup
// keeping up?  Every CTA of that kernel adds to four cumulative device counters
// -- pairs, fallbacks, polls of iterative lanes on a full ring, tiles an
// iterative warp served itself -- and CTA 0 copies them to host-mapped memory
// (posted writes at the end of the kernel: no stream operation, no
// synchronisation).  A launch reads whatever has landed and, once at least 2^16
// more pairs are accounted for, decides which instance the next launches get:
// the plain one switches to the self-serving one (TC_WS_SELF) when producers
// polled a full ring more than TC_WS_SELF_ON times per tile, the self-serving one
// back when fewer than TC_WS_SELF_OFF of its tiles were served that way.
// Measured (2^24 pairs of the cfg1 generator, fp64): separation U[-0.1, 0.5]
// (cfg1) 0.01 polls per tile, plain 2.024 ms / self-serving 2.054; U[0.05, 0.5]
// 1.9 polls, 2.271 / 2.185; U[0.1, 0.5] 2.6 polls, 2.347 / 2.232; cfg3's
// near-parallel class 706 polls, 0.365 / 0.259 ms per 2^20 pairs; its edge-edge
// class 0.5 polls, 0.169 / 0.176.  The first launches of a process, and the
// launches right after a change of workload, run the previous choice.
#ifndef TC_WS_SELF_ON
#define TC_WS_SELF_ON 1.0
#endif
#ifndef TC_WS_SELF_OFF
#define TC_WS_SELF_OFF 0.01
#endif
// With few fallbacks the warpgroup that waits for them is a quarter of the SM
// idle: the fused kernel, whose 16 warps all iterate, is 4 % faster (2^24 far
// pairs, 0.1-3 % fallbacks: 1.59-1.71 ms against 1.52-1.65; at no fallbacks
// 1.678 / 1.547; the lines cross near 17 %).  Below TC_WS_FUSED_BELOW
// fallbacks per pair the next launches use it, above TC_WS_FUSED_ABOVE the
// warp-specialised kernel again.
#ifndef TC_WS_FUSED_BELOW
#define TC_WS_FUSED_BELOW 0.08
#endif
#ifndef TC_WS_FUSED_ABOVE
#define TC_WS_FUSED_ABOVE 0.12
#endif
struct FallbackHistory {
    enum Mode { PLAIN = 0, SELF = 1, FUSED = 2 };
    unsigned long long* counters = nullptr;      // host-mapped snapshot {seq, pairs, fallbacks, ring polls, self-served tiles, seq}
    unsigned long long* dev_counters = nullptr;  // the kernels' cumulative counters + snapshot sequence (device memory)
    std::mutex mu;
    unsigned long long seen[4] = {0, 0, 0, 0};
    int cur = PLAIN;
    std::once_flag once;
    int mode() {
        if (!dev_counters) return PLAIN;
        std::lock_guard<std::mutex> lk(mu);
        unsigned long long c[4];
        volatile unsigned long long* hh = counters;
        const unsigned long long s_end = hh[5];
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int k = 0; k < 4; ++k) c[k] = hh[1 + k];
        std::atomic_thread_fence(std::memory_order_acquire);
        if (hh[0] != s_end) return cur;  // a kernel is writing its snapshot: decide at the next launch
        if (c[0] >= seen[0] + 65536 && c[1] >= seen[1] && c[2] >= seen[2] && c[3] >= seen[3]) {
            const double pairs = (double)(c[0] - seen[0]), tiles = pairs / 32.0;
            const double rate = (double)(c[1] - seen[1]) / pairs;
            if (cur == PLAIN) {
                if ((double)(c[2] - seen[2]) > TC_WS_SELF_ON * tiles) cur = SELF;
                else if (rate < TC_WS_FUSED_BELOW) cur = FUSED;
            } else if (cur == SELF) {
                if ((double)(c[3] - seen[3]) < TC_WS_SELF_OFF * tiles) cur = PLAIN;
            } else if (rate > TC_WS_FUSED_ABOVE) {
                cur = PLAIN;
            }
            for (int k = 0; k < 4; ++k) seen[k] = c[k];
        }
        return cur;
    }
    bool high() { return mode() == SELF; }
};
static FallbackHistory& fallback_history() {
    static FallbackHistory hist[kMaxDevices];
    FallbackHistory& h = hist[current_device()];
    std::call_once(h.once, [&h] {
        void *p = nullptr, *d = nullptr;
        if (cudaHostAlloc(&p, 6 * sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable) ==
                cudaSuccess &&
            cudaMalloc(&d, 5 * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMemset(d, 0, 5 * sizeof(unsigned long long)) == cudaSuccess) {
            memset(p, 0, 6 * sizeof(unsigned long long));
            h.counters = static_cast<unsigned long long*>(p);
            h.dev_counters = static_cast<unsigned long long*>(d);
        } else {
            cudaGetLastError();  // no history: the plain instance every time
        }
    });
    return h;
}

template <typename K>
static int64_t grid_for(K kernel, int64_t n, size_t smem = 0, int threads = BLOCK) {
    if (smem > 16 * 1024) {
        // opt in to the dynamic shared memory: static + dynamic may pass the
        // 48 KB default even when the dynamic part alone does not (the call is
        // cheap and idempotent)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int64_t tiles = (n + threads - 1) / threads;
    int64_t full = (int64_t)sm_count() * per_sm;
    const int64_t cap = g_max_ctas.load(std::memory_order_relaxed);
    if (cap > 0 && full > cap) full = cap;
    return tiles < full ? tiles : full;
}

enum Variant { V_COMPARISON = 0, V_ITERATIVE = 1, V_HYBRID = 2 };

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; raising its release threshold once keeps freed blocks cached between
// calls, so per-call workspaces cost no cudaMalloc/cudaFree synchronisation.
static void pool_init() {
    static std::once_flag pool_once[kMaxDevices];
    const int dev = current_device();
    std::call_once(pool_once[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

template <typename T, bool STRICT, bool SOA>
static int launch3(int variant, const Args<T>& a, cudaStream_t s) {
    if (variant == V_COMPARISON) {
        auto k = comparison_kernel<T, STRICT, SOA>;
        const size_t smem = scratch_bytes<T>(BS_CMP);  // crossing scratch + pair slot
        k<<<(unsigned)grid_for(k, a.n, smem, BS_CMP), BS_CMP, smem, s>>>(a);
    } else if (variant == V_ITERATIVE) {
        auto k = iterative_kernel<T, STRICT, SOA>;
        const size_t smem = sizeof(T) * 2 * SLOT * BS_ITER;  // double-buffered pair slots
        k<<<(unsigned)grid_for(k, a.n, smem, BS_ITER), BS_ITER, smem, s>>>(a);
    } else if constexpr (TC_WSW && !STRICT && sizeof(T) == 8) {
        // warp-specialised hybrid with warp-granular fallback: one CTA per SM
        constexpr int IW = TC_WSW_IW, FW = TC_WSW_FW;
        auto k = hybrid_wsw_kernel<T, STRICT, SOA, IW, FW>;
        const size_t smem = wsw_smem_bytes<T, IW, FW>();
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t ctas = (a.n + 32 * IW - 1) / (32 * IW);
        int64_t g = ctas < sm_count() ? ctas : sm_count();
        const int64_t cap = g_max_ctas.load(std::memory_order_relaxed);  // test knob
        if (cap > 0 && g > cap) g = cap;
        k<<<(unsigned)g, 32 * (IW + FW), smem, s>>>(a);
    } else {
        constexpr bool WS = TC_HYBRID_WS && (!STRICT || TC_WS_STRICT) &&
                            (sizeof(T) == 8 ? TC_WS_IW_F64 : TC_WS_IW_F32) > 0;
        Args<T> aw = a;
        int mode = FallbackHistory::PLAIN;
        if constexpr (WS) {
            // which kernel this device's recent fast hybrid launches ask for (fallback_history)
            // (not while the caller captures a graph: the history's first use allocates, and a
            // captured launch would freeze one choice anyway -- it gets the plain instance)
            cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(s, &cap_status) != cudaSuccess) {
                cudaGetLastError();
                cap_status = cudaStreamCaptureStatusNone;
            }
            if (TC_WS_SELF >= 1 && cap_status == cudaStreamCaptureStatusNone) {
                FallbackHistory& fh = fallback_history();
                aw.hist = fh.dev_counters;
                aw.hist_host = fh.counters;
                mode = TC_WS_SELF == 2 ? (int)FallbackHistory::SELF : fh.mode();
            }
#ifdef TC_X_FORCE_MODE  // tests of one kernel on any batch (tools/libcmp.py)
            mode = TC_X_FORCE_MODE;
#endif
        }
        bool launched = false;
        if constexpr (WS) {
            if (mode != FallbackHistory::FUSED) {
                // warp-specialised hybrid: one CTA per SM
                constexpr int IW = sizeof(T) == 8 ? TC_WS_IW_F64 : (TC_WS_IW_F32 > 0 ? TC_WS_IW_F32 : 1);
                constexpr int FWG = sizeof(T) == 8 ? TC_WS_FWG_F64 : TC_WS_FWG_F32;
                // the full-record instance (every column, no ids) has no per-column null tests
                const bool full = TC_WS_FULL && full_record(aw);
                const bool self = mode == FallbackHistory::SELF;
                auto k = full ? (self ? hybrid_ws_kernel<T, STRICT, SOA, IW, FWG, true, true>
                                      : hybrid_ws_kernel<T, STRICT, SOA, IW, FWG, true, false>)
                              : (self ? hybrid_ws_kernel<T, STRICT, SOA, IW, FWG, false, true>
                                      : hybrid_ws_kernel<T, STRICT, SOA, IW, FWG, false, false>);
                const size_t smem = ws_smem_bytes<T, IW, FWG>(self);
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                const int64_t ctas = (aw.n + 32 * IW - 1) / (32 * IW);
                int64_t g = ctas < sm_count() ? ctas : sm_count();
                const int64_t cap = g_max_ctas.load(std::memory_order_relaxed);  // test knob
                if (cap > 0 && g > cap) g = cap;
                k<<<(unsigned)g, 32 * IW + FWG * WS_FB, smem, s>>>(aw);
                launched = true;
            }
        }
        if constexpr (WS && TC_WQ) {
            if (!launched) {
                // few fallbacks: every warp iterates and serves its own queue of open pairs
                const bool full = TC_WS_FULL && full_record(aw);
                auto k = full ? hybrid_wq_kernel<T, STRICT, SOA, true> : hybrid_wq_kernel<T, STRICT, SOA, false>;
                const size_t smem = wq_smem_bytes<T>();
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                const int64_t ctas = (aw.n + 32 * WQ_WARPS - 1) / (32 * WQ_WARPS);
                int64_t g = ctas < sm_count() ? ctas : sm_count();
                const int64_t cap = g_max_ctas.load(std::memory_order_relaxed);  // test knob
                if (cap > 0 && g > cap) g = cap;
                k<<<(unsigned)g, 32 * WQ_WARPS, smem, s>>>(aw);
                launched = true;
            }
        }
        if (!launched) {
            // the fused kernel: strict builds (and, without TC_WQ, fast batches with few fallbacks)
            auto k = hybrid_kernel<T, STRICT, SOA>;
#ifndef TC_X_PAD
#define TC_X_PAD 0
#endif
            const size_t smem =
                scratch_bytes<T>(BS_HYB) + (TC_TILE_CPASYNC ? sizeof(T) * SLOT * BS_HYB : 0) + TC_X_PAD;
            k<<<(unsigned)grid_for(k, aw.n, smem, BS_HYB), BS_HYB, smem, s>>>(aw);
        }
    }
    g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : set_err("kernel launch", e);
}

static bool params_ok(const tc_params* p) {
    return p && p->epsilon > 0.0 && p->n_iterative >= 1 && p->c_factor > 0.0 && p->alpha_iterative > 0.0 &&
           p->alpha_regulariser > 0.0;
}

template <typename T>
static int run_device(int variant, const T* tri_a, const T* tri_b, int64_t n, const T* eps, const uint8_t* allow,
                      const tc_params* p, T* distance, T* pa, T* pb, T* ba, T* bb, int8_t* kind, uint8_t* ids,
                      tc_stats* stats, void* stream) {
    if (n < 0 || !params_ok(p)) {
        snprintf(g_err, sizeof(g_err), "invalid argument (n=%lld or params)", (long long)n);
        return TC_EINVAL;
    }
    if (n == 0) return TC_OK;
    if (!tri_a || !tri_b) {
        snprintf(g_err, sizeof(g_err), "NULL triangle input");
        return TC_EINVAL;
    }
    Args<T> a;
    a.tri_a = tri_a; a.tri_b = tri_b; a.n = n; a.eps = eps; a.eps_scalar = (T)p->epsilon; a.allow = allow;
    a.distance = distance; a.pa = pa; a.pb = pb; a.ba = ba; a.bb = bb; a.kind = kind;
    a.ids = (p->flags & TC_EMIT_IDS) ? ids : nullptr;
    a.stats = stats;
    a.c_factor = p->c_factor; a.alpha_it = p->alpha_iterative; a.alpha_reg = p->alpha_regulariser;
    a.move_factor = p->move_factor; a.start_coord = p->start_coord; a.n_iterative = p->n_iterative;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool strict = p->flags & TC_STRICT, soa = p->flags & TC_SOA;
    if (strict) return soa ? launch3<T, true, true>(variant, a, s) : launch3<T, true, false>(variant, a, s);
    return soa ? launch3<T, false, true>(variant, a, s) : launch3<T, false, false>(variant, a, s);
}

template <typename T>
static int run_blocks(const T* meshes, int32_t tris, int64_t n_meshes, const int32_t* mesh_tris, const T* motions,
                      const int32_t* blocks, int64_t nb,
                      const T* block_eps, const tc_params* p, int64_t max_contacts, int32_t* c_idx, T* c_dist,
                      T* c_pa, T* c_pb, int64_t* n_contacts, tc_stats* stats, void* stream) {
    if (!params_ok(p) || nb < 0 || tris < 1 || n_meshes < 1 || max_contacts < 0 || !n_contacts ||
        (max_contacts > 0 && !c_idx) || (p->flags & (TC_SOA | TC_EMIT_IDS))) {
        snprintf(g_err, sizeof(g_err), "invalid argument (blocks)");
        return TC_EINVAL;
    }
    if (nb == 0) return TC_OK;
    if (!meshes || !blocks) return TC_EINVAL;
    const size_t smem = sizeof(T) * (SCR * BS_BLK + 18 * (size_t)tris);
    if (smem > 200 * 1024) {
        snprintf(g_err, sizeof(g_err), "tris_per_mesh %d too large for shared-memory staging", tris);
        return TC_EINVAL;
    }
    BlockArgs<T> a;
    a.meshes = meshes; a.motions = motions; a.tris = tris; a.n_meshes = n_meshes; a.mesh_tris = mesh_tris;
    a.blocks = blocks; a.nb = nb;
    a.block_eps = block_eps; a.eps_scalar = (T)p->epsilon; a.max_contacts = max_contacts;
    a.c_idx = c_idx; a.c_dist = c_dist; a.c_pa = c_pa; a.c_pb = c_pb;
    a.n_contacts = reinterpret_cast<unsigned long long*>(n_contacts);
    a.stats = stats;
    a.c_factor = p->c_factor; a.alpha_it = p->alpha_iterative; a.alpha_reg = p->alpha_regulariser;
    a.move_factor = p->move_factor; a.start_coord = p->start_coord; a.n_iterative = p->n_iterative;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto launch = [&](auto k) {
        const int64_t g = grid_for(k, nb * (int64_t)BS_BLK, smem, BS_BLK);
        k<<<(unsigned)(g < nb ? g : nb), BS_BLK, smem, s>>>(a);
    };
    if (p->flags & TC_STRICT) launch(blocks_hybrid_kernel<T, true>);
    else launch(blocks_hybrid_kernel<T, false>);
    g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : set_err("blocks launch", e);
}

// Host driver of the multiscale traversal: one hybrid launch + unfolding per
// round, until the frontier is empty (one 8-byte read-back per round).
template <typename T>
static int run_multiscale(const T* tris, const int32_t* owner, const T* motions, const T* node_eps,
                          const int32_t* child_off, const int32_t* child_ids,
                          const uint8_t* is_fine, const int32_t* height, int32_t max_height, const int32_t* roots,
                          int64_t n_pairs, const tc_params* p, int64_t max_contacts, int32_t* c_idx, T* c_pa,
                          T* c_pb, int64_t* n_contacts_host, int64_t* checks_host, tc_stats* stats_host,
                          void* stream) {
    if (!params_ok(p) || n_pairs < 0 || max_height < 0 || max_height > 31 || max_contacts < 0 ||
        (p->flags & (TC_SOA | TC_EMIT_IDS)) || !n_contacts_host || (motions && !owner)) {
        snprintf(g_err, sizeof(g_err), "invalid argument (multiscale)");
        return TC_EINVAL;
    }
    *n_contacts_host = 0;
    if (n_pairs == 0) return TC_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    // device scratch (frontier, kind, counts/offsets, tallies) from the
    // stream-ordered pool: a call costs no cudaMalloc/cudaFree synchronisation
    pool_init();
    struct Buf {
        void* p = nullptr;
        cudaStream_t s = nullptr;
        ~Buf() { if (p) cudaFreeAsync(p, s); }
    };
    Buf fr_cur, kbuf, cbuf, obuf, tallies, scan_tmp;
    int64_t cap = n_pairs > 1024 ? n_pairs : 1024;
    auto alloc = [&](Buf& b, size_t bytes) -> cudaError_t {
        if (b.p) cudaFreeAsync(b.p, s);
        b.p = nullptr;
        b.s = s;
        return cudaMallocAsync(&b.p, bytes, s);
    };
    auto grow = [&](int64_t need) -> cudaError_t {
        cudaError_t r = cudaSuccess;
        if (need <= cap && kbuf.p) return r;
        cap = need > 2 * cap ? need : 2 * cap;
        if ((r = alloc(kbuf, cap)) != cudaSuccess) return r;
        if ((r = alloc(cbuf, sizeof(int64_t) * (cap + 1))) != cudaSuccess) return r;
        if ((r = alloc(obuf, sizeof(int64_t) * (cap + 1))) != cudaSuccess) return r;
        return r;
    };
    if ((e = alloc(fr_cur, 3 * sizeof(int32_t) * cap)) != cudaSuccess) return set_err("cudaMalloc", e);
    if ((e = grow(cap)) != cudaSuccess) return set_err("cudaMalloc", e);
    // tallies: n_contacts, checks[32], stats
    const size_t tb = sizeof(unsigned long long) * 33 + sizeof(tc_stats);
    if ((e = alloc(tallies, tb)) != cudaSuccess) return set_err("cudaMalloc", e);
    auto* d_nc = static_cast<unsigned long long*>(tallies.p);
    auto* d_checks = d_nc + 1;
    auto* d_stats = reinterpret_cast<tc_stats*>(d_checks + 32);
    cudaMemsetAsync(tallies.p, 0, sizeof(unsigned long long) * 33, s);
    stats_reset_kernel<<<1, 1, 0, s>>>(d_stats);
    g_launches++;
    // initial frontier: the roots
    {
        int32_t* fa = static_cast<int32_t*>(fr_cur.p);
        std::vector<int32_t> h(3 * n_pairs);
        for (int64_t k = 0; k < n_pairs; ++k) {
            h[k] = roots[2 * k];
            h[n_pairs + k] = roots[2 * k + 1];
            h[2 * n_pairs + k] = (int32_t)k;
        }
        // planar: [fa | fb | tag] with stride = current frontier length
        cudaMemcpyAsync(fa, h.data(), sizeof(int32_t) * 3 * n_pairs, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
    }
    int64_t n = n_pairs;
    const size_t smem = scratch_bytes<T>(BS_FRONT);
    size_t scan_bytes = 0;
    while (n > 0) {
        if ((e = grow(n)) != cudaSuccess) return set_err("cudaMalloc", e);
        int32_t* fa = static_cast<int32_t*>(fr_cur.p);
        int32_t* fb = fa + n;
        int32_t* ftag = fb + n;
        FrontierArgs<T> a;
        a.tris = tris; a.owner = owner; a.motions = motions; a.node_eps = node_eps; a.is_fine = is_fine; a.height = height;
        a.fa = fa; a.fb = fb; a.ftag = ftag; a.n = n;
        a.kind = static_cast<int8_t*>(kbuf.p);
        a.max_contacts = max_contacts; a.c_idx = c_idx; a.c_pa = c_pa; a.c_pb = c_pb;
        a.n_contacts = d_nc; a.checks = d_checks; a.max_height = max_height; a.stats = d_stats;
        a.c_factor = p->c_factor; a.alpha_it = p->alpha_iterative; a.alpha_reg = p->alpha_regulariser;
        a.move_factor = p->move_factor; a.start_coord = p->start_coord; a.n_iterative = p->n_iterative;
        if (p->flags & TC_STRICT) {
            auto k = frontier_hybrid_kernel<T, true>;
            k<<<(unsigned)grid_for(k, n, smem, BS_FRONT), BS_FRONT, smem, s>>>(a);
        } else {
            auto k = frontier_hybrid_kernel<T, false>;
            k<<<(unsigned)grid_for(k, n, smem, BS_FRONT), BS_FRONT, smem, s>>>(a);
        }
        g_launches++;
        const unsigned g = (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
        int64_t* cnt = static_cast<int64_t*>(cbuf.p);
        int64_t* off = static_cast<int64_t*>(obuf.p);
        frontier_count_kernel<<<g, 256, 0, s>>>(a.kind, fa, fb, n, is_fine, child_off, cnt);
        g_launches++;
        size_t need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, off, (int)(n + 1), s);
        if (need > scan_bytes) {
            if ((e = alloc(scan_tmp, need)) != cudaSuccess) return set_err("cudaMalloc", e);
            scan_bytes = need;
        }
        // count[n] must be 0 for the (n+1)-long scan: the tail entry is the total
        cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), s);
        cub::DeviceScan::ExclusiveSum(scan_tmp.p, scan_bytes, cnt, off, (int)(n + 1), s);
        g_launches++;
        int64_t total = 0;
        cudaMemcpyAsync(&total, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return set_err("multiscale round", e);
        if (total > 0) {
            Buf next;
            next.s = s;
            if ((e = cudaMallocAsync(&next.p, 3 * sizeof(int32_t) * total, s)) != cudaSuccess)
                return set_err("cudaMallocAsync", e);
            int32_t* na = static_cast<int32_t*>(next.p);
            frontier_write_kernel<<<g, 256, 0, s>>>(fa, fb, ftag, n, cnt, off, is_fine, child_off, child_ids, na,
                                                    na + total, na + 2 * total);
            g_launches++;
            std::swap(fr_cur.p, next.p);
        }
        n = total;
    }
    struct {
        unsigned long long nc, checks[32];
        tc_stats st;
    } h;
    static_assert(sizeof(h) == sizeof(unsigned long long) * 33 + sizeof(tc_stats), "tally layout");
    cudaMemcpyAsync(&h, tallies.p, sizeof(h), cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return set_err("multiscale", e);
    if ((e = cudaGetLastError()) != cudaSuccess) return set_err("multiscale", e);
    const unsigned long long h_nc = h.nc;
    const unsigned long long* h_checks = h.checks;
    const tc_stats& h_stats = h.st;
    *n_contacts_host = (int64_t)h_nc;
    if (checks_host)
        for (int k = 0; k <= max_height; ++k) checks_host[k] += (int64_t)h_checks[k];
    if (stats_host) {
        stats_host->iterative += h_stats.iterative;
        stats_host->comparison += h_stats.comparison;
        stats_host->fallback += h_stats.fallback;
        stats_host->degenerate += h_stats.degenerate;
        stats_host->contacts += h_stats.contacts;
        stats_host->intersecting += h_stats.intersecting;
        if (h_stats.min_distance < stats_host->min_distance) stats_host->min_distance = h_stats.min_distance;
    }
    if (h_stats.degenerate > 0) {
        snprintf(g_err, sizeof(g_err), "degenerate triangle in comparison fallback");
        return TC_EDEGENERATE;
    }
    return TC_OK;
}

// ---- host pipeline ----------------------------------------------------------------------
// tc_run_host_*: the pair range is processed in chunks on NS streams; chunk c
// uses slot c % NS -- H2D of its inputs, the kernel, D2H of its outputs -- so
// the copies of one chunk overlap the kernels and copies of its neighbours.
//
// Caller arrays may be pinned (cudaHostAlloc / cudaHostRegister: the DMA
// engines read and write them directly) or pageable, like the drop-in's numpy
// arrays.  cudaMemcpyAsync on pageable memory goes through the driver's
// bounce buffer synchronously and would serialise the pipeline, so each
// pageable array is staged through the slot's own pinned buffers by a pool of
// host threads: the inputs of chunk c are copied in while the GPU works on the
// chunks before it, and the results of chunk c - NS are copied out to the
// caller before its slot is reused.

struct CopyPiece {
    char* dst;
    const char* src;
    size_t bytes;
};

// Parallel memcpy on persistent host threads (the caller takes part).
class CopyPool {
  public:
    explicit CopyPool(int workers) {
        for (int i = 0; i < workers; ++i) th_.emplace_back([this] { worker(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void copy(const std::vector<CopyPiece>& segs) {
        size_t total = 0;
        for (const auto& sg : segs) total += sg.bytes;
        if (!total) return;
        const size_t parts = th_.size() + 1;
        const size_t piece = std::max<size_t>(total / (2 * parts) + 1, size_t(1) << 20);
        std::vector<CopyPiece> local;
        for (const auto& sg : segs)
            for (size_t o = 0; o < sg.bytes; o += piece)
                local.push_back({sg.dst + o, sg.src + o, std::min(piece, sg.bytes - o)});
        if (th_.empty() || local.size() == 1) {
            for (const auto& pc : local) memcpy(pc.dst, pc.src, pc.bytes);
            return;
        }
        {
            // no worker may still be inside drain() of the previous generation
            std::unique_lock<std::mutex> l(mu_);
            done_cv_.wait(l, [this] { return active_ == 0; });
            pieces_.swap(local);
            next_.store(0);
            left_.store(pieces_.size());
            ++gen_;
            ++active_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> l(mu_);
        --active_;
        done_cv_.notify_all();
        done_cv_.wait(l, [this] { return left_.load() == 0; });
    }

  private:
    void drain() {
        for (;;) {
            const size_t i = next_.fetch_add(1);
            if (i >= pieces_.size()) break;
            memcpy(pieces_[i].dst, pieces_[i].src, pieces_[i].bytes);
            if (left_.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> l(mu_);
                done_cv_.notify_all();
            }
        }
    }
    void worker() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                ++active_;
            }
            drain();
            {
                std::lock_guard<std::mutex> l(mu_);
                --active_;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::vector<CopyPiece> pieces_;
    std::atomic<size_t> next_{0}, left_{0};
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    int active_ = 0;
    bool stop_ = false;
};

struct HostSlot {
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
    void* dbuf = nullptr;   // device chunk buffers
    size_t dcap = 0;
    char* hin = nullptr;    // pinned staging of pageable inputs
    size_t hin_cap = 0;
    char* hout = nullptr;   // pinned staging of pageable outputs
    size_t hout_cap = 0;
    bool busy = false;      // work enqueued since the last finish
    std::vector<CopyPiece> out;  // staged results to copy to the caller
};

#ifndef TC_HOST_NS
#define TC_HOST_NS 3
#endif
struct HostCtx {
    static constexpr int NS = TC_HOST_NS;
    std::mutex mu;
    bool init = false;
    HostSlot slot[NS];
    tc_stats* dstats = nullptr;
    std::unique_ptr<CopyPool> pool;
};
static HostCtx g_host[kMaxDevices];  // one per device (current device of the calling thread)

static bool host_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // unregistered host memory on older runtimes: clear the error
        return false;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged;
}

static cudaError_t grow_pinned(char*& buf, size_t& cap, size_t need) {
    if (need <= cap) return cudaSuccess;
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    cap = 0;
    const cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&buf), need, cudaHostAllocDefault);
    if (e == cudaSuccess) cap = need;
    return e;
}

// Wait for a slot's work and copy its staged results to the caller.
static cudaError_t finish_slot(HostCtx& h, HostSlot& S) {
    if (!S.busy) return cudaSuccess;
    const cudaError_t e = cudaEventSynchronize(S.done);
    if (e == cudaSuccess) h.pool->copy(S.out);
    S.out.clear();
    S.busy = false;
    return e;
}

template <typename T>
static int run_host(int variant, const T* tri_a, const T* tri_b, int64_t n, const T* eps, const uint8_t* allow,
                    const tc_params* p, T* distance, T* pa, T* pb, T* ba, T* bb, int8_t* kind, uint8_t* ids,
                    tc_stats* stats) {
    if (n < 0 || !params_ok(p) || (n > 0 && (!tri_a || !tri_b)) || variant < 0 || variant > 2) {
        snprintf(g_err, sizeof(g_err), "invalid argument");
        return TC_EINVAL;
    }
    if (p->flags & TC_SOA) {
        snprintf(g_err, sizeof(g_err), "host entry points take the (n,3,3) layout only");
        return TC_EINVAL;
    }
    HostCtx& h = g_host[current_device()];
    std::lock_guard<std::mutex> lock(h.mu);
    cudaError_t e;
    if (!h.init) {
        for (auto& S : h.slot) {
            if ((e = cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking)) != cudaSuccess)
                return set_err("cudaStreamCreate", e);
            if ((e = cudaEventCreateWithFlags(&S.done, cudaEventDisableTiming)) != cudaSuccess)
                return set_err("cudaEventCreate", e);
        }
        if ((e = cudaMalloc(&h.dstats, sizeof(tc_stats))) != cudaSuccess) return set_err("cudaMalloc", e);
        const char* v = getenv("TC_HOST_THREADS");  // host copy threads (pageable staging)
        const int hw = (int)std::thread::hardware_concurrency();
        const int nt = v ? atoi(v) : std::min(std::max(hw, 1), 16);
        h.pool.reset(new CopyPool(std::max(nt, 1) - 1));
        h.init = true;
    }
    const bool want_ids = (p->flags & TC_EMIT_IDS) && ids;
    // which caller arrays are pageable (staged) and the staging bytes per pair
    struct Arr {
        const void* src;  // caller array (input or output)
        size_t per;       // bytes per pair
        bool staged;
    };
    Arr in[4] = {{tri_a, 9 * sizeof(T), false}, {tri_b, 9 * sizeof(T), false}, {eps, sizeof(T), false},
                 {allow, 1, false}};
    Arr out[7] = {{distance, sizeof(T), false}, {pa, 3 * sizeof(T), false}, {pb, 3 * sizeof(T), false},
                  {ba, 2 * sizeof(T), false}, {bb, 2 * sizeof(T), false}, {kind, 1, false},
                  {want_ids ? ids : nullptr, 4, false}};
    size_t in_per = 0, out_per = 0, dev_per = 0;
    for (auto& a : in) {
        if (!a.src) continue;
        a.staged = !host_pinned(a.src);
        if (a.staged) in_per += a.per;
        dev_per += a.per;
    }
    for (auto& a : out) {
        if (!a.src) continue;
        a.staged = !host_pinned(a.src);
        if (a.staged) out_per += a.per;
        dev_per += a.per;
    }
    // pairs per pipeline chunk (TC_HOST_CHUNK overrides): n / 8 within [64K,
    // 1M] when every array is pinned (DMA only); with staged arrays smaller
    // chunks, n / 16 within [64K, 256K], overlap the copy threads' work with
    // the transfers more finely (measured: 2^24 pairs 71 -> 65 ms)
    int64_t chunk;
    {
        const char* v = getenv("TC_HOST_CHUNK");
        const long long c = v ? atoll(v) : 0;
        const bool staged = in_per + out_per > 0;
        chunk = c >= 4096 ? (int64_t)c
                          : std::min<int64_t>(int64_t(1) << (staged ? 18 : 20),
                                              std::max<int64_t>(65536, n / (staged ? 16 : 8)));
        chunk = (chunk + 4095) & ~int64_t(4095);
    }
    const int64_t cmax = n < chunk ? (n > 0 ? n : 1) : chunk;
    const size_t slack = 256 * 16;  // 256-byte alignment of every carved array
    for (auto& S : h.slot) {
        const size_t need = dev_per * (size_t)cmax + slack;
        if (need > S.dcap) {
            if (S.dbuf) cudaFree(S.dbuf);
            S.dbuf = nullptr;
            S.dcap = 0;
            if ((e = cudaMalloc(&S.dbuf, need)) != cudaSuccess) return set_err("cudaMalloc", e);
            S.dcap = need;
        }
        if (in_per && (e = grow_pinned(S.hin, S.hin_cap, in_per * (size_t)cmax + slack)) != cudaSuccess)
            return set_err("cudaHostAlloc", e);
        if (out_per && (e = grow_pinned(S.hout, S.hout_cap, out_per * (size_t)cmax + slack)) != cudaSuccess)
            return set_err("cudaHostAlloc", e);
    }
    cudaStream_t s0 = h.slot[0].st;
    stats_reset_kernel<<<1, 1, 0, s0>>>(h.dstats);
    g_launches++;
    cudaEventRecord(h.slot[0].done, s0);
    for (int k = 1; k < HostCtx::NS; ++k) cudaStreamWaitEvent(h.slot[k].st, h.slot[0].done, 0);
    int rc = TC_OK;
    cudaError_t herr = cudaSuccess;
    for (int64_t c0 = 0, ci = 0; c0 < n && rc == TC_OK; c0 += chunk, ++ci) {
        const int64_t m = (n - c0) < chunk ? (n - c0) : chunk;
        HostSlot& S = h.slot[ci % HostCtx::NS];
        // the slot's staging buffers are free once its previous chunk is done
        if ((e = finish_slot(h, S)) != cudaSuccess) {
            herr = e;
            break;
        }
        cudaStream_t s = S.st;
        char* dbase = static_cast<char*>(S.dbuf);
        char* ibase = S.hin;
        char* obase = S.hout;
        auto carve = [](char*& b, size_t bytes) {
            char* r = b;
            b += (bytes + 255) & ~size_t(255);
            return r;
        };
        void* dptr[4] = {nullptr, nullptr, nullptr, nullptr};
        const char* hsrc[4] = {nullptr, nullptr, nullptr, nullptr};
        std::vector<CopyPiece> stage_in;
        for (int k = 0; k < 4; ++k) {
            if (!in[k].src) continue;
            const size_t bytes = in[k].per * (size_t)m;
            hsrc[k] = static_cast<const char*>(in[k].src) + in[k].per * (size_t)c0;
            dptr[k] = carve(dbase, bytes);
            if (in[k].staged) {
                char* st = carve(ibase, bytes);
                stage_in.push_back({st, hsrc[k], bytes});
                hsrc[k] = st;
            }
        }
        h.pool->copy(stage_in);  // fill the pinned staging before its DMA is enqueued
        for (int k = 0; k < 4; ++k)
            if (dptr[k]) cudaMemcpyAsync(dptr[k], hsrc[k], in[k].per * (size_t)m, cudaMemcpyHostToDevice, s);
        void* optr[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        for (int k = 0; k < 7; ++k)
            if (out[k].src) optr[k] = carve(dbase, out[k].per * (size_t)m);
        rc = run_device<T>(variant, (const T*)dptr[0], (const T*)dptr[1], m, (const T*)dptr[2],
                           (const uint8_t*)dptr[3], p, (T*)optr[0], (T*)optr[1], (T*)optr[2], (T*)optr[3],
                           (T*)optr[4], (int8_t*)optr[5], (uint8_t*)optr[6], h.dstats, s);
        for (int k = 0; k < 7; ++k) {
            if (!out[k].src) continue;
            const size_t bytes = out[k].per * (size_t)m;
            char* dst = static_cast<char*>(const_cast<void*>(out[k].src)) + out[k].per * (size_t)c0;
            if (out[k].staged) {
                char* st = carve(obase, bytes);
                S.out.push_back({dst, st, bytes});
                dst = st;
            }
            cudaMemcpyAsync(dst, optr[k], bytes, cudaMemcpyDeviceToHost, s);
        }
        cudaEventRecord(S.done, s);
        S.busy = true;
    }
    for (auto& S : h.slot) {
        e = finish_slot(h, S);
        if (herr == cudaSuccess) herr = e;
    }
    tc_stats hs;
    cudaMemcpy(&hs, h.dstats, sizeof(tc_stats), cudaMemcpyDeviceToHost);  // after every slot is done
    if (rc != TC_OK) return rc;
    if (herr == cudaSuccess) herr = cudaGetLastError();
    if (herr != cudaSuccess) return set_err("host pipeline", herr);
    if (stats) {
        stats->iterative += hs.iterative;
        stats->comparison += hs.comparison;
        stats->fallback += hs.fallback;
        stats->degenerate += hs.degenerate;
        stats->contacts += hs.contacts;
        stats->intersecting += hs.intersecting;
        if (hs.min_distance < stats->min_distance) stats->min_distance = hs.min_distance;
    }
    if (variant == V_HYBRID && hs.degenerate > 0) {
        snprintf(g_err, sizeof(g_err), "degenerate triangle in comparison fallback");
        return TC_EDEGENERATE;
    }
    return TC_OK;
}

// Pinned host blocks for result arrays (tc_host_alloc / tc_host_free): a
// caller that allocates its outputs here gets them written by DMA directly
// (tc_run_host_* sees pinned memory and skips the copy-out staging).  Freed
// blocks are cached by size (2 MB granules) up to TC_HOST_POOL_MB (default
// 16 GB), so steady-state calls never pay cudaHostAlloc.
struct HostPool {
    std::mutex mu;
    std::vector<std::pair<size_t, void*>> free_blocks;
    std::vector<std::pair<void*, size_t>> live;
    size_t cached = 0;
    size_t cap() const {
        const char* v = getenv("TC_HOST_POOL_MB");
        return (size_t)(v ? atoll(v) : 16384) << 20;
    }
};
static HostPool g_pool;

static void* host_alloc(int64_t bytes) {
    if (bytes <= 0) return nullptr;
    const size_t sz = ((size_t)bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    std::lock_guard<std::mutex> l(g_pool.mu);
    // best fit among cached blocks of [sz, 2 sz]
    size_t best = g_pool.free_blocks.size();
    for (size_t k = 0; k < g_pool.free_blocks.size(); ++k) {
        const size_t b = g_pool.free_blocks[k].first;
        if (b >= sz && b <= 2 * sz && (best == g_pool.free_blocks.size() || b < g_pool.free_blocks[best].first))
            best = k;
    }
    if (best < g_pool.free_blocks.size()) {
        const size_t bsz = g_pool.free_blocks[best].first;
        void* p = g_pool.free_blocks[best].second;
        g_pool.free_blocks.erase(g_pool.free_blocks.begin() + best);
        g_pool.cached -= bsz;
        g_pool.live.push_back({p, bsz});
        return p;
    }
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, sz, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        // release the cache and retry once
        for (auto& b : g_pool.free_blocks) cudaFreeHost(b.second);
        g_pool.free_blocks.clear();
        g_pool.cached = 0;
        cudaGetLastError();
        if ((e = cudaHostAlloc(&p, sz, cudaHostAllocPortable)) != cudaSuccess) {
            set_err("cudaHostAlloc", e);
            return nullptr;
        }
    }
    g_pool.live.push_back({p, sz});
    return p;
}

static int host_free(void* p) {
    if (!p) return TC_OK;
    std::lock_guard<std::mutex> l(g_pool.mu);
    for (size_t k = 0; k < g_pool.live.size(); ++k) {
        if (g_pool.live[k].first == p) {
            const size_t sz = g_pool.live[k].second;
            g_pool.live.erase(g_pool.live.begin() + k);
            if (g_pool.cached + sz <= g_pool.cap()) {
                g_pool.free_blocks.push_back({sz, p});
                g_pool.cached += sz;
            } else {
                cudaFreeHost(p);
            }
            return TC_OK;
        }
    }
    snprintf(g_err, sizeof(g_err), "tc_host_free: %p was not allocated by tc_host_alloc", p);
    return TC_EINVAL;
}

template <typename T>
static int run_cpt(const T* P, const T* Tr, int64_t n, T* closest, T* bary, void* stream) {
    if (n < 0 || (n > 0 && (!P || !Tr))) return TC_EINVAL;
    if (n == 0) return TC_OK;
    auto k = cpt_kernel<T>;
    k<<<(unsigned)grid_for(k, n), BLOCK, 0, reinterpret_cast<cudaStream_t>(stream)>>>(P, Tr, n, closest, bary);
    g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : set_err("cpt launch", e);
}

template <typename T>
static int run_ptd(const T* P, const T* Tr, int64_t n_tris, const int32_t* tri_index, int64_t n, T* distance,
                   T* closest, void* stream) {
    if (n < 0 || n_tris < 0 || (n > 0 && (!P || !Tr || !distance)) || (!tri_index && n > n_tris)) return TC_EINVAL;
    if (n == 0) return TC_OK;
    auto k = ptd_kernel<T>;
    k<<<(unsigned)grid_for(k, n), BLOCK, 0, reinterpret_cast<cudaStream_t>(stream)>>>(P, Tr, tri_index, n, distance,
                                                                                       closest);
    g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : set_err("point-triangle launch", e);
}

template <typename T>
static int run_degenerate(const T* Tr, int64_t n, double rel_tol, uint8_t* mask, void* stream) {
    if (n < 0 || (n > 0 && (!Tr || !mask))) return TC_EINVAL;
    if (n == 0) return TC_OK;
    auto k = degenerate_kernel<T>;
    k<<<(unsigned)grid_for(k, n), BLOCK, 0, reinterpret_cast<cudaStream_t>(stream)>>>(Tr, n, rel_tol, mask);
    g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : set_err("degenerate launch", e);
}

// Synchronous host-pointer helpers: one temporary device buffer per call.
template <typename T>
static int run_cpt_host(const T* P, const T* Tr, int64_t n, T* closest, T* bary) {
    if (n < 0 || (n > 0 && (!P || !Tr))) return TC_EINVAL;
    if (n == 0) return TC_OK;
    char* d = nullptr;
    const size_t bytes = sizeof(T) * 17 * (size_t)n;
    cudaError_t e = cudaMalloc(&d, bytes);
    if (e != cudaSuccess) return set_err("cudaMalloc", e);
    T* dP = (T*)d;
    T* dT = dP + 3 * n;
    T* dC = dT + 9 * n;
    T* dB = dC + 3 * n;
    cudaMemcpy(dP, P, sizeof(T) * 3 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dT, Tr, sizeof(T) * 9 * n, cudaMemcpyHostToDevice);
    int rc = run_cpt<T>(dP, dT, n, dC, dB, nullptr);
    if (rc == TC_OK) {
        if (closest) cudaMemcpy(closest, dC, sizeof(T) * 3 * n, cudaMemcpyDeviceToHost);
        if (bary) cudaMemcpy(bary, dB, sizeof(T) * 2 * n, cudaMemcpyDeviceToHost);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = set_err("cpt host", e);
    }
    cudaFree(d);
    return rc;
}

template <typename T>
static int run_degenerate_host(const T* Tr, int64_t n, double rel_tol, uint8_t* mask) {
    if (n < 0 || (n > 0 && (!Tr || !mask))) return TC_EINVAL;
    if (n == 0) return TC_OK;
    char* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(T) * 9 * (size_t)n + (size_t)n);
    if (e != cudaSuccess) return set_err("cudaMalloc", e);
    T* dT = (T*)d;
    uint8_t* dM = (uint8_t*)(dT + 9 * n);
    cudaMemcpy(dT, Tr, sizeof(T) * 9 * n, cudaMemcpyHostToDevice);
    int rc = run_degenerate<T>(dT, n, rel_tol, dM, nullptr);
    if (rc == TC_OK) {
        cudaMemcpy(mask, dM, n, cudaMemcpyDeviceToHost);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = set_err("degenerate host", e);
    }
    cudaFree(d);
    return rc;
}

}  // namespace tc

// ---- C ABI ------------------------------------------------------------------------------
extern "C" {

void tc_params_default(tc_params* p) {
    p->epsilon = 1e-2;
    p->c_factor = 1.0;
    p->alpha_iterative = 10.0;
    p->alpha_regulariser = 1e-4;
    p->move_factor = 0.25;
    p->start_coord = 1.0 / 3.0;
    p->n_iterative = 4;
    p->flags = 0;
}

int tc_abi_version(void) { return TC_ABI_VERSION; }
const char* tc_last_error(void) { return tc::g_err; }
int64_t tc_launch_count(void) { return tc::g_launches.load(); }

}  // extern "C"

namespace tc {
// NCCL entry points, resolved from libnccl.so.2 on first use so the library
// loads (and every other entry point works) without NCCL present.  A process
// that already loaded an NCCL (e.g. torch's) gets that copy: same soname.
struct NcclApi {
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
static const NcclApi* nccl_api() {
    static NcclApi api;
    static bool ok = false;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        ok = api.group_start && api.group_end && api.all_reduce && api.error_string;
    });
    return ok ? &api : nullptr;
}
}  // namespace tc

extern "C" {

int tc_allreduce_stats(tc_stats* stats, void* nccl_comm, void* stream) {
    if (!stats || !nccl_comm) {
        snprintf(tc::g_err, sizeof(tc::g_err), "tc_allreduce_stats: NULL stats or communicator");
        return TC_EINVAL;
    }
    const tc::NcclApi* api = tc::nccl_api();
    if (!api) {
        snprintf(tc::g_err, sizeof(tc::g_err), "tc_allreduce_stats: libnccl.so.2 not found");
        return TC_ENODEVICE;
    }
    auto comm = reinterpret_cast<ncclComm_t>(nccl_comm);
    auto s = reinterpret_cast<cudaStream_t>(stream);
    // one group: SUM of the six int64 tallies, MIN of the fp64 minimum distance
    ncclResult_t r = api->group_start();
    if (r == ncclSuccess) {
        const ncclResult_t r1 = api->all_reduce(stats, stats, 6, ncclInt64, ncclSum, comm, s);
        const ncclResult_t r2 =
            api->all_reduce(&stats->min_distance, &stats->min_distance, 1, ncclFloat64, ncclMin, comm, s);
        r = api->group_end();
        if (r1 != ncclSuccess) r = r1;
        else if (r2 != ncclSuccess) r = r2;
    }
    if (r != ncclSuccess) {
        snprintf(tc::g_err, sizeof(tc::g_err), "tc_allreduce_stats: %s", api->error_string(r));
        return TC_ECUDA;
    }
    return TC_OK;
}

void tc_debug_set_max_ctas(int64_t max_ctas) { tc::g_max_ctas.store(max_ctas > 0 ? max_ctas : 0); }
void tc_debug_fallback_history(uint64_t out[4]) {
    tc::FallbackHistory& h = tc::fallback_history();
    for (int k = 0; k < 4; ++k) out[k] = h.counters ? ((volatile unsigned long long*)h.counters)[1 + k] : 0;
}
int tc_debug_fallback_rate_high(void) { return TC_WS_SELF == 1 && tc::fallback_history().high() ? 1 : 0; }
int tc_debug_hybrid_mode(void) { return TC_WS_SELF == 1 ? tc::fallback_history().mode() : 0; }

void* tc_host_alloc(int64_t bytes) { return tc::host_alloc(bytes); }
int tc_host_free(void* p) { return tc::host_free(p); }

int64_t tc_fma_probe(int fp64, int64_t blocks, int iters, void* sink, void* stream) {
    if (blocks < 1 || iters < 1 || !sink) return -1;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (fp64) tc::fma_probe_kernel<double><<<(unsigned)blocks, tc::BLOCK, 0, s>>>((double*)sink, iters);
    else tc::fma_probe_kernel<float><<<(unsigned)blocks, tc::BLOCK, 0, s>>>((float*)sink, iters);
    tc::g_launches++;
    if (cudaGetLastError() != cudaSuccess) return -1;
    return (int64_t)2 * 8 * 16 * iters * blocks * tc::BLOCK;
}

int tc_random_pairs_soa_f64(uint64_t seed, int64_t start, int64_t n, double sep_lo, double sep_hi, double* planes,
                            void* stream) {
    if (n < 0 || start < 0 || (n > 0 && !planes)) return TC_EINVAL;
    if (n == 0) return TC_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)tc::sm_count() * 8);
    tc::random_pairs_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        seed, start, n, sep_lo, sep_hi, planes);
    tc::g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : tc::set_err("random pairs launch", e);
}

int tc_stats_reset(tc_stats* stats, void* stream) {
    if (!stats) return TC_EINVAL;
    tc::stats_reset_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(stats);
    tc::g_launches++;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : tc::set_err("stats reset", e);
}

#define TC_DEVICE_ENTRY(NAME, VARIANT, T)                                                                   \
    int NAME(const T* tri_a, const T* tri_b, int64_t n, const T* eps, const tc_params* p, T* distance,      \
             T* point_a, T* point_b, T* bary_a, T* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats,     \
             void* stream) {                                                                                \
        return tc::run_device<T>(VARIANT, tri_a, tri_b, n, eps, nullptr, p, distance, point_a, point_b,    \
                                 bary_a, bary_b, kind, ids, stats, stream);                                 \
    }
TC_DEVICE_ENTRY(tc_comparison_f64, tc::V_COMPARISON, double)
TC_DEVICE_ENTRY(tc_comparison_f32, tc::V_COMPARISON, float)
TC_DEVICE_ENTRY(tc_iterative_f64, tc::V_ITERATIVE, double)
TC_DEVICE_ENTRY(tc_iterative_f32, tc::V_ITERATIVE, float)
#undef TC_DEVICE_ENTRY

int tc_hybrid_f64(const double* tri_a, const double* tri_b, int64_t n, const double* eps, const uint8_t* allow_fb,
                  const tc_params* p, double* distance, double* point_a, double* point_b, double* bary_a,
                  double* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats, void* stream) {
    return tc::run_device<double>(tc::V_HYBRID, tri_a, tri_b, n, eps, allow_fb, p, distance, point_a, point_b,
                                  bary_a, bary_b, kind, ids, stats, stream);
}
int tc_hybrid_f32(const float* tri_a, const float* tri_b, int64_t n, const float* eps, const uint8_t* allow_fb,
                  const tc_params* p, float* distance, float* point_a, float* point_b, float* bary_a,
                  float* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats, void* stream) {
    return tc::run_device<float>(tc::V_HYBRID, tri_a, tri_b, n, eps, allow_fb, p, distance, point_a, point_b,
                                 bary_a, bary_b, kind, ids, stats, stream);
}

int tc_closest_point_triangle_f64(const double* points, const double* tris, int64_t n, double* closest,
                                  double* bary, void* stream) {
    return tc::run_cpt<double>(points, tris, n, closest, bary, stream);
}
int tc_closest_point_triangle_f32(const float* points, const float* tris, int64_t n, float* closest, float* bary,
                                  void* stream) {
    return tc::run_cpt<float>(points, tris, n, closest, bary, stream);
}
int tc_point_triangle_distance_f64(const double* points, const double* tris, int64_t n_tris,
                                   const int32_t* tri_index, int64_t n, double* distance, double* closest,
                                   void* stream) {
    return tc::run_ptd<double>(points, tris, n_tris, tri_index, n, distance, closest, stream);
}
int tc_point_triangle_distance_f32(const float* points, const float* tris, int64_t n_tris, const int32_t* tri_index,
                                   int64_t n, float* distance, float* closest, void* stream) {
    return tc::run_ptd<float>(points, tris, n_tris, tri_index, n, distance, closest, stream);
}
int tc_degenerate_mask_f64(const double* tris, int64_t n, double rel_tol, uint8_t* mask, void* stream) {
    return tc::run_degenerate<double>(tris, n, rel_tol, mask, stream);
}
int tc_degenerate_mask_f32(const float* tris, int64_t n, double rel_tol, uint8_t* mask, void* stream) {
    return tc::run_degenerate<float>(tris, n, rel_tol, mask, stream);
}

int tc_closest_point_triangle_host_f64(const double* points, const double* tris, int64_t n, double* closest,
                                       double* bary) {
    return tc::run_cpt_host<double>(points, tris, n, closest, bary);
}
int tc_closest_point_triangle_host_f32(const float* points, const float* tris, int64_t n, float* closest,
                                       float* bary) {
    return tc::run_cpt_host<float>(points, tris, n, closest, bary);
}
int tc_degenerate_mask_host_f64(const double* tris, int64_t n, double rel_tol, uint8_t* mask) {
    return tc::run_degenerate_host<double>(tris, n, rel_tol, mask);
}
int tc_degenerate_mask_host_f32(const float* tris, int64_t n, double rel_tol, uint8_t* mask) {
    return tc::run_degenerate_host<float>(tris, n, rel_tol, mask);
}

int tc_blocks_hybrid_f64(const double* meshes, int32_t tris_per_mesh, int64_t n_meshes,
                         const int32_t* mesh_tris, const double* motions,
                         const int32_t* blocks,
                         int64_t n_blocks, const double* block_eps, const tc_params* p, int64_t max_contacts,
                         int32_t* contact_idx, double* contact_distance, double* contact_point_a,
                         double* contact_point_b, int64_t* n_contacts, tc_stats* stats, void* stream) {
    return tc::run_blocks<double>(meshes, tris_per_mesh, n_meshes, mesh_tris, motions, blocks, n_blocks, block_eps, p, max_contacts,
                                  contact_idx, contact_distance, contact_point_a, contact_point_b, n_contacts,
                                  stats, stream);
}
int tc_blocks_hybrid_f32(const float* meshes, int32_t tris_per_mesh, int64_t n_meshes,
                         const int32_t* mesh_tris, const float* motions,
                         const int32_t* blocks,
                         int64_t n_blocks, const float* block_eps, const tc_params* p, int64_t max_contacts,
                         int32_t* contact_idx, float* contact_distance, float* contact_point_a,
                         float* contact_point_b, int64_t* n_contacts, tc_stats* stats, void* stream) {
    return tc::run_blocks<float>(meshes, tris_per_mesh, n_meshes, mesh_tris, motions, blocks, n_blocks, block_eps, p, max_contacts,
                                 contact_idx, contact_distance, contact_point_a, contact_point_b, n_contacts, stats,
                                 stream);
}

int tc_multiscale_f64(const double* tris, const int32_t* node_owner, const double* motions, const double* node_eps, const int32_t* child_off, const int32_t* child_ids,
                      const uint8_t* is_fine, const int32_t* height, int32_t max_height, const int32_t* roots,
                      int64_t n_pairs, const tc_params* p, int64_t max_contacts, int32_t* contact_idx,
                      double* contact_point_a, double* contact_point_b, int64_t* n_contacts, int64_t* checks,
                      tc_stats* stats, void* stream) {
    return tc::run_multiscale<double>(tris, node_owner, motions, node_eps, child_off, child_ids, is_fine, height, max_height, roots,
                                      n_pairs, p, max_contacts, contact_idx, contact_point_a, contact_point_b,
                                      n_contacts, checks, stats, stream);
}
int tc_multiscale_f32(const float* tris, const int32_t* node_owner, const float* motions, const float* node_eps, const int32_t* child_off, const int32_t* child_ids,
                      const uint8_t* is_fine, const int32_t* height, int32_t max_height, const int32_t* roots,
                      int64_t n_pairs, const tc_params* p, int64_t max_contacts, int32_t* contact_idx,
                      float* contact_point_a, float* contact_point_b, int64_t* n_contacts, int64_t* checks,
                      tc_stats* stats, void* stream) {
    return tc::run_multiscale<float>(tris, node_owner, motions, node_eps, child_off, child_ids, is_fine, height, max_height, roots,
                                     n_pairs, p, max_contacts, contact_idx, contact_point_a, contact_point_b,
                                     n_contacts, checks, stats, stream);
}

int tc_run_host_f64(int variant, const double* tri_a, const double* tri_b, int64_t n, const double* eps,
                    const uint8_t* allow_fb, const tc_params* p, double* distance, double* point_a,
                    double* point_b, double* bary_a, double* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats) {
    return tc::run_host<double>(variant, tri_a, tri_b, n, eps, allow_fb, p, distance, point_a, point_b, bary_a,
                                bary_b, kind, ids, stats);
}
int tc_run_host_f32(int variant, const float* tri_a, const float* tri_b, int64_t n, const float* eps,
                    const uint8_t* allow_fb, const tc_params* p, float* distance, float* point_a, float* point_b,
                    float* bary_a, float* bary_b, int8_t* kind, uint8_t* ids, tc_stats* stats) {
    return tc::run_host<float>(variant, tri_a, tri_b, n, eps, allow_fb, p, distance, point_a, point_b, bary_a,
                               bary_b, kind, ids, stats);
}

}  // extern "C"
