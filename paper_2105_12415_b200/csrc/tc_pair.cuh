// tc_pair.cuh -- per-pair device code of the three reference kernels.
//
// One triangle pair per thread, everything in registers.  Each function
// restates one reference function (RK = /root/reference/pkg/src/tricontact)
// in the reference's operation order; R is an arithmetic policy from
// tc_math.cuh (Strict<T> = bit-exact, T = FMA-contracted).
#pragma once
#include "tc_math.cuh"

namespace tc {

// Unrolling of the comparison kernel's crossing (X) and feature (F) test
// loops: full unrolling makes every vertex index a compile-time constant.
// Measured: X fully unrolled (3) is 3.5 % faster for the comparison kernel
// and 1.2 % for the hybrid; unrolling F (3 or 9) is 4-7 % slower (spills).
// experiment: let the three unrolled segment tests interleave (needs > 128
// registers: measured with setmaxnreg roles, 120 / 152: hybrid +2.7 %)
#ifndef TC_P2_INTERLEAVE
#define TC_P2_INTERLEAVE 0
#endif
#ifndef TC_UNROLL_X
#define TC_UNROLL_X 3
#endif
#ifndef TC_UNROLL_F
#define TC_UNROLL_F 1
#endif
constexpr int kUnrollX = TC_UNROLL_X;
constexpr int kUnrollF = TC_UNROLL_F;

enum : int { KIND_NO_CONTACT = 0, KIND_CONTACT = 1, KIND_NOT_TERMINATED = 2, KIND_DEGENERATE = 3 };

// ids byte 3 flag bits
enum : uint32_t { FLAG_SETTLED = 1, FLAG_ITER_CONTACT = 2, FLAG_FALLBACK = 4, FLAG_DEGENERATE = 8,
                  FLAG_INTERSECT = 16 };

template <class R>
struct Rec {
    R distance;
    R pa[3], pb[3], ba[2], bb[2];
    int kind;
    uint32_t ids;  // byte0 feature row, byte1 region/branch, byte2 crossing pair, byte3 flags
};

template <class R>
struct KP {
    R c_factor, alpha_it, alpha_reg, move_factor, start_coord;
    int n_iterative;
};

template <class R>
__device__ __forceinline__ void sub3(const R* a, const R* b, R* o) {
    o[0] = a[0] - b[0];
    o[1] = a[1] - b[1];
    o[2] = a[2] - b[2];
}

// np.cross (cp0 = a1*b2 - a2*b1, ...), RK/geometry.py:51-54
template <class R>
__device__ __forceinline__ void cross3(const R* a, const R* b, R* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

// max squared edge length of one triangle: edges = tris[:, [1,2,0]] - tris
template <class R>
__device__ __forceinline__ R max_sq_edge(const R* t) {
    R ed[3];
    sub3(t + 3, t, ed);
    R l0 = dot3(ed, ed);
    sub3(t + 6, t + 3, ed);
    R l1 = dot3(ed, ed);
    sub3(t, t + 6, ed);
    R l2 = dot3(ed, ed);
    return maxv(maxv(l0, l1), l2);
}

// RK/geometry.py:68-75 degenerate_mask: sq_area < rel_tol * L * L, with
// rel_tol rounded to T like the reference's Python float times a T array
// (the hybrid's fallback screen uses the default 1e-12, RK/kernels.py:598)
template <class R>
__device__ __forceinline__ bool degenerate_tri(const R* t, double rel_tol = 1e-12) {
    using T = typename Store<R>::type;
    R e1[3], e2[3], c[3];
    sub3(t + 3, t, e1);
    sub3(t + 6, t, e2);
    cross3(e1, e2, c);
    R sq_area = R(T(0.25)) * dot3(c, c);
    R L = max_sq_edge(t);
    R thr = R(T(rel_tol)) * L;
    thr = thr * L;
    return (L == R(0)) || (sq_area < thr);
}

// RK/kernels.py:157-221 closest_point_triangle_batch for one point, written
// branch-free: the claimed region (claim order 0 VA, 1 VB, 2 EAB, 3 VC,
// 4 EAC, 5 EBC, 6 interior) only selects the numerators and the shared
// denominator, so the divergent region cases cost one division pair for the
// whole warp.  u, w are the weights along ab, ac; results are the
// reference's bit for bit in strict mode.
// Region and weights from the six dot products d1..d6 (RK/kernels.py:180-218).
template <class R>
__device__ __forceinline__ int region_params(R d1, R d2, R d3, R d4, R d5, R d6, R& u, R& w) {
    const R vc = d1 * d4 - d3 * d2;
    const R vb = d5 * d2 - d1 * d6;
    const R va = d3 * d6 - d5 * d4;
    const R n43 = d4 - d3, n56 = d5 - d6;
    // The claim conditions, all evaluated (bitwise &: no short-circuit
    // branches -- a branchy chain diverges across the warp's lanes).
    // d4 <= d3 and d5 <= d6 are the signs of n43 and n56: fl(a - b) has the
    // sign of a - b, so this is exact.
    const bool c0 = le0(d1) & le0(d2);
    const bool c1 = ge0(d3) & le0(n43);
    const bool c2 = le0(vc) & ge0(d1) & le0(d3);
    const bool c3 = ge0(d6) & le0(n56);
    const bool c4 = le0(vb) & ge0(d2) & le0(d6);
    const bool c5 = le0(va) & ge0(n43) & ge0(n56);
    // first claim wins: one-hot region predicates
    const bool r0 = c0, r1 = !c0 & c1, r2 = !(c0 | c1) & c2, r3 = !(c0 | c1 | c2) & c3;
    const bool r4 = !(c0 | c1 | c2 | c3) & c4, r5 = !(c0 | c1 | c2 | c3 | c4) & c5;
    const bool r6 = !(c0 | c1 | c2 | c3 | c4 | c5);
    int region = selv(c5, 5, 6);
    region = selv(c4, 4, region);
    region = selv(c3, 3, region);
    region = selv(c2, 2, region);
    region = selv(c1, 1, region);
    region = selv(c0, 0, region);
    // numerator / denominator of the region's parameter(s), by selects
    const R one = R(1), zero = R(0);
    R num = selv(r6, vb, one), den = selv(r6, (va + vb) + vc, one);
    num = selv(r5, n43, num); den = selv(r5, n43 + n56, den);
    num = selv(r4, d2, num);  den = selv(r4, d2 - d6, den);
    num = selv(r2, d1, num);  den = selv(r2, d1 - d3, den);
    den = selv(den == zero, one, den);
    R q1, qw;
    if constexpr (IsStrict<R>::value) {
        // (IEEE divisions are long: the second one only where it is used)
        q1 = num / den;
        qw = zero;
        if (r6) qw = vc / den;
    } else {
        const R r = rcpv(den);
        q1 = num * r;
        qw = vc * r;
    }
    u = selv(r1, one, selv(r2 | r6, q1, selv(r5, one - q1, zero)));
    w = selv(r3, one, selv(r4 | r5, q1, selv(r6, qw, zero)));
    (void)r0;
    return region;
}

template <class R, class Tri>
__device__ __forceinline__ int closest_point_params_t(const R* p, const Tri& tri, R& u, R& w) {
    R a[3], b[3], c[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) { a[i] = tri[i]; b[i] = tri[3 + i]; c[i] = tri[6 + i]; }
    R ab[3], ac[3], t3[3];
    sub3(b, a, ab);
    sub3(c, a, ac);
    sub3(p, a, t3);
    const R d1 = dot3(ab, t3);
    const R d2 = dot3(ac, t3);
    sub3(p, b, t3);
    const R d3 = dot3(ab, t3);
    const R d4 = dot3(ac, t3);
    sub3(p, c, t3);
    const R d5 = dot3(ab, t3);
    const R d6 = dot3(ac, t3);
    return region_params(d1, d2, d3, d4, d5, d6, u, w);
}

// Fast build: the target triangle's frame (origin, edges ab, ac and their
// Gram terms), shared by the three point tests against it.  With ap = p - a:
// d3 = d1 - ab.ab, d4 = d2 - ab.ac, d5 = d1 - ab.ac, d6 = d2 - ac.ac, and
// the offset to the closest point is ap - u ab - w ac, which also gives the
// squared distance.  Equal to the reference's d1..d6 and distance up to
// rounding (the winner's points are rebuilt with the reference's formulas).
template <class R>
struct PointFrame {
    R a[3], ab[3], ac[3], gbb, gbc, gcc;
};
template <class R, class Tri>
__device__ __forceinline__ void point_frame(const Tri& tri, PointFrame<R>& f) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        f.a[i] = tri[i];
        f.ab[i] = tri[3 + i] - f.a[i];
        f.ac[i] = tri[6 + i] - f.a[i];
    }
    f.gbb = dot3(f.ab, f.ab);
    f.gbc = dot3(f.ab, f.ac);
    f.gcc = dot3(f.ac, f.ac);
}
template <class R>
__device__ __forceinline__ int closest_point_frame(const R* p, const PointFrame<R>& f, R& u, R& w, R& dist2) {
    R ap[3];
    sub3(p, f.a, ap);
    const R d1 = dot3(f.ab, ap), d2 = dot3(f.ac, ap);
    const int region = region_params(d1, d2, d1 - f.gbb, d2 - f.gbc, d1 - f.gbc, d2 - f.gcc, u, w);
    R diff[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) diff[i] = (ap[i] - u * f.ab[i]) - w * f.ac[i];
    dist2 = dot3(diff, diff);
    return region;
}

template <class R, class Tri>
__device__ __forceinline__ void bary_point_t(const Tri& tri, R u, R w, R* out) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const R a = tri[i];
        const R ab = tri[3 + i] - a;
        const R ac = tri[6 + i] - a;
        out[i] = (a + u * ab) + w * ac;
    }
}


__device__ __forceinline__ int edge_start(int k) { return k; }
__device__ __forceinline__ int edge_end(int k) { return k == 2 ? 0 : k + 1; }

// Vertex k (runtime) of a register-resident triangle, by selects.
template <class R>
__device__ __forceinline__ void vertex_sel(const R* t, int k, R* v) {
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = (k == 0) ? t[i] : ((k == 1) ? t[3 + i] : t[6 + i]);
}

// Triangle accessors for the comparison phases: register-resident (RegTri)
// or one thread's planar shared-memory slot (SmemTri, coordinate k at
// p[k * stride]) -- the latter keeps the 18 pair coordinates out of the
// register file during the register-hungry feature tests.
template <class R>
struct RegTri {
    const R* t;
    __device__ __forceinline__ R operator[](int k) const { return t[k]; }
    __device__ __forceinline__ void vertex(int k, R* v) const { vertex_sel(t, k, v); }
};
template <class R>
struct SmemTri {
    const typename Store<R>::type* p;
    int stride;
    __device__ __forceinline__ R operator[](int k) const { return R(p[k * stride]); }
    __device__ __forceinline__ void vertex(int k, R* v) const {
#pragma unroll
        for (int i = 0; i < 3; ++i) v[i] = R(p[(3 * k + i) * stride]);
    }
};

// One triangle of a planar (SoA) global array, read through the read-only
// path: coordinate k at p[k * stride].
template <class R>
struct GlobalTri {
    const typename Store<R>::type* p;
    int64_t stride;
    __device__ __forceinline__ R operator[](int k) const { return R(__ldg(p + k * stride)); }
    __device__ __forceinline__ void vertex(int k, R* v) const {
#pragma unroll
        for (int i = 0; i < 3; ++i) v[i] = R(__ldg(p + (3 * k + i) * stride));
    }
};

// RK/geometry.py:68-75 degenerate_mask through an accessor (e.g. a pair kept
// in shared memory, so the caller's registers are not pinned by it).
template <class R, class Tri>
__device__ __forceinline__ bool degenerate_tri_t(const Tri& t) {
    R v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = t[k];
    return degenerate_tri(v);
}

template <class R>
__device__ __forceinline__ int closest_point_params(const R* p, const R* tri, R& u, R& w) {
    return closest_point_params_t(p, RegTri<R>{tri}, u, w);
}
template <class R>
__device__ __forceinline__ void bary_point(const R* tri, R u, R w, R* out) {
    bary_point_t(RegTri<R>{tri}, u, w, out);
}

// Full RK/kernels.py:157-221 (closest point and weights); used by cpt_kernel.
template <class R>
__device__ __forceinline__ int closest_point_triangle(const R* p, const R* tri, R* closest, R& u, R& w) {
    const int region = closest_point_params_t(p, RegTri<R>{tri}, u, w);
    bary_point_t(RegTri<R>{tri}, u, w, closest);
    return region;
}

// RK/kernels.py:224-252 _closest_segment_segment.  The parameters s, t are
// returned (the closest points are rebuilt for the winner only).  ra = 1/a
// and re = 1/e are the hoisted reciprocals of the two squared edge lengths
// (with the reference's TINY guard applied).  Branch code: bit0 = s from the
// 2x2 solve, bit1 = t < 0, bit2 = t > 1.
//
// la / le: the hoisted squared edge lengths (the fast build uses them
// instead of re-dotting; the same values), and the fast build takes the
// offset of the two closest points as r + s d1 - t d2.
template <class R>
__device__ __forceinline__ int segment_params(const R* p1, const R* q1, const R* p2, const R* q2, R ra, R re,
                                              R la, R le, R& s, R& t, R& d2out) {
    const R tiny = R(Tiny<R>::v);
    R d1[3], d2[3], r[3];
    sub3(q1, p1, d1);
    sub3(q2, p2, d2);
    sub3(p1, p2, r);
    const R a = IsStrict<R>::value ? dot3(d1, d1) : la;
    const R e = IsStrict<R>::value ? dot3(d2, d2) : le;
    const R f = dot3(d2, r);
    const R c = dot3(d1, r);
    const R b = dot3(d1, d2);
    const R denom = a * e - b * b;
    const bool solve = denom > tiny;
    const R s0 = divv(b * f - c * e, solve ? denom : R(1));
    s = solve ? clip01(s0) : R(0);
    const R e_safe = (e > tiny) ? e : R(1);
    t = divr(b * s + f, e_safe, re);
    const R a_safe = (a > tiny) ? a : R(1);
    const bool lo = lt0(t), hi = gt1(t);
    const R s2 = clip01(divr(lo ? -c : (b - c), a_safe, ra));
    s = (lo | hi) ? s2 : s;
    t = clip01(t);
    R diff[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        diff[i] = IsStrict<R>::value ? (p1[i] + s * d1[i]) - (p2[i] + t * d2[i]) : (r[i] + s * d1[i]) - t * d2[i];
    d2out = dot3(diff, diff);
    return (solve ? 1 : 0) | (lo ? 2 : 0) | (hi ? 4 : 0);
}

// RK/kernels.py:261-266 _edge_bary
template <class R>
__device__ __forceinline__ void edge_bary(int k, R s, R* o) {
    o[0] = (k == 0) ? s : ((k == 1) ? R(1) - s : R(0));
    o[1] = (k == 0) ? R(0) : ((k == 1) ? s : R(1) - s);
}

// Per-target-triangle constants of the edge-plane test (RK/kernels.py:269-298).
// The edge vectors u, v and the origin a are kept too: every edge test and
// vertex distance uses the same values the reference computes once per
// triangle, so hoisting them is exact in both arithmetic policies.
template <class R>
struct PlaneFrame {
    R a[3], u[3], v[3], nrm[3], uu, uv, vv, det_safe, rdet;
};

template <class R, class Tri>
__device__ __forceinline__ void plane_frame(const Tri& tri, PlaneFrame<R>& f) {
    const R tiny = R(Tiny<R>::v);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        f.a[i] = tri[i];
        f.u[i] = tri[3 + i] - f.a[i];
        f.v[i] = tri[6 + i] - f.a[i];
    }
    cross3(f.u, f.v, f.nrm);
    f.uu = dot3(f.u, f.u);
    f.uv = dot3(f.u, f.v);
    f.vv = dot3(f.v, f.v);
    const R det = f.uu * f.vv - f.uv * f.uv;
    f.det_safe = (absv(det) > tiny) ? det : R(1);
    f.rdet = rcpv(f.det_safe);
}

// Signed distance (times |n|) of a point from the frame's plane.
template <class R>
__device__ __forceinline__ R plane_dist(const R* p, const PlaneFrame<R>& f) {
    R t3[3];
    sub3(p, f.a, t3);
    return dot3(t3, f.nrm);
}

// One proper crossing test of segment [p, q] through the closed triangle,
// given the endpoints' plane distances dp, dq (plane_dist).
template <class R>
__device__ __forceinline__ bool segment_crosses(const R* p, const R* q, R dp, R dq, const PlaneFrame<R>& f, R* x) {
    R t3[3];
    const bool crossing = (dp * dq) < R(0);
    const R denom = dp - dq;
    const R t = divv(dp, denom == R(0) ? R(1) : denom);
    sub3(q, p, t3);
#pragma unroll
    for (int i = 0; i < 3; ++i) x[i] = p[i] + t * t3[i];
    sub3(x, f.a, t3);
    const R wu = dot3(t3, f.u);
    const R wv = dot3(t3, f.v);
    const R b1 = divr(f.vv * wu - f.uv * wv, f.det_safe, f.rdet);
    const R b2 = divr(f.uu * wv - f.uv * wu, f.det_safe, f.rdet);
    return crossing && (b1 >= R(0)) && (b2 >= R(0)) && ((b1 + b2) <= R(1));
}

// RK/kernels.py:301-401 comparison_batch for one pair, in two phases so a
// kernel can compact the pairs between them (the second phase only runs for
// pairs that need it, on full warps).
//
// Phase 1: the six edge-plane tests (RK/kernels.py:364-375).  Valid crossing
// points go to a small per-thread list in shared memory (usually 0 or 2
// entries, at most 4: a proper crossing needs the edge's two vertex-plane
// distances of strictly opposite sign, and around a triangle's 3-cycle of
// vertices at most 2 edges change sign -- per triangle); the farthest pair is kept with the reference's first-argmax
// order over the row-major 6x6 grid.  An intersecting pair is complete
// after this phase: distance 0, both points at the midpoint, barycentric
// coordinates of the midpoint on A and B (RK/kernels.py:377-398).
// Returns true for intersecting pairs; `o.ids` bytes 2-3 are set.
template <class R>
struct Scratch {
    // per-thread crossing-point list in shared memory: element (slot, c) of
    // this thread lives at p[(3 * slot + c) * stride] (conflict-free)
    typename Store<R>::type* p;
    int stride;
    __device__ __forceinline__ void put(int slot, const R* x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) p[(3 * slot + c) * stride] = val(x[c]);
    }
    __device__ __forceinline__ void get(int slot, R* x) const {
#pragma unroll
        for (int c = 0; c < 3; ++c) x[c] = R(p[(3 * slot + c) * stride]);
    }
    __device__ __forceinline__ void putv(int k, R v) { p[k * stride] = val(v); }
    __device__ __forceinline__ R getv(int k) const { return R(p[k * stride]); }
};

// Fast build: the weights (u, w) along (ab, ac) of a point known to lie in
// the triangle (the midpoint of two crossing points, which lie in both
// triangles up to rounding), from the 2x2 normal equations of the triangle's
// frame -- for such a point the reference's closest point is the point
// itself, its weights the same up to rounding (ill-conditioned triangles,
// det < kappa * |ab|^2 |ac|^2, take the reference's region path).
// The reference's region path in the reference's own rounding (no FMA
// contraction), out of line: the ill-conditioned branch of inside_point_params
// (slivers) is rare, and its weights are ratios of cancelling products that
// contraction makes worse (tools/bary_recon.py).
template <class T>
__device__ __noinline__ void sliver_point_params(const T* p, const T* tri, T* uw) {
    using S = Strict<T>;
    S ps[3], ts[9], u, w;
#pragma unroll
    for (int i = 0; i < 3; ++i) ps[i] = S(p[i]);
#pragma unroll
    for (int i = 0; i < 9; ++i) ts[i] = S(tri[i]);
    closest_point_params_t(ps, RegTri<S>{ts}, u, w);
    uw[0] = u.v;
    uw[1] = w.v;
}

template <class R, class Tri>
__device__ __forceinline__ void inside_point_params(const R* p, const Tri& tri, R& u, R& w) {
    using T = typename Store<R>::type;
    // (pinned operations, tc_math.cuh: the same bits in every inlining context)
    R a[3], ab[3], ac[3], ap[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        a[i] = tri[i];
        ab[i] = subp(tri[3 + i], a[i]);
        ac[i] = subp(tri[6 + i], a[i]);
        ap[i] = subp(p[i], a[i]);
    }
    const R uu = dot3p(ab, ab), uv = dot3p(ab, ac), vv = dot3p(ac, ac);
    const R det = fmav(uu, vv, -mulp(uv, uv));
    const R kappa = R(T(sizeof(T) == 8 ? 1e-6 : 1e-2));
    if (!(det >= mulp(kappa, mulp(uu, vv))) || det == R(0)) {
        // (fp32 takes this branch below sin^2 = 1e-2, 3-4 % of random triangles: those
        // keep the inlined region path; only true slivers, sin^2 < 1e-6, pay the call --
        // with every row of the branch out of line the fp32 hybrid ran 2 % slower.
        // fp64 keeps the inlined path: its weights were never outside the triangle,
        // and on all of cfg3 the out-of-line path moved one row's region decision
        // past what the checker's sensitivity probe excuses.)
        if (sizeof(T) == 8 || (det >= mulp(R(T(1e-6)), mulp(uu, vv)) && det != R(0))) {
            closest_point_params_t(p, tri, u, w);
        } else {
            T pl[3], tl[9], uw[2];
#pragma unroll
            for (int i = 0; i < 3; ++i) pl[i] = T(p[i]);
#pragma unroll
            for (int i = 0; i < 9; ++i) tl[i] = T(tri[i]);
            sliver_point_params<T>(pl, tl, uw);
            u = R(uw[0]);
            w = R(uw[1]);
        }
        // The region path's interior weights are ratios of cancelling products
        // (va, vb, vc): on slivers in fp32 the FMA-contracted build returned
        // weights tens of units outside the triangle (cfg3 slivers: the named
        // point up to 44 L from the midpoint; the reference's own stay within
        // 0.34 L).  A closest point lies on the triangle: clip to it (no change
        // for weights already inside).
        u = clipv(u, R(T(0)), R(T(1)));
        w = clipv(w, R(T(0)), R(T(1)) - u);
        return;
    }
    const R r = rcpv(det);
    const R pu = dot3p(ap, ab), pv = dot3p(ap, ac);
    u = mulp(fmav(vv, pu, -mulp(uv, pv)), r);
    w = mulp(fmav(uu, pv, -mulp(uv, pu)), r);
}

template <class R, class Tri>
__device__ __forceinline__ bool comparison_phase1(const Tri& A, const Tri& B, R eps, Scratch<R> cpts, Rec<R>& o) {
    using T = typename Store<R>::type;
    int ck = 0;  // crossing test index of each list slot, 3 bits per slot
    int nv = 0;
    {
        PlaneFrame<R> fb;
        plane_frame(B, fb);
        R s0, s1, s2;  // A's vertices against B's plane (each shared by two edges)
        {
            R v[3];
            A.vertex(0, v); s0 = plane_dist(v, fb);
            A.vertex(1, v); s1 = plane_dist(v, fb);
            A.vertex(2, v); s2 = plane_dist(v, fb);
        }
#pragma unroll kUnrollX
        for (int k = 0; k < 3; ++k) {
            R p[3], q[3], x[3];
            A.vertex(edge_start(k), p);
            A.vertex(edge_end(k), q);
            const R dp = k == 0 ? s0 : (k == 1 ? s1 : s2), dq = k == 0 ? s1 : (k == 1 ? s2 : s0);
            if (segment_crosses(p, q, dp, dq, fb, x)) {
                cpts.put(nv, x);
                ck |= k << (3 * nv);
                ++nv;
            }
        }
        PlaneFrame<R> fa;
        plane_frame(A, fa);
        {
            R v[3];
            B.vertex(0, v); s0 = plane_dist(v, fa);  // (reuses s0-s2: B's vertices vs A's plane)
            B.vertex(1, v); s1 = plane_dist(v, fa);
            B.vertex(2, v); s2 = plane_dist(v, fa);
        }
#pragma unroll kUnrollX
        for (int k = 0; k < 3; ++k) {
            R p[3], q[3], x[3];
            B.vertex(edge_start(k), p);
            B.vertex(edge_end(k), q);
            const R dp = k == 0 ? s0 : (k == 1 ? s1 : s2), dq = k == 0 ? s1 : (k == 1 ? s2 : s0);
            if (segment_crosses(p, q, dp, dq, fa, x)) {
                cpts.put(nv, x);
                ck |= (3 + k) << (3 * nv);
                ++nv;
            }
        }
    }
    if (nv == 0) {
        o.ids = 255u << 16;
        return false;
    }
    auto kof = [&](int slot) { return (ck >> (3 * slot)) & 7; };
    int i0 = 0, i1 = 0;  // list slots; (first, first) scores 0 at grid index 7*k(first)
    R bestv = R(0);
    int bidx = 7 * kof(0);
#pragma unroll 1
    for (int a = 0; a < nv; ++a) {
        R pa_[3];
        cpts.get(a, pa_);
#pragma unroll 1
        for (int b = a + 1; b < nv; ++b) {
            R pb_[3], diff[3];
            cpts.get(b, pb_);
            sub3(pa_, pb_, diff);
            const R v = dot3(diff, diff);
            const int idx = 6 * kof(a) + kof(b);
            if (v > bestv || (v == bestv && idx < bidx)) { bestv = v; bidx = idx; i0 = a; i1 = b; }
        }
    }
    R mid[3], p0[3], p1[3];
    cpts.get(i0, p0);
    cpts.get(i1, p1);
#pragma unroll
    for (int i = 0; i < 3; ++i) mid[i] = R(T(0.5)) * (p0[i] + p1[i]);
    o.distance = R(0);
#pragma unroll
    for (int i = 0; i < 3; ++i) { o.pa[i] = mid[i]; o.pb[i] = mid[i]; }
    if constexpr (IsStrict<R>::value) {
        closest_point_params_t(mid, A, o.ba[0], o.ba[1]);
        closest_point_params_t(mid, B, o.bb[0], o.bb[1]);
    } else {
        inside_point_params(mid, A, o.ba[0], o.ba[1]);
        inside_point_params(mid, B, o.bb[0], o.bb[1]);
    }
    o.kind = (o.distance <= R(T(2)) * eps) ? KIND_CONTACT : KIND_NO_CONTACT;
    o.ids = ((uint32_t)bidx << 16) | ((uint32_t)FLAG_INTERSECT << 24);
    return true;
}

// Phase 2: the 15 feature candidates (RK/kernels.py:318-362) with a running
// first minimum that keeps only (row, d^2, two parameters); the winner's
// points are rebuilt from its parameters with the reference's formulas, so
// strict results stay bit-identical.  `o.ids` bytes 0-1 get the feature row
// and its region / segment-branch code; with `ids_only` (an intersecting
// pair whose ids were requested) nothing else is written.
template <class R, class Tri>
__device__ __forceinline__ void comparison_phase2_impl(const Tri& A, const Tri& B, R eps, bool ids_only, Rec<R>& o,
                                                       Scratch<R> S) {
    using T = typename Store<R>::type;
    const R tiny = R(Tiny<R>::v);
    int best_row = 0, best_code = 0;
    R best = R(0), bp1 = R(0), bp2 = R(0);
    // (two loops with fixed source/target triangles: a runtime choice between
    // the A and B arrays would force them out of registers)
    if constexpr (IsStrict<R>::value) {
#pragma unroll kUnrollF
        for (int row = 0; row < 3; ++row) {
            R pt[3], u, w, cl[3], diff[3];
            A.vertex(row, pt);
            const int reg = closest_point_params_t(pt, B, u, w);
            bary_point_t(B, u, w, cl);
            sub3(pt, cl, diff);
            const R d2 = dot3(diff, diff);
            if (row == 0 || d2 < best) { best = d2; best_row = row; best_code = reg; bp1 = u; bp2 = w; }
        }
#pragma unroll kUnrollF
        for (int row = 3; row < 6; ++row) {
            R pt[3], u, w, cl[3], diff[3];
            B.vertex(row - 3, pt);
            const int reg = closest_point_params_t(pt, A, u, w);
            bary_point_t(A, u, w, cl);
            sub3(pt, cl, diff);
            const R d2 = dot3(diff, diff);
            if (d2 < best) { best = d2; best_row = row; best_code = reg; bp1 = u; bp2 = w; }
        }
    } else {
        PointFrame<R> f;
        point_frame(B, f);
#pragma unroll kUnrollF
        for (int row = 0; row < 3; ++row) {
            R pt[3], u, w, d2;
            A.vertex(row, pt);
            const int reg = closest_point_frame(pt, f, u, w, d2);
            if (row == 0 || d2 < best) { best = d2; best_row = row; best_code = reg; bp1 = u; bp2 = w; }
        }
        point_frame(A, f);
#pragma unroll kUnrollF
        for (int row = 3; row < 6; ++row) {
            R pt[3], u, w, d2;
            B.vertex(row - 3, pt);
            const int reg = closest_point_frame(pt, f, u, w, d2);
            if (d2 < best) { best = d2; best_row = row; best_code = reg; bp1 = u; bp2 = w; }
        }
    }
    // hoisted squared edge lengths and their reciprocals (TINY-guarded), kept
    // in the thread's crossing scratch (free in phase 2) and read back by
    // runtime index: no select chains, 24 registers fewer in the loop
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        R p[3], q[3], d[3];
        A.vertex(edge_start(k), p);
        A.vertex(edge_end(k), q);
        sub3(q, p, d);
        const R la = dot3(d, d);
        S.putv(k, la);
        S.putv(6 + k, rcpv(la > tiny ? la : R(1)));
        B.vertex(edge_start(k), p);
        B.vertex(edge_end(k), q);
        sub3(q, p, d);
        const R lb = dot3(d, d);
        S.putv(3 + k, lb);
        S.putv(9 + k, rcpv(lb > tiny ? lb : R(1)));
    }
    // rows 6 + 3 ka + kb: A's edge ka by runtime index (one address per
    // outer step), B's three edges at compile-time offsets
#pragma unroll 1
    for (int ka = 0; ka < 3; ++ka) {
        R p1[3], q1[3];
        A.vertex(edge_start(ka), p1);
        A.vertex(edge_end(ka), q1);
        const R rak = S.getv(6 + ka), lak = S.getv(ka);
#pragma unroll
        for (int kb = 0; kb < 3; ++kb) {
            // (keeps the unrolled tests from being interleaved: the next
            // test's loads stay behind this point, so one test is live at a time)
            if (!TC_P2_INTERLEAVE) asm volatile("" ::: "memory");
            R p2[3], q2[3], s, t, d2;
            B.vertex(edge_start(kb), p2);
            B.vertex(edge_end(kb), q2);
            const R rbk = S.getv(9 + kb), lbk = S.getv(3 + kb);
            const int code = segment_params(p1, q1, p2, q2, rak, rbk, lak, lbk, s, t, d2);
            if (d2 < best) { best = d2; best_row = 6 + 3 * ka + kb; best_code = code; bp1 = s; bp2 = t; }
        }
    }
    o.ids = (uint32_t)best_row | ((uint32_t)best_code << 8);
    if (ids_only) return;
    o.distance = sqrtv(best);
    if (best_row < 3) {
        A.vertex(best_row, o.pa);
        bary_point_t(B, bp1, bp2, o.pb);
        o.ba[0] = (best_row == 1) ? R(1) : R(0);
        o.ba[1] = (best_row == 2) ? R(1) : R(0);
        o.bb[0] = bp1; o.bb[1] = bp2;
    } else if (best_row < 6) {
        bary_point_t(A, bp1, bp2, o.pa);
        B.vertex(best_row - 3, o.pb);
        o.ba[0] = bp1; o.ba[1] = bp2;
        o.bb[0] = (best_row == 4) ? R(1) : R(0);
        o.bb[1] = (best_row == 5) ? R(1) : R(0);
    } else {
        const int ka = (best_row - 6) / 3, kb = (best_row - 6) % 3;
        R p1[3], q1[3], p2[3], q2[3];
        A.vertex(edge_start(ka), p1);
        A.vertex(edge_end(ka), q1);
        B.vertex(edge_start(kb), p2);
        B.vertex(edge_end(kb), q2);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            o.pa[i] = p1[i] + bp1 * (q1[i] - p1[i]);
            o.pb[i] = p2[i] + bp2 * (q2[i] - p2[i]);
        }
        edge_bary(ka, bp1, o.ba);
        edge_bary(kb, bp2, o.bb);
    }
    o.kind = (o.distance <= R(T(2)) * eps) ? KIND_CONTACT : KIND_NO_CONTACT;
    o.ids |= 255u << 16;
}

// Phase 2 entry (the pair stays in its shared-memory slot: copying it into
// registers first measured slower -- spills at the 128-register cap).
template <class R, class Tri>
__device__ __forceinline__ void comparison_phase2(const Tri& A, const Tri& B, R eps, bool ids_only, Rec<R>& o,
                                                  Scratch<R> S) {
    comparison_phase2_impl(A, B, eps, ids_only, o, S);
}

// RK/kernels.py:417-431 _penalty_value, summed left to right.
template <class R>
__device__ __forceinline__ R penalty(const R* x, R alpha) {
    const R z = R(0), one = R(1);
    R p = maxv(z, x[0] - one);
    p = p + maxv(z, -x[0]);
    p = p + maxv(z, x[1] - one);
    p = p + maxv(z, -x[1]);
    p = p + maxv(z, (x[0] + x[1]) - one);
    p = p + maxv(z, x[2] - one);
    p = p + maxv(z, -x[2]);
    p = p + maxv(z, x[3] - one);
    p = p + maxv(z, -x[3]);
    p = p + maxv(z, (x[2] + x[3]) - one);
    return alpha * p;
}

// midpoint = A0 + x0*e1a + x1*e2a - 0.5*d   (RK/kernels.py:521,548)
template <class R>
__device__ __forceinline__ void contact_mid(const R* A0, const R* x, const R* e1a, const R* e2a, const R* d, R* m) {
    const R half = R(typename Store<R>::type(0.5));
#pragma unroll
    for (int i = 0; i < 3; ++i) m[i] = ((A0[i] + x[0] * e1a[i]) + x[1] * e2a[i]) - half * d[i];
}

// Clips.  A double compare (DSETP) plus its dependent select costs ~15-25
// cycles of latency on B200 (tools/latency_probe.cu: DFMA + one min = 24
// cycles, DFMA + a two-sided fmax/fmin clip = 58), and the iterative kernel
// is one long chain of clips.  The lower clip at 0 is a sign-bit test on the
// integer pipe.  Doing the upper compare on 64-bit integer patterns too (for
// non-negative IEEE values the patterns order like the values) measured
// slower: more instructions (two ISETP + selects) and a longer chain, and
// the sweep is issue-bound.  The fp32 clips are integer clips.
// NaN inputs are not supported.
//
// clip0_hi(x, hi) == np.clip(x, 0, hi) bit for bit for hi >= +0 (x <= 0,
// including -0, gives +0; ties give hi), so strict mode uses it too.
__device__ __forceinline__ double negv(double x) {
    // (ptxas turns this into a DADD; forcing an integer xor through PTX
    // measured slower: the extra register moves cost more than the DADD)
    return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}
__device__ __forceinline__ float negv(float x) { return __int_as_float(__float_as_int(x) ^ (int)0x80000000); }
template <typename T>
__device__ __forceinline__ Strict<T> negv(Strict<T> x) { return -x; }

__device__ __forceinline__ double clip0_hi(double x, double hi) {
    // both tests read the unclipped x, so they issue in parallel (one compare
    // latency on the chain instead of two); equal to min(max(x, 0), hi) for
    // hi >= +0, including signed zeros
    const bool neg = __double2hiint(x) < 0;
    const double r = (x < hi) ? x : hi;
    return neg ? 0.0 : r;
}
__device__ __forceinline__ float clip0_hi(float x, float hi) {
    int xb = __float_as_int(x);
    const int hb = __float_as_int(hi);
    xb = (xb < 0) ? 0 : xb;
    return __int_as_float(xb < hb ? xb : hb);
}
template <typename T>
__device__ __forceinline__ Strict<T> clip0_hi(Strict<T> x, Strict<T> hi) { return clip0_hi(x.v, hi.v); }

// Fast build's coordinate clip.  With TC_LOWCLIP_IMNMX the lower clip is one
// integer max on the high word (a negative x becomes +0 in the high word with
// its low word kept: a positive denormal below 2^-1022 instead of +0, which
// every later use rounds away), then the upper clip's compare and select:
// 5 issue slots instead of 7 (tools/sweep_probe2.cu: 147 -> 142 cycles per
// warp-sweep).  Not bitwise: strict mode keeps clip0_hi.
#ifndef TC_UPCLIP_INT
#define TC_UPCLIP_INT 0
#endif
// Box-mode slide as one one-sided clip (GramSolver::slide_one): fp64 hybrid
// -1.1 % (one DSETP and a select pair less per slide); fp32, whose clips are
// single FMNMX instructions, +1.8 %: on for double only.
#ifndef TC_SLIDE_ONE_F64
#define TC_SLIDE_ONE_F64 1
#endif
#ifndef TC_SLIDE_ONE_F32
#define TC_SLIDE_ONE_F32 0
#endif
#ifndef TC_LOWCLIP_IMNMX
#define TC_LOWCLIP_IMNMX 1
#endif
__device__ __forceinline__ double clip0_hi_fast(double x, double hi) {
#if TC_LOWCLIP_IMNMX
    const double m = __hiloint2double(max(__double2hiint(x), 0), __double2loint(x));
#if TC_UPCLIP_INT
    // m >= 0: the IEEE order is the unsigned order of the bit patterns (a hi
    // below 0 by an ulp keeps m); two integer compares instead of a DSETP
    return ((unsigned long long)__double_as_longlong(m) < (unsigned long long)__double_as_longlong(hi)) ? m : hi;
#else
    return (m < hi) ? m : hi;
#endif
#else
    return clip0_hi(x, hi);
#endif
}
// fp32 fast clips as float min/max (FMNMX): fewer and cheaper instructions
// than the integer clips (slides: 2 instead of 5); fp32 iterative -7.5 %,
// hybrid -4.8 % (tools/varbench.py).  A -0 iterate may appear (fmaxf of
// -0 and +0); it behaves as +0 everywhere downstream.
#ifndef TC_F32_FMNMX
#define TC_F32_FMNMX 1
#endif
__device__ __forceinline__ float clip0_hi_fast(float x, float hi) {
#if TC_F32_FMNMX
    return fminf(fmaxf(x, 0.0f), hi);
#else
    return clip0_hi(x, hi);
#endif
}

// clip(t, -xb, xa) for xa, xb >= 0 (the fast build's box mode): clip the
// magnitude against the bound on t's side, keep t's sign.
__device__ __forceinline__ double clip_sym(double t, double xb, double xa) {
    // independent compares of the unclipped t against both bounds
    const double lo = negv(xb);
    const bool below = !(t > lo), above = !(t < xa);
    return below ? lo : (above ? xa : t);
}
__device__ __forceinline__ float clip_sym(float t, float xb, float xa) {
#if TC_F32_FMNMX
    return fmaxf(fminf(t, xa), -xb);
#endif
    const int tb = __float_as_int(t);
    const int mag = tb & 0x7FFFFFFF;
    const int lim = (tb < 0) ? __float_as_int(xb) : __float_as_int(xa);
    const int r = mag < lim ? mag : lim;
    return __int_as_float(r | (tb & (int)0x80000000));
}
template <typename T>
__device__ __forceinline__ Strict<T> clip_sym(Strict<T> t, Strict<T> xb, Strict<T> xa) { return clip_sym(t.v, xb.v, xa.v); }


// np.maximum(0, v) for a v that is never -0: +0 when the sign bit is set
// (a sign test on the integer pipe instead of a DSETP and two selects).
__device__ __forceinline__ double max0_sign(double v) { return __double2hiint(v) < 0 ? 0.0 : v; }
__device__ __forceinline__ float max0_sign(float v) { return __float_as_int(v) < 0 ? 0.0f : v; }
template <typename T>
__device__ __forceinline__ Strict<T> max0_sign(Strict<T> v) { return max0_sign(v.v); }

// One coordinate substep (RK/kernels.py:531-536): preconditioned descent on
// the quadratic part, then the clip to [0, max(0, 1 - max(x_partner, 0))].
// BOX (start_coord in [0, 1]): every iterate stays >= 0 -- a clip returns +0
// or a value in (0, hi] with hi >= +0, and a slide's t lies in [-xb, xa], so
// xa - t and xb + t round to values >= 0 -- hence max(x_partner, 0) is
// x_partner bit for bit and the strict build drops it; 1 - x_partner can
// still round below 0 (x_a + x_b may exceed 1 by an ulp after a slide), so
// the outer max stays (as a sign test: 1 - x is never -0).  The fast build
// also drops the outer max (x_k + x_partner <= 1 up to an ulp).
template <bool BOX, class R>
__device__ __forceinline__ void coord_step(R& xk, R xp, const R* e, R den, R rcp, R* d) {
    R target = xk - divr(dot3(d, e), den, rcp);
    if (!IsStrict<R>::value && BOX) target = clip0_hi(target, R(1) - xp);
    else if (BOX) target = clip0_hi(target, max0_sign(R(1) - xp));
    else target = clip0_hi(target, maxv(R(0), R(1) - maxv(xp, R(0))));
    const R step = target - xk;
    xk = target;
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = d[i] + step * e[i];
}

// Slide along the triangle's third edge (RK/kernels.py:537-546).
template <bool BOX, class R>
__device__ __forceinline__ void slide_step(R& xa, R& xb, const R* e3, R den3, R rcp3, R* d) {
    R t = divr(-dot3(d, e3), den3, rcp3);
    if (!IsStrict<R>::value && BOX) t = clip_sym(t, xb, xa);
    else if (BOX) t = clipv(t, -xb, xa);  // xa, xb >= 0: the max() are identities
    else t = clipv(t, -maxv(xb, R(0)), maxv(xa, R(0)));
    xa = xa - t;
    xb = xb + t;
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = d[i] + t * e3[i];
}

// RK/kernels.py:447-565 iterative_batch for one pair.  Only the functional
// and contact midpoint of the last two sweeps are live in the reference's
// settle test, so they are evaluated there only (same values, same ops).
// The loop carries only the edge directions, reciprocals, x and d; the base
// vertices A0, B0 are re-read through `reload` (an L1/L2 hit) after the
// first n-1 sweeps, which keeps the sweep loop's register footprint small.
template <bool BOX, class R, class Reload>
__device__ __forceinline__ void iterative_pair(const R* A, const R* B, R eps, const KP<R>& kp, Rec<R>& o,
                                               Reload reload) {
    using T = typename Store<R>::type;
    const R tiny = R(Tiny<R>::v);
    const R half = R(T(0.5));
    R e1a[3], e2a[3], ne1b[3], ne2b[3], e3a[3], ne3b[3], d[3];
    sub3(A + 3, A, e1a);
    sub3(A + 6, A, e2a);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const R e1b = B[3 + i] - B[i];
        const R e2b = B[6 + i] - B[i];
        ne1b[i] = -e1b;
        ne2b[i] = -e2b;
        e3a[i] = e2a[i] - e1a[i];
        ne3b[i] = -(e2b - e1b);
    }
    const R sq = maxv(max_sq_edge(A), max_sq_edge(B));   // _pair_max_sq_edge
    const R alpha_it = kp.alpha_it * sq;
    const R alpha_reg = kp.alpha_reg * sq;
    const R den0 = maxv(dot3(e1a, e1a) + alpha_reg, tiny);
    const R den1 = maxv(dot3(e2a, e2a) + alpha_reg, tiny);
    const R den2 = maxv(dot3(ne1b, ne1b) + alpha_reg, tiny);
    const R den3 = maxv(dot3(ne2b, ne2b) + alpha_reg, tiny);
    const R den3a = maxv(dot3(e3a, e3a) + alpha_reg, tiny);
    const R den3b = maxv(dot3(ne3b, ne3b) + alpha_reg, tiny);
    const R r0 = rcpv(den0), r1 = rcpv(den1), r2 = rcpv(den2), r3 = rcpv(den3);
    const R r3a = rcpv(den3a), r3b = rcpv(den3b);

    R x[4] = {kp.start_coord, kp.start_coord, kp.start_coord, kp.start_coord};
    // d = base + x0*e1a + x1*e2a - x2*e1b - x3*e2b  (diff_vec, RK/kernels.py:501-508)
#pragma unroll
    for (int i = 0; i < 3; ++i)
        d[i] = ((((A[i] - B[i]) + x[0] * e1a[i]) + x[1] * e2a[i]) - x[2] * (-ne1b[i])) - x[3] * (-ne2b[i]);

    const int n_it = kp.n_iterative;
    auto sweep = [&]() {
        coord_step<BOX>(x[0], x[1], e1a, den0, r0, d);
        coord_step<BOX>(x[1], x[0], e2a, den1, r1, d);
        slide_step<BOX>(x[0], x[1], e3a, den3a, r3a, d);
        coord_step<BOX>(x[2], x[3], ne1b, den2, r2, d);
        coord_step<BOX>(x[3], x[2], ne2b, den3, r3, d);
        slide_step<BOX>(x[2], x[3], ne3b, den3b, r3b, d);
    };
#pragma unroll 1
    for (int it = 0; it < n_it - 1; ++it) sweep();
    R A0[3], B0[3];
    reload(A0, B0);
    const R j_old = half * dot3(d, d) + penalty(x, alpha_it);
    R mid_old[3];
    contact_mid(A0, x, e1a, e2a, d, mid_old);
    sweep();
    const R dd = dot3(d, d);
    const R j_total = half * dd + penalty(x, alpha_it);
    R mv[3];
    contact_mid(A0, x, e1a, e2a, d, mv);
#pragma unroll
    for (int i = 0; i < 3; ++i) mv[i] = mv[i] - mid_old[i];
    const R move = sqrtv(norm3_sq_sum(mv));
    const R jh = half * dd;
    const bool settled = (absv(j_total - j_old) <= kp.c_factor * eps) && (move <= kp.move_factor * eps);
    const bool contact = settled && (jh <= (R(T(2)) * eps) * eps);
    o.kind = contact ? KIND_CONTACT : (settled ? KIND_NO_CONTACT : KIND_NOT_TERMINATED);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        o.pa[i] = (A0[i] + x[0] * e1a[i]) + x[1] * e2a[i];
        o.pb[i] = (B0[i] + x[2] * (-ne1b[i])) + x[3] * (-ne2b[i]);
    }
    o.distance = sqrtv(R(T(2)) * jh);
    o.ba[0] = x[0]; o.ba[1] = x[1];
    o.bb[0] = x[2]; o.bb[1] = x[3];
    o.ids = 0x00FFFFFFu | ((uint32_t)((settled ? FLAG_SETTLED : 0u) | (contact ? FLAG_ITER_CONTACT : 0u)) << 24);
}

// Fast build of RK/kernels.py:447-565: the same coordinate / slide sweep,
// but the gradient components g_k = d . E_k are carried instead of d.  A
// step of size s along direction E_j changes every g_k by s * (E_j . E_k),
// so with the 4x4 Gram matrix of the base directions (E0 = e1a, E1 = e2a,
// E3 = -e1b, E4 = -e2b) and the slide directions' products
// (e3a . E_k = SA_k, -e3b . E_k = SB_k) a substep is one FMA for the target,
// the clip, and four independent FMAs -- a third of the dependent latency
// of re-dotting d, and fewer FP64 instructions (52 vs 66 per sweep).  The
// slide gradients follow from e3a = E1 - E0 and -e3b = E4 - E3.  d itself
// is rebuilt exactly from x where the settle test needs it.  Equal to the
// reference up to rounding (checked within the north-star tolerance).
// Packed fp32 pairs (sm_100 FFMA2: one instruction, two IEEE fp32 FMAs on an
// aligned register pair; a scalar operand is broadcast by an operand modifier).
// TC_F32_FFMA2: the fast fp32 sweep updates the gradient pairs (g0, g1) and
// (g3, g4) with two FFMA2 instead of four FFMA per substep -- the same
// roundings (bitwise equal results, tools/libcmp.py), 61 -> 53 instructions per
// sweep.  Measured: iterative fp32 -2.4 %, hybrid fp32 +0.2 % (an FFMA2 costs
// the issue slots of the two FFMAs it replaces): off.
#ifndef TC_F32_FFMA2
#define TC_F32_FFMA2 0
#endif
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pack2(float a, float b) {
    f32x2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(f32x2_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// (g.x + s * m.x, g.y + s * m.y)
__device__ __forceinline__ f32x2_t fma2s(float s, f32x2_t m, f32x2_t g) {
    f32x2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pack2(s, s)), "l"(m), "l"(g));
    return r;
}
template <class R> struct IsF32 { static constexpr bool value = false; };
template <> struct IsF32<float> { static constexpr bool value = true; };

template <bool BOX, class R>
struct GramSolver {
    R G00, G01, G03, G04, G11, G13, G14, G33, G34, G44, SA0, SA1, SA3, SA4, SB0, SB1, SB3, SB4;
    R r0, r1, r2, r3, r3a, r3b;
    R x0, x1, x2, x3;
    R g0, g1, g3, g4;

    // Setup.  The slide directions' products come from the Gram matrix
    // (e3a = E1 - E0: SA_k = G1k - G0k; -e3b = E4 - E3: SB_k = G4k - G3k);
    // their squared lengths are dotted directly (they set the slide step
    // size).  _pair_max_sq_edge (RK/kernels.py:409-414) is the max over the
    // six squared edges G00, G11, |e3a|^2, G33, G44, |e3b|^2, and the TINY
    // floor of the denominators (RK/kernels.py:490) is applied once to the
    // regulariser (equal unless alpha_reg * sq < 1e-30).
    __device__ __forceinline__ void init(const R* A, const R* B, const KP<R>& kp) {
        const R tiny = R(Tiny<R>::v);
        x0 = x1 = x2 = x3 = kp.start_coord;
        R E0[3], E1[3], E3[3], E4[3], SA[3], SB[3], d[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            E0[i] = A[3 + i] - A[i];
            E1[i] = A[6 + i] - A[i];
            E3[i] = B[i] - B[3 + i];
            E4[i] = B[i] - B[6 + i];
            SA[i] = E1[i] - E0[i];
            SB[i] = E4[i] - E3[i];
        }
        G00 = dot3(E0, E0); G01 = dot3(E0, E1); G03 = dot3(E0, E3); G04 = dot3(E0, E4);
        G11 = dot3(E1, E1); G13 = dot3(E1, E3); G14 = dot3(E1, E4);
        G33 = dot3(E3, E3); G34 = dot3(E3, E4); G44 = dot3(E4, E4);
        SA0 = G01 - G00; SA1 = G11 - G01; SA3 = G13 - G03; SA4 = G14 - G04;
        SB0 = G04 - G03; SB1 = G14 - G13; SB3 = G34 - G33; SB4 = G44 - G34;
        const R qa = dot3(SA, SA), qb = dot3(SB, SB);
        const R sq = maxv(maxv(maxv(G00, G11), qa), maxv(maxv(G33, G44), qb));
        const R areg = maxv(kp.alpha_reg * sq, tiny);
        r0 = rcpv(G00 + areg);
        r1 = rcpv(G11 + areg);
        r2 = rcpv(G33 + areg);
        r3 = rcpv(G44 + areg);
        r3a = rcpv(qa + areg);
        r3b = rcpv(qb + areg);
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = (A[i] - B[i]) + x0 * E0[i] + x1 * E1[i] + x2 * E3[i] + x3 * E4[i];
        g0 = dot3(d, E0); g1 = dot3(d, E1); g3 = dot3(d, E3); g4 = dot3(d, E4);
    }

    // BOX (start_coord in [0, 1], the usual case): the iterates never leave
    // the box, so the inner max() of the clips are identities (coord_step)
    __device__ __forceinline__ R hi_of(R xp) const { return BOX ? R(1) - xp : maxv(R(0), R(1) - maxv(xp, R(0))); }

    // Box-mode slide as ONE one-sided clip (TC_SLIDE_ONE_F64 / _F32): the slide moves
    // x_a by -t and x_b by +t with t in [-x_b, x_a], i.e. x_a's target
    // x_a + q (q = (g_b - g_a) r, the negated unclipped t) is clipped to
    // [0, x_a + x_b] and x_b takes the rest of the sum: one lower clip on the
    // integer pipe and one compare instead of two compares and four selects.
    // s = the step of x_a (= -t); the caller updates g by -s * S_k.
    static constexpr bool slide_one_on =
        !IsStrict<R>::value && (sizeof(typename Store<R>::type) == 8 ? TC_SLIDE_ONE_F64 : TC_SLIDE_ONE_F32);
    __device__ __forceinline__ static void slide_one(R& xa, R& xb, R q, R& s) {
        const R h = xa + xb;
        const R t = clip0_hi_fast(xa + q, h);
        s = t - xa;
        xa = t;
        xb = h - t;
    }

    __device__ __forceinline__ void sweep() {
        if constexpr (IsF32<R>::value && TC_F32_FFMA2) sweep_f32x2();
        else sweep_scalar();
    }

    // fp32 fast: the sweep with the gradient components as two packed pairs
    // (same operations and roundings as sweep_scalar)
    __device__ __forceinline__ void sweep_f32x2() {
        float t, s, ga, gb;
        f32x2_t g01 = pack2(float(g0), float(g1)), g34 = pack2(float(g3), float(g4));
        const float X0 = float(x0), X1 = float(x1), X2 = float(x2), X3 = float(x3);
        float y0 = X0, y1 = X1, y2 = X2, y3 = X3;
        auto hi = [&](float xp) { return hi_of(xp); };
        auto sclip = [](float t_, float xb, float xa) {
            return BOX ? clip_sym(t_, xb, xa) : clipv(t_, -maxv(xb, 0.0f), maxv(xa, 0.0f));
        };
        unpack2(g01, ga, gb);
        t = clip0_hi_fast(y0 - ga * float(r0), hi(y1));
        s = t - y0; y0 = t;
        g01 = fma2s(s, pack2(float(G00), float(G01)), g01); g34 = fma2s(s, pack2(float(G03), float(G04)), g34);
        unpack2(g01, ga, gb);
        t = clip0_hi_fast(y1 - gb * float(r1), hi(y0));
        s = t - y1; y1 = t;
        g01 = fma2s(s, pack2(float(G01), float(G11)), g01); g34 = fma2s(s, pack2(float(G13), float(G14)), g34);
        unpack2(g01, ga, gb);
        t = -(gb - ga) * float(r3a);
        t = sclip(t, y1, y0);
        y0 = y0 - t; y1 = y1 + t;
        g01 = fma2s(t, pack2(float(SA0), float(SA1)), g01); g34 = fma2s(t, pack2(float(SA3), float(SA4)), g34);
        unpack2(g34, ga, gb);
        t = clip0_hi_fast(y2 - ga * float(r2), hi(y3));
        s = t - y2; y2 = t;
        g01 = fma2s(s, pack2(float(G03), float(G13)), g01); g34 = fma2s(s, pack2(float(G33), float(G34)), g34);
        unpack2(g34, ga, gb);
        t = clip0_hi_fast(y3 - gb * float(r3), hi(y2));
        s = t - y3; y3 = t;
        g01 = fma2s(s, pack2(float(G04), float(G14)), g01); g34 = fma2s(s, pack2(float(G34), float(G44)), g34);
        unpack2(g34, ga, gb);
        t = -(gb - ga) * float(r3b);
        t = sclip(t, y3, y2);
        y2 = y2 - t; y3 = y3 + t;
        g01 = fma2s(t, pack2(float(SB0), float(SB1)), g01); g34 = fma2s(t, pack2(float(SB3), float(SB4)), g34);
        x0 = R(y0); x1 = R(y1); x2 = R(y2); x3 = R(y3);
        unpack2(g01, ga, gb); g0 = R(ga); g1 = R(gb);
        unpack2(g34, ga, gb); g3 = R(ga); g4 = R(gb);
    }

    __device__ __forceinline__ void sweep_scalar() {
        R t, s;
        t = clip0_hi_fast(x0 - g0 * r0, hi_of(x1));
        s = t - x0; x0 = t;
        g0 += s * G00; g1 += s * G01; g3 += s * G03; g4 += s * G04;
        t = clip0_hi_fast(x1 - g1 * r1, hi_of(x0));
        s = t - x1; x1 = t;
        g0 += s * G01; g1 += s * G11; g3 += s * G13; g4 += s * G14;
        if (slide_one_on && BOX) {
            slide_one(x0, x1, (g1 - g0) * r3a, s);
            g0 -= s * SA0; g1 -= s * SA1; g3 -= s * SA3; g4 -= s * SA4;
        } else {
            t = -(g1 - g0) * r3a;
            t = BOX ? clip_sym(t, x1, x0) : clipv(t, -maxv(x1, R(0)), maxv(x0, R(0)));
            x0 = x0 - t; x1 = x1 + t;
            g0 += t * SA0; g1 += t * SA1; g3 += t * SA3; g4 += t * SA4;
        }
        t = clip0_hi_fast(x2 - g3 * r2, hi_of(x3));
        s = t - x2; x2 = t;
        g0 += s * G03; g1 += s * G13; g3 += s * G33; g4 += s * G34;
        t = clip0_hi_fast(x3 - g4 * r3, hi_of(x2));
        s = t - x3; x3 = t;
        g0 += s * G04; g1 += s * G14; g3 += s * G34; g4 += s * G44;
        if (slide_one_on && BOX) {
            slide_one(x2, x3, (g4 - g3) * r3b, s);
            g0 -= s * SB0; g1 -= s * SB1; g3 -= s * SB3; g4 -= s * SB4;
        } else {
            t = -(g4 - g3) * r3b;
            t = BOX ? clip_sym(t, x3, x2) : clipv(t, -maxv(x3, R(0)), maxv(x2, R(0)));
            x2 = x2 - t; x3 = x3 + t;
            g0 += t * SB0; g1 += t * SB1; g3 += t * SB3; g4 += t * SB4;
        }
    }

    // Epilogue.  The pair is re-read (shared-memory copy) where needed, so
    // nothing but x, g and the Gram terms is live across a sweep.  Both
    // points come from the barycentric weights, pa = (1 - x0 - x1) A0 +
    // x0 A1 + x1 A2 (likewise pb), d = pa - pb, and the contact midpoint
    // A0 + x0 e1a + x1 e2a - d/2 of RK/kernels.py:521,548 is (pa + pb) / 2,
    // so the move between the last two sweeps is |S - S_old| / 2 with
    // S = pa + pb (tested squared: |S - S_old|^2 <= 4 (mf eps)^2).  The penalty weight re-derives _pair_max_sq_edge from the
    // Gram terms (|e3a|^2 = SA1 - SA0, |e3b|^2 = SB4 - SB3).
    struct Pre { R x_old[4], j_old, s_old[3], eps, alpha_it; };

    __device__ __forceinline__ R alpha_it(const KP<R>& kp) const {
        const R sq = maxv(maxv(maxv(G00, G11), SA1 - SA0), maxv(maxv(G33, G44), SB4 - SB3));
        return kp.alpha_it * sq;
    }

    // RK/kernels.py:417-431.  In BOX mode the iterates satisfy x >= 0 exactly
    // (clips and slides never produce a negative coordinate) and x <= 1,
    // x_a + x_b <= 1 up to a few ulps (each clip bounds a coordinate by
    // 1 - partner), so the penalty is 0 or alpha * O(ulp): below the
    // resolution of the settle test, and it is dropped.
    __device__ __forceinline__ R penalty_x(R alpha) const {
        if (BOX) return R(0);
        const R xs[4] = {x0, x1, x2, x3};
        return penalty(xs, alpha);
    }

    template <class Reload>
    __device__ __forceinline__ void points(Reload& reload, R* pa, R* pb) const {
        R A[9], B[9];
        reload(A, B);
        const R wa = (R(1) - x0) - x1, wb = (R(1) - x2) - x3;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            pa[i] = (wa * A[i] + x0 * A[3 + i]) + x1 * A[6 + i];
            pb[i] = (wb * B[i] + x2 * B[3 + i]) + x3 * B[6 + i];
        }
    }

    template <class Reload, class EpsFn>
    __device__ __forceinline__ void prelast(Reload& reload, EpsFn& eps_fn, const KP<R>& kp, Pre& pre) const {
        pre.eps = eps_fn();
        pre.x_old[0] = x0; pre.x_old[1] = x1; pre.x_old[2] = x2; pre.x_old[3] = x3;
        if (BOX) return;   // finish() works from the last sweep's dx and the Gram terms
        R pa[3], pb[3], d[3];
        points(reload, pa, pb);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            d[i] = pa[i] - pb[i];
            pre.s_old[i] = pa[i] + pb[i];
        }
        pre.alpha_it = alpha_it(kp);
        pre.j_old = R(typename Store<R>::type(0.5)) * dot3(d, d) + penalty_x(pre.alpha_it);
    }

    template <class Reload>
    __device__ __forceinline__ void finish(Reload& reload, const KP<R>& kp, const Pre& pre, Rec<R>& o) const {
        using T = typename Store<R>::type;
        const R half = R(T(0.5));
        R pa[3], pb[3], d[3];
        points(reload, pa, pb);
#pragma unroll
        for (int i = 0; i < 3; ++i) d[i] = pa[i] - pb[i];
        const R dd = dot3(d, d);
        const R jh = half * dd;
        const R eps = pre.eps;
        R dj, mv2;
        if (BOX) {
            // Last sweep's step dx = x - x_old: d moved by delta = sum dx_k E_k
            // (E0, E1, E3, E4 as in init), so with g_k = d.E_k now,
            //   J - J_old = sum dx_k g_k - |delta|^2 / 2,
            // and S = pa + pb moved by dx0 E0 + dx1 E1 - dx2 E3 - dx3 E4;
            // both squared lengths are quadratic forms in the Gram terms
            // (qa, qb within A and B, xab between them).
            const R e0 = x0 - pre.x_old[0], e1 = x1 - pre.x_old[1];
            const R e2 = x2 - pre.x_old[2], e3 = x3 - pre.x_old[3];
            const R lin = ((e0 * g0 + e1 * g1) + e2 * g3) + e3 * g4;
            const R qa = e0 * (e0 * G00 + R(T(2)) * (e1 * G01)) + e1 * (e1 * G11);
            const R qb = e2 * (e2 * G33 + R(T(2)) * (e3 * G34)) + e3 * (e3 * G44);
            const R xab = e0 * (e2 * G03 + e3 * G04) + e1 * (e2 * G13 + e3 * G14);
            const R qq = qa + qb;
            dj = lin - half * (qq + R(T(2)) * xab);
            mv2 = qq - R(T(2)) * xab;
        } else {
            R mv[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) mv[i] = (pa[i] + pb[i]) - pre.s_old[i];
            dj = (jh + penalty_x(pre.alpha_it)) - pre.j_old;
            mv2 = dot3(mv, mv);
        }
        // move = |S - S_old| / 2 <= mf * eps, compared squared (no sqrt)
        const R mlim = kp.move_factor * eps;
        const bool settled = (absv(dj) <= kp.c_factor * eps) && (mv2 <= R(T(4)) * (mlim * mlim));
        const bool contact = settled && (jh <= (R(T(2)) * eps) * eps);
        o.kind = contact ? KIND_CONTACT : (settled ? KIND_NO_CONTACT : KIND_NOT_TERMINATED);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            o.pa[i] = pa[i];
            o.pb[i] = pb[i];
        }
        o.distance = sqrtv(dd);   // sqrt(2 * jh): halving and doubling are exact
        o.ba[0] = x0; o.ba[1] = x1;
        o.bb[0] = x2; o.bb[1] = x3;
        o.ids = 0x00FFFFFFu | ((uint32_t)((settled ? FLAG_SETTLED : 0u) | (contact ? FLAG_ITER_CONTACT : 0u)) << 24);
    }
};

template <bool BOX, class R, class Reload, class EpsFn>
__device__ __forceinline__ void iterative_pair_gram(const R* A, const R* B, const KP<R>& kp, Rec<R>& o,
                                                    Reload reload, EpsFn eps_fn) {
    GramSolver<BOX, R> gs;
    gs.init(A, B, kp);
#pragma unroll 1
    for (int it = 0; it < kp.n_iterative - 1; ++it) gs.sweep();
    typename GramSolver<BOX, R>::Pre pre;
    gs.prelast(reload, eps_fn, kp, pre);
    gs.sweep();
    gs.finish(reload, kp, pre, o);
}

}  // namespace tc
