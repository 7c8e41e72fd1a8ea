// tc_pair.cuh -- per-pair device code of the three reference kernels.
//
// One triangle pair per thread, everything in registers.  Each function
// restates one reference function (RK = /root/reference/pkg/src/tricontact)
// in the reference's operation order; R is an arithmetic policy from
// tc_math.cuh (Strict<T> = bit-exact, T = FMA-contracted).
#pragma once
#include "tc_math.cuh"

namespace tc {

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

// RK/geometry.py:68-75 degenerate_mask, rel_tol = 1e-12
template <class R>
__device__ __forceinline__ bool degenerate_tri(const R* t) {
    using T = typename Store<R>::type;
    R e1[3], e2[3], c[3];
    sub3(t + 3, t, e1);
    sub3(t + 6, t, e2);
    cross3(e1, e2, c);
    R sq_area = R(T(0.25)) * dot3(c, c);
    R L = max_sq_edge(t);
    R thr = R(T(1e-12)) * L;
    thr = thr * L;
    return (L == R(0)) || (sq_area < thr);
}

// RK/kernels.py:157-221 closest_point_triangle_batch for one point.
// Returns the claimed region in claim order 0 VA, 1 VB, 2 EAB, 3 VC, 4 EAC,
// 5 EBC, 6 interior; u, w are the weights along ab, ac.
template <class R>
__device__ __forceinline__ int closest_point_triangle(const R* p, const R* tri, R* closest, R& u, R& w) {
    const R* a = tri;
    const R* b = tri + 3;
    const R* c = tri + 6;
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
    const R vc = d1 * d4 - d3 * d2;
    const R vb = d5 * d2 - d1 * d6;
    const R va = d3 * d6 - d5 * d4;
    u = R(0);
    w = R(0);
    int region;
    if (d1 <= R(0) && d2 <= R(0)) {
        region = 0;
    } else if (d3 >= R(0) && d4 <= d3) {
        region = 1;
        u = R(1);
    } else if (vc <= R(0) && d1 >= R(0) && d3 <= R(0)) {
        region = 2;
        const R den = d1 - d3;
        u = d1 / (den == R(0) ? R(1) : den);
    } else if (d6 >= R(0) && d5 <= d6) {
        region = 3;
        w = R(1);
    } else if (vb <= R(0) && d2 >= R(0) && d6 <= R(0)) {
        region = 4;
        const R den = d2 - d6;
        w = d2 / (den == R(0) ? R(1) : den);
    } else if (va <= R(0) && (d4 - d3) >= R(0) && (d5 - d6) >= R(0)) {
        region = 5;
        const R n1 = d4 - d3;
        const R den = n1 + (d5 - d6);
        const R t = n1 / (den == R(0) ? R(1) : den);
        u = R(1) - t;
        w = t;
    } else {
        region = 6;
        R den = (va + vb) + vc;
        den = (den == R(0)) ? R(1) : den;
        u = vb / den;
        w = vc / den;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) closest[i] = (a[i] + u * ab[i]) + w * ac[i];
    return region;
}

// RK/kernels.py:224-252 _closest_segment_segment.  Branch code: bit0 = s
// from the 2x2 solve (denom > TINY), bit1 = t < 0, bit2 = t > 1.
template <class R>
__device__ __forceinline__ int segment_segment(const R* p1, const R* q1, const R* p2, const R* q2, R& s, R& t,
                                               R* c1, R* c2) {
    const R tiny = R(Tiny<R>::v);
    R d1[3], d2[3], r[3];
    sub3(q1, p1, d1);
    sub3(q2, p2, d2);
    sub3(p1, p2, r);
    const R a = dot3(d1, d1);
    const R e = dot3(d2, d2);
    const R f = dot3(d2, r);
    const R c = dot3(d1, r);
    const R b = dot3(d1, d2);
    const R denom = a * e - b * b;
    int code = 0;
    if (denom > tiny) {
        code = 1;
        s = clipv((b * f - c * e) / denom, R(0), R(1));
    } else {
        s = R(0);
    }
    t = (b * s + f) / ((e > tiny) ? e : R(1));
    const R a_safe = (a > tiny) ? a : R(1);
    if (t < R(0)) {
        code |= 2;
        s = clipv((-c) / a_safe, R(0), R(1));
    } else if (t > R(1)) {
        code |= 4;
        s = clipv((b - c) / a_safe, R(0), R(1));
    }
    t = clipv(t, R(0), R(1));
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        c1[i] = p1[i] + s * d1[i];
        c2[i] = p2[i] + t * d2[i];
    }
    return code;
}

// RK/kernels.py:269-298 _segment_triangle_crossings for one segment: proper
// crossing (strict dp*dq < 0) through the closed triangle.
template <class R>
__device__ __forceinline__ bool segment_crosses(const R* p, const R* q, const R* tri, R* x) {
    const R tiny = R(Tiny<R>::v);
    const R* a = tri;
    R u[3], v[3], nrm[3], t3[3];
    sub3(tri + 3, a, u);
    sub3(tri + 6, a, v);
    cross3(u, v, nrm);
    sub3(p, a, t3);
    const R dp = dot3(t3, nrm);
    sub3(q, a, t3);
    const R dq = dot3(t3, nrm);
    const bool crossing = (dp * dq) < R(0);
    const R denom = dp - dq;
    const R t = dp / (denom == R(0) ? R(1) : denom);
    sub3(q, p, t3);
#pragma unroll
    for (int i = 0; i < 3; ++i) x[i] = p[i] + t * t3[i];
    sub3(x, a, t3);
    const R uu = dot3(u, u);
    const R uv = dot3(u, v);
    const R vv = dot3(v, v);
    const R wu = dot3(t3, u);
    const R wv = dot3(t3, v);
    const R det = uu * vv - uv * uv;
    const R det_safe = (absv(det) > tiny) ? det : R(1);
    const R b1 = (vv * wu - uv * wv) / det_safe;
    const R b2 = (uu * wv - uv * wu) / det_safe;
    return crossing && (b1 >= R(0)) && (b2 >= R(0)) && ((b1 + b2) <= R(1));
}

__device__ __forceinline__ int edge_start(int k) { return k; }
__device__ __forceinline__ int edge_end(int k) { return k == 2 ? 0 : k + 1; }

// RK/kernels.py:261-266 _edge_bary
template <class R>
__device__ __forceinline__ void edge_bary(int k, R s, R* o) {
    if (k == 0) { o[0] = s; o[1] = R(0); }
    else if (k == 1) { o[0] = R(1) - s; o[1] = s; }
    else { o[0] = R(0); o[1] = R(1) - s; }
}

// RK/kernels.py:301-401 comparison_batch for one pair: 6 point-triangle +
// 9 segment-segment candidates with a running first-minimum (argmin ties go
// to the lowest row), then 6 edge-plane crossings; an intersecting pair
// reports distance 0 at the midpoint of its two farthest-apart crossing
// points (first argmax over the 6x6 grid).
template <class R>
__device__ __noinline__ void comparison_pair(const R* A, const R* B, R eps, Rec<R>& o) {
    R best = R(0), cl[3], diff[3], u, w, d2;
    int best_row = 0, best_code = 0;
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
        const R* pt = A + 3 * k;
        const int reg = closest_point_triangle(pt, B, cl, u, w);
        sub3(pt, cl, diff);
        d2 = dot3(diff, diff);
        if (k == 0 || d2 < best) {
            best = d2; best_row = k; best_code = reg;
#pragma unroll
            for (int i = 0; i < 3; ++i) { o.pa[i] = pt[i]; o.pb[i] = cl[i]; }
            o.ba[0] = (k == 1) ? R(1) : R(0);
            o.ba[1] = (k == 2) ? R(1) : R(0);
            o.bb[0] = u; o.bb[1] = w;
        }
    }
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
        const R* pt = B + 3 * k;
        const int reg = closest_point_triangle(pt, A, cl, u, w);
        sub3(pt, cl, diff);
        d2 = dot3(diff, diff);
        if (d2 < best) {
            best = d2; best_row = 3 + k; best_code = reg;
#pragma unroll
            for (int i = 0; i < 3; ++i) { o.pa[i] = cl[i]; o.pb[i] = pt[i]; }
            o.ba[0] = u; o.ba[1] = w;
            o.bb[0] = (k == 1) ? R(1) : R(0);
            o.bb[1] = (k == 2) ? R(1) : R(0);
        }
    }
#pragma unroll 1
    for (int row = 6; row < 15; ++row) {
        const int ka = (row - 6) / 3, kb = (row - 6) % 3;
        R s, t, c1[3], c2[3];
        const int code = segment_segment(A + 3 * edge_start(ka), A + 3 * edge_end(ka), B + 3 * edge_start(kb),
                                         B + 3 * edge_end(kb), s, t, c1, c2);
        sub3(c1, c2, diff);
        d2 = dot3(diff, diff);
        if (d2 < best) {
            best = d2; best_row = row; best_code = code;
#pragma unroll
            for (int i = 0; i < 3; ++i) { o.pa[i] = c1[i]; o.pb[i] = c2[i]; }
            edge_bary(ka, s, o.ba);
            edge_bary(kb, t, o.bb);
        }
    }
    o.distance = sqrtv(best);

    // six edge-to-plane tests (RK/kernels.py:364-375)
    R pts[6][3];
    uint32_t ok = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (segment_crosses(A + 3 * edge_start(k), A + 3 * edge_end(k), B, pts[k])) ok |= 1u << k;
        if (segment_crosses(B + 3 * edge_start(k), B + 3 * edge_end(k), A, pts[k + 3])) ok |= 8u << k;
    }
    uint32_t pair_id = 255;
    if (ok) {
        // first argmax over the row-major 6x6 grid; invalid pairs score -1
        R bestv = R(-1);
        int bi = 0;
#pragma unroll
        for (int i0 = 0; i0 < 6; ++i0) {
#pragma unroll
            for (int i1 = 0; i1 < 6; ++i1) {
                if (((ok >> i0) & 1u) && ((ok >> i1) & 1u)) {
                    sub3(pts[i0], pts[i1], diff);
                    const R v = dot3(diff, diff);
                    if (v > bestv) { bestv = v; bi = i0 * 6 + i1; }
                }
            }
        }
        const int i0 = bi / 6, i1 = bi % 6;
        R mid[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            R a0 = R(0), a1 = R(0);
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                if (j == i0) a0 = pts[j][i];
                if (j == i1) a1 = pts[j][i];
            }
            mid[i] = R(typename Store<R>::type(0.5)) * (a0 + a1);
        }
        pair_id = (uint32_t)bi;
        o.distance = R(0);
#pragma unroll
        for (int i = 0; i < 3; ++i) { o.pa[i] = mid[i]; o.pb[i] = mid[i]; }
        closest_point_triangle(mid, A, cl, o.ba[0], o.ba[1]);
        closest_point_triangle(mid, B, cl, o.bb[0], o.bb[1]);
    }
    o.kind = (o.distance <= R(typename Store<R>::type(2)) * eps) ? KIND_CONTACT : KIND_NO_CONTACT;
    o.ids = (uint32_t)best_row | ((uint32_t)best_code << 8) | (pair_id << 16) | ((ok ? FLAG_INTERSECT : 0u) << 24);
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

// One coordinate substep (RK/kernels.py:531-536): preconditioned descent on
// the quadratic part, then the clip to [0, max(0, 1 - max(x_partner, 0))].
template <class R>
__device__ __forceinline__ void coord_step(R& xk, R xp, const R* e, R den, R rcp, R* d) {
    R target = xk - divr(dot3(d, e), den, rcp);
    const R hi = maxv(R(0), R(1) - maxv(xp, R(0)));
    target = clipv(target, R(0), hi);
    const R step = target - xk;
    xk = target;
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = d[i] + step * e[i];
}

// Slide along the triangle's third edge (RK/kernels.py:537-546).
template <class R>
__device__ __forceinline__ void slide_step(R& xa, R& xb, const R* e3, R den3, R rcp3, R* d) {
    R t = divr(-dot3(d, e3), den3, rcp3);
    t = clipv(t, -maxv(xb, R(0)), maxv(xa, R(0)));
    xa = xa - t;
    xb = xb + t;
#pragma unroll
    for (int i = 0; i < 3; ++i) d[i] = d[i] + t * e3[i];
}

// RK/kernels.py:447-565 iterative_batch for one pair.  Only the functional
// and contact midpoint of the last two sweeps are live in the reference's
// settle test, so they are evaluated there only (same values, same ops).
template <class R>
__device__ __forceinline__ void iterative_pair(const R* A, const R* B, R eps, const KP<R>& kp, Rec<R>& o) {
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

    R j_old = R(0), mid_old[3];
    const int n_it = kp.n_iterative;
#pragma unroll 1
    for (int it = 0; it < n_it; ++it) {
        if (it == n_it - 1) {
            j_old = half * dot3(d, d) + penalty(x, alpha_it);
            contact_mid(A, x, e1a, e2a, d, mid_old);
        }
        coord_step(x[0], x[1], e1a, den0, r0, d);
        coord_step(x[1], x[0], e2a, den1, r1, d);
        slide_step(x[0], x[1], e3a, den3a, r3a, d);
        coord_step(x[2], x[3], ne1b, den2, r2, d);
        coord_step(x[3], x[2], ne2b, den3, r3, d);
        slide_step(x[2], x[3], ne3b, den3b, r3b, d);
    }
    const R dd = dot3(d, d);
    const R j_total = half * dd + penalty(x, alpha_it);
    R mv[3];
    contact_mid(A, x, e1a, e2a, d, mv);
#pragma unroll
    for (int i = 0; i < 3; ++i) mv[i] = mv[i] - mid_old[i];
    const R move = sqrtv(norm3_sq_sum(mv));
    const R jh = half * dd;
    const bool settled = (absv(j_total - j_old) <= kp.c_factor * eps) && (move <= kp.move_factor * eps);
    const bool contact = settled && (jh <= (R(T(2)) * eps) * eps);
    o.kind = contact ? KIND_CONTACT : (settled ? KIND_NO_CONTACT : KIND_NOT_TERMINATED);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        o.pa[i] = (A[i] + x[0] * e1a[i]) + x[1] * e2a[i];
        o.pb[i] = (B[i] + x[2] * (-ne1b[i])) + x[3] * (-ne2b[i]);
    }
    o.distance = sqrtv(R(T(2)) * jh);
    o.ba[0] = x[0]; o.ba[1] = x[1];
    o.bb[0] = x[2]; o.bb[1] = x[3];
    o.ids = 0x00FFFFFFu | ((uint32_t)((settled ? FLAG_SETTLED : 0u) | (contact ? FLAG_ITER_CONTACT : 0u)) << 24);
}

}  // namespace tc
