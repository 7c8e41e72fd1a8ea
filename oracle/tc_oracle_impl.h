/*
 * tc_oracle_impl.h -- per-pair restatement of RK/kernels.py, instantiated for
 * REAL = double (SFX f64) and REAL = float (SFX f32) by tc_oracle.c.
 *
 * TEST INFRASTRUCTURE ONLY (see tc_oracle.h).  Compiled with
 * -ffp-contract=off: every +,-,*,/ below is one IEEE round-to-nearest
 * operation in the order numpy evaluates the reference's array expressions.
 *
 * Requires: REAL, SFX, SQRT, DOT3_ORDER_02_1 (1 for the float64 einsum reduction
 * order (p0+p2)+p1, 0 for float32's (p0+p1)+p2), CAT(a,b).
 */

#define FN(name) CAT(name, SFX)

/* numpy einsum("ij,ij->i") over a contiguous 3-vector (pinned, oracle/README.md). */
static inline REAL FN(dot3_)(const REAL* a, const REAL* b) {
    REAL p0 = a[0] * b[0];
    REAL p1 = a[1] * b[1];
    REAL p2 = a[2] * b[2];
#if DOT3_ORDER_02_1
    REAL s = p0 + p2;
    return s + p1;
#else
    REAL s = p0 + p1;
    return s + p2;
#endif
}

static inline void FN(sub3_)(const REAL* a, const REAL* b, REAL* o) {
    o[0] = a[0] - b[0];
    o[1] = a[1] - b[1];
    o[2] = a[2] - b[2];
}

/* np.cross for 3-vectors: cp0 = a1*b2 - a2*b1, ... */
static inline void FN(cross3_)(const REAL* a, const REAL* b, REAL* o) {
    REAL t;
    o[0] = a[1] * b[2]; t = a[2] * b[1]; o[0] = o[0] - t;
    o[1] = a[2] * b[0]; t = a[0] * b[2]; o[1] = o[1] - t;
    o[2] = a[0] * b[1]; t = a[1] * b[0]; o[2] = o[2] - t;
}

/* np.clip semantics for non-NaN input: min(max(x, lo), hi). */
static inline REAL FN(clip_)(REAL x, REAL lo, REAL hi) {
    x = (x > lo) ? x : lo;
    return (x < hi) ? x : hi;
}

/* np.maximum(a, b) for non-NaN input. */
static inline REAL FN(max_)(REAL a, REAL b) { return (a >= b) ? a : b; }

/* Decision margins of the last helper call on this thread (test-side tie
 * classification of the FMA build, tests/parity.py); they do not feed back
 * into any result. */
static __thread double FN(tl_pt_d_), FN(tl_pt_v_), FN(tl_seg_), FN(tl_cx_plane_), FN(tl_cx_inside_), FN(tl_cx_cond_);

static inline double FN(fabsd_)(double x) { return x < 0 ? -x : x; }
static inline double FN(mind_)(double a, double b) { return a < b ? a : b; }
static inline double FN(max_d_)(double a, double b) { return a > b ? a : b; }

/* RK/geometry.py:68-75 degenerate_mask: sq_area < rel_tol * L * L, rel_tol
 * rounded to REAL like the reference's Python float times a REAL array. */
static int FN(degenerate_tol_one_)(const REAL* t, double rel_tol) {
    REAL e1[3], e2[3], c[3], ed[3];
    FN(sub3_)(t + 3, t, e1);
    FN(sub3_)(t + 6, t, e2);
    FN(cross3_)(e1, e2, c);
    REAL sq_area = (REAL)0.25 * FN(dot3_)(c, c);
    /* edges = tris[:, [1, 2, 0]] - tris */
    REAL l0, l1, l2, L;
    FN(sub3_)(t + 3, t, ed); l0 = FN(dot3_)(ed, ed);
    FN(sub3_)(t + 6, t + 3, ed); l1 = FN(dot3_)(ed, ed);
    FN(sub3_)(t, t + 6, ed); l2 = FN(dot3_)(ed, ed);
    L = FN(max_)(FN(max_)(l0, l1), l2);
    REAL thr = (REAL)rel_tol * L;
    thr = thr * L;
    return (L == (REAL)0) || (sq_area < thr);
}

/* the hybrid's screen uses the reference default (RK/kernels.py:598) */
static int FN(degenerate_one_)(const REAL* t) { return FN(degenerate_tol_one_)(t, 1e-12); }

/* RK/kernels.py:157-221 closest_point_triangle_batch, one point.
 * Returns the region claimed, in claim order: 0 VA, 1 VB, 2 EAB, 3 VC,
 * 4 EAC, 5 EBC, 6 interior. */
static int FN(closest_point_triangle_one_)(const REAL* p, const REAL* tri, REAL* closest,
                                           REAL* u_out, REAL* w_out) {
    const REAL* a = tri;
    const REAL* b = tri + 3;
    const REAL* c = tri + 6;
    REAL ab[3], ac[3], ap[3], bp[3], cp[3];
    FN(sub3_)(b, a, ab);
    FN(sub3_)(c, a, ac);
    FN(sub3_)(p, a, ap);
    REAL d1 = FN(dot3_)(ab, ap);
    REAL d2 = FN(dot3_)(ac, ap);
    FN(sub3_)(p, b, bp);
    REAL d3 = FN(dot3_)(ab, bp);
    REAL d4 = FN(dot3_)(ac, bp);
    FN(sub3_)(p, c, cp);
    REAL d5 = FN(dot3_)(ab, cp);
    REAL d6 = FN(dot3_)(ac, cp);
    REAL t1, t2;
    t1 = d1 * d4; t2 = d3 * d2; REAL vc = t1 - t2;
    t1 = d5 * d2; t2 = d1 * d6; REAL vb = t1 - t2;
    t1 = d3 * d6; t2 = d5 * d4; REAL va = t1 - t2;
    {
        double m = FN(fabsd_)(d1);
        m = FN(mind_)(m, FN(fabsd_)(d2)); m = FN(mind_)(m, FN(fabsd_)(d3));
        m = FN(mind_)(m, FN(fabsd_)(d4)); m = FN(mind_)(m, FN(fabsd_)(d5));
        m = FN(mind_)(m, FN(fabsd_)(d6)); m = FN(mind_)(m, FN(fabsd_)((double)d4 - d3));
        m = FN(mind_)(m, FN(fabsd_)((double)d5 - d6));
        FN(tl_pt_d_) = m;
        FN(tl_pt_v_) = FN(mind_)(FN(mind_)(FN(fabsd_)(va), FN(fabsd_)(vb)), FN(fabsd_)(vc));
    }
    REAL u = 0, w = 0;
    int region;
    if (d1 <= 0 && d2 <= 0) {
        region = 0;
    } else if (d3 >= 0 && d4 <= d3) {
        region = 1;
        u = 1;
    } else if (vc <= 0 && d1 >= 0 && d3 <= 0) {
        region = 2;
        REAL den = d1 - d3;
        u = d1 / (den == 0 ? (REAL)1 : den);
    } else if (d6 >= 0 && d5 <= d6) {
        region = 3;
        w = 1;
    } else if (vb <= 0 && d2 >= 0 && d6 <= 0) {
        region = 4;
        REAL den = d2 - d6;
        w = d2 / (den == 0 ? (REAL)1 : den);
    } else if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
        region = 5;
        REAL n1 = d4 - d3, n2 = d5 - d6;
        REAL den = n1 + n2;
        REAL t = n1 / (den == 0 ? (REAL)1 : den);
        u = 1 - t;
        w = t;
    } else {
        region = 6;
        REAL den = va + vb;
        den = den + vc;
        den = (den == 0) ? (REAL)1 : den;
        u = vb / den;
        w = vc / den;
    }
    for (int i = 0; i < 3; ++i) {
        REAL q = u * ab[i];
        q = a[i] + q;
        REAL r = w * ac[i];
        closest[i] = q + r;
    }
    *u_out = u;
    *w_out = w;
    return region;
}

#define TC_TINY_ ((REAL)1e-30)

/* RK/kernels.py:224-252 _closest_segment_segment.  Returns a branch code:
 * bit0 = denom > TINY (s from the 2x2 solve), bit1 = t < 0, bit2 = t > 1. */
static int FN(segment_segment_)(const REAL* p1, const REAL* q1, const REAL* p2, const REAL* q2,
                                REAL* s_out, REAL* t_out, REAL* c1, REAL* c2) {
    REAL d1[3], d2[3], r[3];
    FN(sub3_)(q1, p1, d1);
    FN(sub3_)(q2, p2, d2);
    FN(sub3_)(p1, p2, r);
    REAL a = FN(dot3_)(d1, d1);
    REAL e = FN(dot3_)(d2, d2);
    REAL f = FN(dot3_)(d2, r);
    REAL c = FN(dot3_)(d1, r);
    REAL b = FN(dot3_)(d1, d2);
    REAL t1 = a * e, t2 = b * b;
    REAL denom = t1 - t2;
    int code = 0;
    REAL s;
    /* the solve / parallel decision: denom = a e sin^2(angle) is rounding
     * noise for nearly parallel segments, so its margin is |denom| / (a e) */
    double sm = FN(fabsd_)((double)denom) / FN(max_d_)((double)a * (double)e, 1e-300);
    if (denom > TC_TINY_) {
        code |= 1;
        t1 = b * f;
        t2 = c * e;
        REAL num = t1 - t2;
        REAL sr = num / denom;
        sm = FN(mind_)(FN(fabsd_)(sr), FN(fabsd_)((double)sr - 1));
        s = FN(clip_)(sr, 0, 1);
    } else {
        s = 0;
    }
    REAL e_safe = (e > TC_TINY_) ? e : (REAL)1;
    REAL t = b * s;
    t = t + f;
    t = t / e_safe;
    sm = FN(mind_)(sm, FN(mind_)(FN(fabsd_)(t), FN(fabsd_)((double)t - 1)));
    REAL a_safe = (a > TC_TINY_) ? a : (REAL)1;
    if (t < 0) {
        code |= 2;
        REAL sr = (-c) / a_safe;
        sm = FN(mind_)(sm, FN(mind_)(FN(fabsd_)(sr), FN(fabsd_)((double)sr - 1)));
        s = FN(clip_)(sr, 0, 1);
    } else if (t > 1) {
        code |= 4;
        REAL bc = b - c;
        REAL sr = bc / a_safe;
        sm = FN(mind_)(sm, FN(mind_)(FN(fabsd_)(sr), FN(fabsd_)((double)sr - 1)));
        s = FN(clip_)(sr, 0, 1);
    }
    FN(tl_seg_) = sm;
    t = FN(clip_)(t, 0, 1);
    for (int i = 0; i < 3; ++i) {
        REAL x = s * d1[i];
        c1[i] = p1[i] + x;
        REAL y = t * d2[i];
        c2[i] = p2[i] + y;
    }
    *s_out = s;
    *t_out = t;
    return code;
}

/* RK/kernels.py:269-298 _segment_triangle_crossings, one segment. */
static int FN(segment_triangle_crossing_)(const REAL* p, const REAL* q, const REAL* tri,
                                          REAL* x) {
    const REAL* a = tri;
    REAL u[3], v[3], nrm[3], pa[3], qa[3], qp[3], wv[3];
    FN(sub3_)(tri + 3, a, u);
    FN(sub3_)(tri + 6, a, v);
    FN(cross3_)(u, v, nrm);
    FN(sub3_)(p, a, pa);
    REAL dp = FN(dot3_)(pa, nrm);
    FN(sub3_)(q, a, qa);
    REAL dq = FN(dot3_)(qa, nrm);
    REAL prod = dp * dq;
    int crossing = prod < 0;
    REAL denom = dp - dq;
    REAL t = dp / (denom == 0 ? (REAL)1 : denom);
    FN(sub3_)(q, p, qp);
    for (int i = 0; i < 3; ++i) {
        REAL y = t * qp[i];
        x[i] = p[i] + y;
    }
    FN(sub3_)(x, a, wv);
    REAL uu = FN(dot3_)(u, u);
    REAL uv = FN(dot3_)(u, v);
    REAL vv = FN(dot3_)(v, v);
    REAL wu = FN(dot3_)(wv, u);
    REAL wvv = FN(dot3_)(wv, v);
    REAL t1 = uu * vv, t2 = uv * uv;
    REAL det = t1 - t2;
    REAL det_safe = (((det < 0) ? -det : det) > TC_TINY_) ? det : (REAL)1;
    t1 = vv * wu; t2 = uv * wvv;
    REAL b1 = (t1 - t2) / det_safe;
    t1 = uu * wvv; t2 = uv * wu;
    REAL b2 = (t1 - t2) / det_safe;
    REAL bs = b1 + b2;
    int inside = (b1 >= 0) && (b2 >= 0) && (bs <= 1);
    {
        double nn = sqrt((double)nrm[0] * nrm[0] + (double)nrm[1] * nrm[1] + (double)nrm[2] * nrm[2]);
        FN(tl_cx_plane_) = nn > 0 ? FN(mind_)(FN(fabsd_)(dp), FN(fabsd_)(dq)) / nn : 0;
        /* conditioning of the 2x2 barycentric solve: (uu + vv)^2 / |det| */
        FN(tl_cx_cond_) = FN(fabsd_)(det) > 0 ? ((double)uu + vv) * ((double)uu + vv) / FN(fabsd_)(det) : 1e300;
        FN(tl_cx_inside_) = crossing ? FN(mind_)(FN(mind_)(FN(fabsd_)(b1), FN(fabsd_)(b2)),
                                                 FN(fabsd_)(1.0 - (double)b1 - b2)) : 1e300;
    }
    return crossing && inside;
}

static const int FN(EDGE_START_)[3] = {0, 1, 2};
static const int FN(EDGE_END_)[3] = {1, 2, 0};

static void FN(edge_bary_)(int k, REAL s, REAL* out) {
    if (k == 0) { out[0] = s; out[1] = 0; }
    else if (k == 1) { out[0] = 1 - s; out[1] = s; }
    else { out[0] = 0; out[1] = 1 - s; }
}

typedef struct {
    REAL distance, pa[3], pb[3], ba[2], bb[2];
    int8_t kind;
    uint8_t ids[4];
    double mg[10]; /* decision margins, see tco_margins_* */
} FN(rec_);

/* RK/kernels.py:301-401 comparison_batch, one pair. */
static void FN(comparison_one_)(const REAL* A, const REAL* B, REAL eps, FN(rec_)* out) {
    REAL best = 0, pa[3], pb[3], ba[2], bb[2];
    int best_row = -1, best_code = 0;
    double second = 1e300, win_margin = 1e300;
    /* squared scale of the pair, to normalise region-test operands */
    double sq = 0;
    {
        double m = 0;
        for (int t = 0; t < 2; ++t) {
            const REAL* T = t ? B : A;
            for (int k = 0; k < 3; ++k) {
                const REAL* p0 = T + 3 * k;
                const REAL* p1 = T + 3 * ((k + 1) % 3);
                double e = 0;
                for (int i = 0; i < 3; ++i) e += ((double)p1[i] - p0[i]) * ((double)p1[i] - p0[i]);
                m = e > m ? e : m;
            }
        }
        sq = m > 0 ? m : 1;
    }
    int row = 0;
    REAL closest[3], diff[3], u, w, d2;
    for (int k = 0; k < 3; ++k, ++row) {
        const REAL* pt = A + 3 * k;
        int reg = FN(closest_point_triangle_one_)(pt, B, closest, &u, &w);
        FN(sub3_)(pt, closest, diff);
        d2 = FN(dot3_)(diff, diff);
        if (best_row >= 0 && !(d2 < best) && d2 < second) second = d2;
        double wm = FN(mind_)(FN(tl_pt_d_) / sq, FN(tl_pt_v_) / (sq * sq));
        if (best_row < 0 || d2 < best) {
            if (best_row >= 0) second = best;
            best = d2; best_row = row; best_code = reg; win_margin = wm;
            for (int i = 0; i < 3; ++i) { pa[i] = pt[i]; pb[i] = closest[i]; }
            ba[0] = (k == 1) ? 1 : 0; ba[1] = (k == 2) ? 1 : 0;
            bb[0] = u; bb[1] = w;
        }
    }
    for (int k = 0; k < 3; ++k, ++row) {
        const REAL* pt = B + 3 * k;
        int reg = FN(closest_point_triangle_one_)(pt, A, closest, &u, &w);
        FN(sub3_)(pt, closest, diff);
        d2 = FN(dot3_)(diff, diff);
        if (best_row >= 0 && !(d2 < best) && d2 < second) second = d2;
        double wm = FN(mind_)(FN(tl_pt_d_) / sq, FN(tl_pt_v_) / (sq * sq));
        if (d2 < best) {
            second = best;
            best = d2; best_row = row; best_code = reg; win_margin = wm;
            for (int i = 0; i < 3; ++i) { pa[i] = closest[i]; pb[i] = pt[i]; }
            ba[0] = u; ba[1] = w;
            bb[0] = (k == 1) ? 1 : 0; bb[1] = (k == 2) ? 1 : 0;
        }
    }
    for (int ka = 0; ka < 3; ++ka) {
        for (int kb = 0; kb < 3; ++kb, ++row) {
            REAL s, t, c1[3], c2[3];
            int code = FN(segment_segment_)(A + 3 * FN(EDGE_START_)[ka], A + 3 * FN(EDGE_END_)[ka],
                                            B + 3 * FN(EDGE_START_)[kb], B + 3 * FN(EDGE_END_)[kb],
                                            &s, &t, c1, c2);
            FN(sub3_)(c1, c2, diff);
            d2 = FN(dot3_)(diff, diff);
            if (!(d2 < best) && d2 < second) second = d2;
            double wm = FN(tl_seg_);
            if (d2 < best) {
                second = best;
                best = d2; best_row = row; best_code = code; win_margin = wm;
                for (int i = 0; i < 3; ++i) { pa[i] = c1[i]; pb[i] = c2[i]; }
                FN(edge_bary_)(ka, s, ba);
                FN(edge_bary_)(kb, t, bb);
            }
        }
    }
    REAL distance = SQRT(best);
    /* six edge-to-plane tests */
    REAL pts[6][3];
    int ok[6], any = 0;
    double cx_plane = 1e300, cx_inside = 1e300, cx_cond = 0;
    for (int k = 0; k < 3; ++k) {
        ok[k] = FN(segment_triangle_crossing_)(A + 3 * FN(EDGE_START_)[k], A + 3 * FN(EDGE_END_)[k], B, pts[k]);
        cx_plane = FN(mind_)(cx_plane, FN(tl_cx_plane_)); cx_inside = FN(mind_)(cx_inside, FN(tl_cx_inside_));
        cx_cond = cx_cond > FN(tl_cx_cond_) ? cx_cond : FN(tl_cx_cond_);
        ok[k + 3] = FN(segment_triangle_crossing_)(B + 3 * FN(EDGE_START_)[k], B + 3 * FN(EDGE_END_)[k], A, pts[k + 3]);
        cx_plane = FN(mind_)(cx_plane, FN(tl_cx_plane_)); cx_inside = FN(mind_)(cx_inside, FN(tl_cx_inside_));
        cx_cond = cx_cond > FN(tl_cx_cond_) ? cx_cond : FN(tl_cx_cond_);
        any |= ok[k] | ok[k + 3];
    }
    uint8_t pair_id = 255;
    if (any) {
        REAL bestv = 0;
        int bi = -1;
        for (int i0 = 0; i0 < 6; ++i0) {
            for (int i1 = 0; i1 < 6; ++i1) {
                REAL v;
                if (ok[i0] && ok[i1]) {
                    FN(sub3_)(pts[i0], pts[i1], diff);
                    v = FN(dot3_)(diff, diff);
                } else {
                    v = -1;
                }
                if (bi < 0 || v > bestv) { bestv = v; bi = i0 * 6 + i1; }
            }
        }
        int i0 = bi / 6, i1 = bi % 6;
        pair_id = (uint8_t)bi;
        REAL mid[3];
        for (int i = 0; i < 3; ++i) {
            REAL s = pts[i0][i] + pts[i1][i];
            mid[i] = (REAL)0.5 * s;
        }
        distance = 0;
        for (int i = 0; i < 3; ++i) { pa[i] = mid[i]; pb[i] = mid[i]; }
        FN(closest_point_triangle_one_)(mid, A, closest, &ba[0], &ba[1]);
        FN(closest_point_triangle_one_)(mid, B, closest, &bb[0], &bb[1]);
    }
    REAL thr = (REAL)2 * eps;
    out->kind = (distance <= thr) ? 1 : 0;
    out->distance = distance;
    for (int i = 0; i < 3; ++i) { out->pa[i] = pa[i]; out->pb[i] = pb[i]; }
    out->ba[0] = ba[0]; out->ba[1] = ba[1];
    out->bb[0] = bb[0]; out->bb[1] = bb[1];
    out->ids[0] = (uint8_t)best_row;
    out->ids[1] = (uint8_t)best_code;
    out->ids[2] = pair_id;
    out->ids[3] = any ? 16 : 0;
    out->mg[0] = second - (double)best;
    out->mg[1] = (double)distance - (double)thr;
    out->mg[2] = cx_plane;
    out->mg[3] = cx_inside;
    out->mg[7] = win_margin;
    out->mg[8] = (double)SQRT(best);
    out->mg[9] = cx_cond;
}

/* RK/kernels.py:417-431 _penalty_value, summed left to right. */
static REAL FN(penalty_)(const REAL* x, REAL alpha) {
    REAL a1 = x[0], b1 = x[1], a2 = x[2], b2 = x[3];
    REAL p = FN(max_)(0, a1 - 1);
    p = p + FN(max_)(0, -a1);
    p = p + FN(max_)(0, b1 - 1);
    p = p + FN(max_)(0, -b1);
    REAL s1 = a1 + b1;
    p = p + FN(max_)(0, s1 - 1);
    p = p + FN(max_)(0, a2 - 1);
    p = p + FN(max_)(0, -a2);
    p = p + FN(max_)(0, b2 - 1);
    p = p + FN(max_)(0, -b2);
    REAL s2 = a2 + b2;
    p = p + FN(max_)(0, s2 - 1);
    return alpha * p;
}

static inline void FN(midpoint_)(const REAL* A0, const REAL* x, const REAL* e1a, const REAL* e2a,
                                 const REAL* d, REAL* m) {
    for (int i = 0; i < 3; ++i) {
        REAL t = x[0] * e1a[i];
        REAL v = A0[i] + t;
        t = x[1] * e2a[i];
        v = v + t;
        t = (REAL)0.5 * d[i];
        m[i] = v - t;
    }
}

/* RK/kernels.py:447-565 iterative_batch, one pair. */
static void FN(iterative_one_)(const REAL* A, const REAL* B, REAL eps, const tco_params* prm,
                               FN(rec_)* out) {
    const REAL* A0 = A;
    const REAL* B0 = B;
    REAL e1a[3], e2a[3], e1b[3], e2b[3], base[3], ne1b[3], ne2b[3];
    FN(sub3_)(A + 3, A0, e1a);
    FN(sub3_)(A + 6, A0, e2a);
    FN(sub3_)(B + 3, B0, e1b);
    FN(sub3_)(B + 6, B0, e2b);
    FN(sub3_)(A0, B0, base);
    for (int i = 0; i < 3; ++i) { ne1b[i] = -e1b[i]; ne2b[i] = -e2b[i]; }
    const REAL* dirs[4] = {e1a, e2a, ne1b, ne2b};

    /* _pair_max_sq_edge (RK/kernels.py:409-414) */
    REAL ed[3], la, lb, l0, l1, l2;
    FN(sub3_)(A + 3, A, ed); l0 = FN(dot3_)(ed, ed);
    FN(sub3_)(A + 6, A + 3, ed); l1 = FN(dot3_)(ed, ed);
    FN(sub3_)(A, A + 6, ed); l2 = FN(dot3_)(ed, ed);
    la = FN(max_)(FN(max_)(l0, l1), l2);
    FN(sub3_)(B + 3, B, ed); l0 = FN(dot3_)(ed, ed);
    FN(sub3_)(B + 6, B + 3, ed); l1 = FN(dot3_)(ed, ed);
    FN(sub3_)(B, B + 6, ed); l2 = FN(dot3_)(ed, ed);
    lb = FN(max_)(FN(max_)(l0, l1), l2);
    REAL sq = FN(max_)(la, lb);
    REAL alpha_it = (REAL)prm->alpha_iterative * sq;
    REAL alpha_reg = (REAL)prm->alpha_regulariser * sq;
    REAL den[4];
    for (int k = 0; k < 4; ++k) {
        REAL v = FN(dot3_)(dirs[k], dirs[k]) + alpha_reg;
        den[k] = FN(max_)(v, TC_TINY_);
    }
    REAL e3a[3], e3b[3], ne3b[3];
    FN(sub3_)(e2a, e1a, e3a);
    FN(sub3_)(e2b, e1b, e3b);
    for (int i = 0; i < 3; ++i) ne3b[i] = -e3b[i];
    REAL den3a = FN(max_)(FN(dot3_)(e3a, e3a) + alpha_reg, TC_TINY_);
    REAL den3b = FN(max_)(FN(dot3_)(e3b, e3b) + alpha_reg, TC_TINY_);

    REAL x[4];
    for (int k = 0; k < 4; ++k) x[k] = (REAL)prm->start_coord;
    REAL d[3];
    for (int i = 0; i < 3; ++i) {
        REAL t = x[0] * e1a[i];
        REAL v = base[i] + t;
        t = x[1] * e2a[i]; v = v + t;
        t = x[2] * e1b[i]; v = v - t;
        t = x[3] * e2b[i]; v = v - t;
        d[i] = v;
    }
    REAL j_total = (REAL)0.5 * FN(dot3_)(d, d) + FN(penalty_)(x, alpha_it);
    REAL j_old = (REAL)INFINITY;
    REAL midpoint[3], new_mid[3];
    FN(midpoint_)(A0, x, e1a, e2a, d, midpoint);
    REAL move = (REAL)INFINITY;
    static const int partner[4] = {1, 0, 3, 2};
    for (int it = 0; it < prm->n_iterative; ++it) {
        j_old = j_total;
        for (int k = 0; k < 4; ++k) {
            const REAL* e = dirs[k];
            REAL g = FN(dot3_)(d, e) / den[k];
            REAL target = x[k] - g;
            REAL hi = FN(max_)(0, 1 - FN(max_)(x[partner[k]], 0));
            target = FN(clip_)(target, 0, hi);
            REAL step = target - x[k];
            x[k] = target;
            for (int i = 0; i < 3; ++i) { REAL t = step * e[i]; d[i] = d[i] + t; }
            if (k & 1) {
                int ka = k - 1, kb = k;
                const REAL* e3 = (k == 1) ? e3a : ne3b;
                REAL den3 = (k == 1) ? den3a : den3b;
                REAL t = (-FN(dot3_)(d, e3)) / den3;
                t = FN(clip_)(t, -FN(max_)(x[kb], 0), FN(max_)(x[ka], 0));
                x[ka] = x[ka] - t;
                x[kb] = x[kb] + t;
                for (int i = 0; i < 3; ++i) { REAL y = t * e3[i]; d[i] = d[i] + y; }
            }
        }
        j_total = (REAL)0.5 * FN(dot3_)(d, d) + FN(penalty_)(x, alpha_it);
        FN(midpoint_)(A0, x, e1a, e2a, d, new_mid);
        REAL mv[3];
        FN(sub3_)(new_mid, midpoint, mv);
        /* np.linalg.norm(axis=1) = sqrt(add.reduce(x*x)) -> (m0^2 + m1^2) + m2^2 */
        REAL s0 = mv[0] * mv[0], s1 = mv[1] * mv[1], s2 = mv[2] * mv[2];
        REAL ss = s0 + s1;
        ss = ss + s2;
        move = SQRT(ss);
        for (int i = 0; i < 3; ++i) midpoint[i] = new_mid[i];
    }
    REAL jh = (REAL)0.5 * FN(dot3_)(d, d);
    REAL dj = j_total - j_old;
    dj = (dj < 0) ? -dj : dj;
    REAL ceps = (REAL)prm->c_factor * eps;
    REAL meps = (REAL)prm->move_factor * eps;
    int settled = (dj <= ceps) && (move <= meps);
    REAL thr = (REAL)2 * eps;
    thr = thr * eps;
    int contact = settled && (jh <= thr);
    out->kind = contact ? 1 : (settled ? 0 : 2);
    for (int i = 0; i < 3; ++i) {
        REAL t = x[0] * e1a[i];
        REAL v = A0[i] + t;
        t = x[1] * e2a[i];
        out->pa[i] = v + t;
        t = x[2] * e1b[i];
        v = B0[i] + t;
        t = x[3] * e2b[i];
        out->pb[i] = v + t;
    }
    out->distance = SQRT((REAL)2 * jh);
    out->ba[0] = x[0]; out->ba[1] = x[1];
    out->bb[0] = x[2]; out->bb[1] = x[3];
    out->ids[0] = 255; out->ids[1] = 255; out->ids[2] = 255;
    out->ids[3] = (uint8_t)((settled ? 1 : 0) | (contact ? 2 : 0));
    out->mg[4] = (double)dj - (double)ceps;
    out->mg[5] = (double)move - (double)meps;
    out->mg[6] = (double)jh - (double)thr;
}

static inline void FN(store_)(const FN(rec_)* r, int64_t i, REAL* distance, REAL* point_a,
                              REAL* point_b, REAL* bary_a, REAL* bary_b, int8_t* kind,
                              uint8_t* ids) {
    if (distance) distance[i] = r->distance;
    if (point_a) for (int k = 0; k < 3; ++k) point_a[3 * i + k] = r->pa[k];
    if (point_b) for (int k = 0; k < 3; ++k) point_b[3 * i + k] = r->pb[k];
    if (bary_a) { bary_a[2 * i] = r->ba[0]; bary_a[2 * i + 1] = r->ba[1]; }
    if (bary_b) { bary_b[2 * i] = r->bb[0]; bary_b[2 * i + 1] = r->bb[1]; }
    if (kind) kind[i] = r->kind;
    if (ids) for (int k = 0; k < 4; ++k) ids[4 * i + k] = r->ids[k];
}

typedef struct {
    const REAL *A, *B, *eps, *P;
    const uint8_t* allow_fb;
    const tco_params* p;
    REAL *distance, *point_a, *point_b, *bary_a, *bary_b;
    int8_t* kind;
    uint8_t* ids;
    int64_t n_fb[TCO_MAX_THREADS], n_deg[TCO_MAX_THREADS];
    double rel_tol;
} FN(ctx_);

static void FN(comparison_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    (void)tid;
    for (int64_t i = lo; i < hi; ++i) {
        FN(rec_) r;
        FN(comparison_one_)(c->A + 9 * i, c->B + 9 * i, c->eps[i], &r);
        FN(store_)(&r, i, c->distance, c->point_a, c->point_b, c->bary_a, c->bary_b, c->kind, c->ids);
    }
}

static void FN(iterative_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    (void)tid;
    for (int64_t i = lo; i < hi; ++i) {
        FN(rec_) r;
        FN(iterative_one_)(c->A + 9 * i, c->B + 9 * i, c->eps[i], c->p, &r);
        FN(store_)(&r, i, c->distance, c->point_a, c->point_b, c->bary_a, c->bary_b, c->kind, c->ids);
    }
}

/* RK/kernels.py:568-605 hybrid_batch body.  Degenerate fallback pairs keep
 * the iterative result with kind 3 (the caller raises DegenerateTriangle,
 * RK/kernels.py:598-600). */
static void FN(hybrid_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    int64_t n_fb = 0, n_deg = 0;
    for (int64_t i = lo; i < hi; ++i) {
        FN(rec_) r;
        const REAL* A = c->A + 9 * i;
        const REAL* B = c->B + 9 * i;
        FN(iterative_one_)(A, B, c->eps[i], c->p, &r);
        int allow = c->allow_fb ? (c->allow_fb[i] != 0) : 1;
        if (r.kind == 2 && allow) {
            if (FN(degenerate_one_)(A) || FN(degenerate_one_)(B)) {
                r.kind = 3;
                r.ids[3] |= 8;
                n_deg++;
            } else {
                uint8_t flags = r.ids[3];
                FN(comparison_one_)(A, B, c->eps[i], &r);
                r.ids[3] |= flags | 4;
                n_fb++;
            }
        }
        FN(store_)(&r, i, c->distance, c->point_a, c->point_b, c->bary_a, c->bary_b, c->kind, c->ids);
    }
    c->n_fb[tid] += n_fb;
    c->n_deg[tid] += n_deg;
}

static void FN(margins_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    (void)tid;
    double* mg = (double*)c->distance;
    for (int64_t i = lo; i < hi; ++i) {
        FN(rec_) rc, ri;
        FN(comparison_one_)(c->A + 9 * i, c->B + 9 * i, c->eps[i], &rc);
        FN(iterative_one_)(c->A + 9 * i, c->B + 9 * i, c->eps[i], c->p, &ri);
        for (int k = 0; k < TCO_N_MARGINS; ++k) mg[TCO_N_MARGINS * i + k] = (k >= 4 && k <= 6) ? ri.mg[k] : rc.mg[k];
    }
}

static void FN(cpt_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    (void)tid;
    for (int64_t i = lo; i < hi; ++i) {
        REAL cl[3], u, w;
        FN(closest_point_triangle_one_)(c->P + 3 * i, c->A + 9 * i, cl, &u, &w);
        if (c->point_a) for (int k = 0; k < 3; ++k) c->point_a[3 * i + k] = cl[k];
        if (c->bary_a) { c->bary_a[2 * i] = u; c->bary_a[2 * i + 1] = w; }
    }
}

static void FN(degenerate_body_)(int64_t lo, int64_t hi, int tid, void* arg) {
    FN(ctx_)* c = (FN(ctx_)*)arg;
    (void)tid;
    for (int64_t i = lo; i < hi; ++i) c->ids[i] = (uint8_t)FN(degenerate_tol_one_)(c->A + 9 * i, c->rel_tol);
}

int FN(tco_comparison_)(const REAL* A, const REAL* B, int64_t n, const REAL* eps,
                        REAL* distance, REAL* point_a, REAL* point_b, REAL* bary_a,
                        REAL* bary_b, int8_t* kind, uint8_t* ids, int threads) {
    if (n < 0 || (n > 0 && (!A || !B || !eps))) return 1;
    FN(ctx_) c = {0};
    c.A = A; c.B = B; c.eps = eps;
    c.distance = distance; c.point_a = point_a; c.point_b = point_b;
    c.bary_a = bary_a; c.bary_b = bary_b; c.kind = kind; c.ids = ids;
    tco_parallel_for(n, threads, FN(comparison_body_), &c);
    return 0;
}

int FN(tco_iterative_)(const REAL* A, const REAL* B, int64_t n, const REAL* eps,
                       const tco_params* p, REAL* distance, REAL* point_a, REAL* point_b,
                       REAL* bary_a, REAL* bary_b, int8_t* kind, uint8_t* ids, int threads) {
    if (n < 0 || !p || (n > 0 && (!A || !B || !eps))) return 1;
    FN(ctx_) c = {0};
    c.A = A; c.B = B; c.eps = eps; c.p = p;
    c.distance = distance; c.point_a = point_a; c.point_b = point_b;
    c.bary_a = bary_a; c.bary_b = bary_b; c.kind = kind; c.ids = ids;
    tco_parallel_for(n, threads, FN(iterative_body_), &c);
    return 0;
}

/* counts[4] (may be NULL) is incremented by {iterative, comparison, fallback,
 * degenerate}; returns 2 when some fallback pair was degenerate. */
int FN(tco_hybrid_)(const REAL* A, const REAL* B, int64_t n, const REAL* eps,
                    const uint8_t* allow_fb, const tco_params* p, REAL* distance,
                    REAL* point_a, REAL* point_b, REAL* bary_a, REAL* bary_b, int8_t* kind,
                    uint8_t* ids, int64_t* counts, int threads) {
    if (n < 0 || !p || (n > 0 && (!A || !B || !eps))) return 1;
    FN(ctx_) c = {0};
    c.A = A; c.B = B; c.eps = eps; c.p = p; c.allow_fb = allow_fb;
    c.distance = distance; c.point_a = point_a; c.point_b = point_b;
    c.bary_a = bary_a; c.bary_b = bary_b; c.kind = kind; c.ids = ids;
    tco_parallel_for(n, threads, FN(hybrid_body_), &c);
    int64_t n_fb = 0, n_deg = 0;
    for (int t = 0; t < TCO_MAX_THREADS; ++t) { n_fb += c.n_fb[t]; n_deg += c.n_deg[t]; }
    if (counts) {
        counts[0] += n;
        counts[1] += n_fb;
        counts[2] += n_fb;
        counts[3] += n_deg;
    }
    return n_deg ? 2 : 0;
}

/* Decision margins per pair (TCO_N_MARGINS = 10 doubles): [0] second-best minus best squared
 * feature distance, [1] distance - 2 eps, [2] min endpoint-to-plane distance
 * of the six crossing tests, [3] min barycentric inside margin of the tests
 * whose endpoints straddle the plane, [4] |dJ| - c eps, [5] move - mf eps,
 * [6] J_hat - 2 eps^2, [7] normalised region / segment-branch margin (incl. the
 * solve-or-parallel decision, |denom| / (a e)) of the
 * winning feature, [8] the feature distance before the crossing override
 * (the answer had no crossing been found), [9] max conditioning
 * (uu + vv)^2 / |det| of the six barycentric solves.  Test-side tie
 * classification only. */
int FN(tco_margins_)(const REAL* A, const REAL* B, int64_t n, const REAL* eps, const tco_params* p,
                     double* margins, int threads) {
    if (n < 0 || !p || (n > 0 && (!A || !B || !eps || !margins))) return 1;
    FN(ctx_) c = {0};
    c.A = A; c.B = B; c.eps = eps; c.p = p; c.distance = (REAL*)margins;
    tco_parallel_for(n, threads, FN(margins_body_), &c);
    return 0;
}

int FN(tco_closest_point_triangle_)(const REAL* P, const REAL* T, int64_t n, REAL* closest,
                                    REAL* bary, int threads) {
    if (n < 0 || (n > 0 && (!P || !T))) return 1;
    FN(ctx_) c = {0};
    c.P = P; c.A = T; c.point_a = closest; c.bary_a = bary;
    tco_parallel_for(n, threads, FN(cpt_body_), &c);
    return 0;
}

int FN(tco_degenerate_)(const REAL* T, int64_t n, double rel_tol, uint8_t* mask, int threads) {
    if (n < 0 || (n > 0 && (!T || !mask))) return 1;
    FN(ctx_) c = {0};
    c.A = T; c.ids = mask; c.rel_tol = rel_tol;
    tco_parallel_for(n, threads, FN(degenerate_body_), &c);
    return 0;
}

/* RK/geometry.py:162-176 RigidMotion.apply_points: points @ R.T + t with R
 * the quaternion's matrix in Python floats rounded to REAL.  NumPy's matmul
 * of (n, 3) x (3, 3) (OpenBLAS in the reference's environment, checked by
 * tests/test_motion_oracle.py) evaluates each row as the FMA chain
 * fma(R_i2, p2, fma(R_i1, p1, R_i0 p0)); the translation is a separate add. */
int FN(tco_apply_motion_)(const REAL* P, int64_t n, const double* q, const REAL* t, REAL* out) {
    if (n < 0 || (n > 0 && (!P || !q || !t || !out))) return 1;
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double m[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                         2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                         2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    REAL R[9];
    for (int k = 0; k < 9; ++k) R[k] = (REAL)m[k];
    for (int64_t k = 0; k < n; ++k) {
        const REAL* p = P + 3 * k;
        for (int i = 0; i < 3; ++i) {
            const REAL prod = R[3 * i] * p[0];
            out[3 * k + i] = FMA(R[3 * i + 2], p[2], FMA(R[3 * i + 1], p[1], prod)) + t[i];
        }
    }
    return 0;
}

#undef TC_TINY_
#undef FN
