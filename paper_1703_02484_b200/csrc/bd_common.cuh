// bd_common.cuh -- shared building blocks of the B200 Brownian-dynamics engine.
//
// Everything here is __host__ __device__ so the step drivers can also be
// compiled for the host test harness (tests/hostemu).
// Bit-exactness contract: the library is compiled with -fmad=false (device)
// and -ffp-contract=off (host), so every a*b+c below rounds twice, exactly
// like the reference's numba/numpy arithmetic.  Where a fused multiply-add is
// wanted (the fast all-pairs kernel) it is written explicitly with fma().
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../../include/bd_b200.h"

#if defined(__CUDACC__)
#define BD_HD __host__ __device__ __forceinline__
#define BD_DEV __device__ __forceinline__
#else
#define BD_HD inline
#define BD_DEV inline
#endif

namespace bd {

// ---------------------------------------------------------------------------
// periodic geometry (core.py:69-90, _kernels.py:20-23)

// reference min-image: d - floor(d/L + 0.5) * L (ties -> -L/2)
BD_HD double mi_ref(double d, double L) { return d - floor(d / L + 0.5) * L; }

// Same value, division-free, for |d| < L (both operands wrapped into [0, L)):
// floor(fl(fl(d/L) + 0.5)) is a monotone step function of d, so it equals +1
// exactly for d >= hi and -1 exactly for d < lo, where hi / lo are its
// breakpoints found once per box by bisection (bd_prepare_params).  The
// subtraction d - n*L is then the very same rounded operation the reference
// performs (n*L is exact for n in {-1, 0, 1}).
BD_HD double mi_fast(double d, double L, double lo, double hi) {
    return d >= hi ? d - L : (d < lo ? d + L : d);
}

BD_HD double mi_exact(double d, const bd_params_t& p) {
    // out-of-range differences (|d| >= L) cannot occur for wrapped inputs;
    // keep the reference formula for them anyway
    return (d < p.L && d > -p.L) ? mi_fast(d, p.L, p.mi_lo, p.mi_hi) : mi_ref(d, p.L);
}

// wrap into [0, L) (core.py:69-78)
BD_HD double wrap1(double x, double L) {
    double q = x - floor(x / L) * L;
    return q >= L ? q - L : q;
}

// ---------------------------------------------------------------------------
// counter-based noise.  Philox4x64-10 keyed (seed, stream),
// counter (pair, call, attempt, purpose); Marsaglia polar transform with an
// fdlibm-style log built from + - * / only.

BD_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#if defined(__CUDA_ARCH__)
    hi = __umul64hi(a, b);
    lo = a * b;
#else
    unsigned __int128 p = (unsigned __int128)a * b;
    hi = (uint64_t)(p >> 64);
    lo = (uint64_t)p;
#endif
}

BD_HD void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c[0], hi0, lo0);
        mulhilo64(0xCA5A826395121157ULL, c[2], hi1, lo1);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
}

BD_HD double u64_to_pm1(uint64_t w) {
    return (double)((int64_t)(w >> 11) - (int64_t)(1ULL << 52)) * 0x1p-52;
}

BD_HD double bits_to_double(uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)b);
#else
    double d;
    memcpy(&d, &b, 8);
    return d;
#endif
}

BD_HD uint64_t double_to_bits(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t b;
    memcpy(&b, &d, 8);
    return b;
#endif
}

// natural log of a positive normal double (fdlibm e_log.c reduction and
// minimax coefficients; no fma, fixed evaluation order)
BD_HD double log_portable(double x) {
    uint64_t b = double_to_bits(x);
    int64_t e = (int64_t)((b >> 52) & 0x7ff) - 1023;
    double m = bits_to_double((b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
    if (m > 1.4142135623730951) {
        m = m * 0.5;
        e += 1;
    }
    const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
    const double LG1 = 6.666666666666735130e-01, LG2 = 3.999999999940941908e-01,
                 LG3 = 2.857142874366239149e-01, LG4 = 2.222219843214978396e-01,
                 LG5 = 1.818357216161805012e-01, LG6 = 1.531383769920937332e-01,
                 LG7 = 1.479819860511658591e-01;
    double f = m - 1.0;
    double s = f / (2.0 + f);
    double z = s * s;
    double w = z * z;
    double t1 = w * (LG2 + w * (LG4 + w * LG6));
    double t2 = z * (LG1 + w * (LG3 + w * (LG5 + w * LG7)));
    double R = t2 + t1;
    double hfsq = 0.5 * f * f;
    double dk = (double)e;
    return dk * LN2_HI - ((hfsq - (s * (hfsq + R) + dk * LN2_LO)) - f);
}

BD_HD void normal_pair(uint64_t seed, uint64_t stream, uint64_t call, uint64_t pair, uint64_t purpose,
                       double& z0, double& z1) {
    for (uint64_t attempt = 0;; ++attempt) {
        uint64_t w[4] = {pair, call, attempt, purpose};
        philox4x64_10(w, seed, stream);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            double v1 = u64_to_pm1(w[2 * q]), v2 = u64_to_pm1(w[2 * q + 1]);
            double s = v1 * v1 + v2 * v2;
            if (s > 0.0 && s < 1.0) {
                double f = sqrt((-2.0 * log_portable(s)) / s);
                z0 = v1 * f;
                z1 = v2 * f;
                return;
            }
        }
    }
}

BD_HD double clampd(double z, double c) { return z < -c ? -c : (z > c ? c : z); }

// ---------------------------------------------------------------------------
// triangulation geometry (triangulation.py:66-117, :181-222)

struct V2 {
    double x, y;
};

BD_HD V2 emb(const double* pos, int64_t v, double sx, double sy, double L) {
    V2 r;
    r.x = pos[2 * v] + sx * L;
    r.y = pos[2 * v + 1] + sy * L;
    return r;
}

BD_HD double cross2(double ux, double uy, double vx, double vy) { return ux * vy - uy * vx; }

// incircle, triangulation.py:66-87 (scale**4 as (s*s)*(s*s))
BD_HD bool incircle(V2 a, V2 b, V2 c, V2 d, double tol) {
    double ax = a.x - d.x, ay = a.y - d.y;
    double bx = b.x - d.x, by = b.y - d.y;
    double cx = c.x - d.x, cy = c.y - d.y;
    double a2 = ax * ax + ay * ay;
    double b2 = bx * bx + by * by;
    double c2 = cx * cx + cy * cy;
    double det = ax * (by * c2 - b2 * cy) - ay * (bx * c2 - b2 * cx) + a2 * (bx * cy - by * cx);
    double s = fabs(ax);
    s = fmax(s, fabs(ay));
    s = fmax(s, fabs(bx));
    s = fmax(s, fabs(by));
    s = fmax(s, fabs(cx));
    s = fmax(s, fabs(cy));
    double s2 = s * s;
    return det > tol * (s2 * s2);
}

// _point_in_triangle, triangulation.py:94-101
BD_HD bool point_in_tri(V2 p, V2 a, V2 b, V2 c) {
    double s1 = cross2(b.x - a.x, b.y - a.y, p.x - a.x, p.y - a.y);
    double s2 = cross2(c.x - b.x, c.y - b.y, p.x - b.x, p.y - b.y);
    double s3 = cross2(a.x - c.x, a.y - c.y, p.x - c.x, p.y - c.y);
    bool pos = (s1 >= 0) & (s2 >= 0) & (s3 >= 0);
    bool neg = (s1 <= 0) & (s2 <= 0) & (s3 <= 0);
    return pos | neg;
}

// _segments_intersect, triangulation.py:104-117
BD_HD bool seg_intersect(V2 p, V2 q, V2 u, V2 v) {
    double d1 = cross2(q.x - p.x, q.y - p.y, u.x - p.x, u.y - p.y);
    double d2 = cross2(q.x - p.x, q.y - p.y, v.x - p.x, v.y - p.y);
    double d3 = cross2(v.x - u.x, v.y - u.y, p.x - u.x, p.y - u.y);
    double d4 = cross2(v.x - u.x, v.y - u.y, q.x - u.x, q.y - u.y);
    if (d1 == 0.0 && d2 == 0.0 && d3 == 0.0 && d4 == 0.0) {
        if (fmax(p.x, q.x) < fmin(u.x, v.x) || fmax(u.x, v.x) < fmin(p.x, q.x)) return false;
        if (fmax(p.y, q.y) < fmin(u.y, v.y) || fmax(u.y, v.y) < fmin(p.y, q.y)) return false;
        return true;
    }
    return (d1 * d2 <= 0.0) && (d3 * d4 <= 0.0);
}

// ---------------------------------------------------------------------------
// host-side parameter preparation (bd_prepare_params)

inline void prepare_params(bd_params_t* p) {
    // breakpoints of g(d) = floor(fl(fl(d/L) + 0.5)): smallest d with g >= 1
    // (mi_hi) and smallest d with g >= 0 (mi_lo), bisection over the ordered
    // doubles.  Host double arithmetic is IEEE binary64 like the device's.
    const double L = p->L;
    auto g = [L](double d) { return floor(d / L + 0.5); };
    auto ord = [](double d) -> int64_t {
        int64_t b;
        if (d >= 0) {
            memcpy(&b, &d, 8);
            return b;
        }
        double m = -d;
        memcpy(&b, &m, 8);
        return -b;
    };
    auto from_ord = [](int64_t o) -> double {
        double d;
        if (o >= 0) {
            memcpy(&d, &o, 8);
            return d;
        }
        int64_t m = -o;
        memcpy(&d, &m, 8);
        return -d;
    };
    int64_t lo = ord(0.0), hi = ord(L);  // g(lo) < 1 <= g(hi)
    while (hi - lo > 1) {
        int64_t mid = lo + (hi - lo) / 2;
        if (g(from_ord(mid)) >= 1.0) hi = mid;
        else lo = mid;
    }
    p->mi_hi = from_ord(hi);
    lo = ord(-L);
    hi = ord(0.0);  // g(lo) < 0 <= g(hi)
    while (hi - lo > 1) {
        int64_t mid = lo + (hi - lo) / 2;
        if (g(from_ord(mid)) >= 0.0) hi = mid;
        else lo = mid;
    }
    p->mi_lo = from_ord(hi);
    const double rc = p->r_cut > 0 ? p->r_cut : 0.0;
    p->r_list = (rc > p->sigma ? rc : p->sigma) + p->skin;
    const int64_t ncx = (int64_t)floor(L / p->r_list);
    p->ncx = ncx < 3 ? 0 : ncx;
}

}  // namespace bd
