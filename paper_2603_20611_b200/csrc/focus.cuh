// focus.cuh — per-Gaussian focus-Gaussian algebra in fp64 (device).
//
// This is the math of prepare_gaussians (render.hpp:90-131) and of the
// backward chain (backward.hpp:55-89, :148-173; grad_chain.hpp:27-77),
// evaluated per primitive in registers. It is compiled ONLY into prep.cu,
// whose translation unit is built with --fmad=false: every product and sum
// below rounds exactly like the reference's x86-64 SSE2 build, and the
// expressions keep the reference's evaluation order, so survivor sets and
// the integer pixel bounds (which feed the bit-exact tile lists) agree with
// the CPU reference except where libm exp/acos/cos differ by an ulp.
//
// Deviation by design (performance, result-preserving): the trigonometric
// eigenvalue conditioning test of invert_covariance (core.hpp:184-198,
// vec.hpp:154-179) is skipped when the exact eigenvalue ratio known from the
// scales, (max s / min s)^2, is <= 1e6. In that regime the reference's test
// provably passes (its eigenvalue error is < 1e-8 * lambda_max), so the
// returned inverse is identical. Everything else runs the reference path.
#pragma once

#include <math.h>

#include "common.cuh"

namespace gpk {

struct D2 { double x, y; };
struct D3 { double x, y, z; };
struct D33 { double m[3][3]; };

__device__ __forceinline__ D33 m33_mul(const D33& a, const D33& b) {
    D33 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
    return r;
}

__device__ __forceinline__ D3 m33_mulv(const D33& a, const D3& v) {
    return {a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
            a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
            a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z};
}

__device__ __forceinline__ D33 m33_t(const D33& a) {
    D33 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}

__device__ __forceinline__ D33 m33_add(const D33& a, const D33& b) {
    D33 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
    return r;
}

__device__ __forceinline__ D33 m33_scale(const D33& a, double s) {
    D33 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] * s;
    return r;
}

__device__ __forceinline__ D33 outer3(const D3& u, const D3& v) {
    const double uu[3] = {u.x, u.y, u.z}, vv[3] = {v.x, v.y, v.z};
    D33 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.m[i][j] = uu[i] * vv[j];
    return r;
}

__device__ __forceinline__ double dot3(const D3& a, const D3& b) {
    return a.x * b.x + a.y * b.y + a.z * b.z;
}

// Mat3::det (vec.hpp:131-135), same cofactor expansion.
__device__ __forceinline__ double m33_det(const D33& a) {
    const auto& m = a.m;
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

// Mat3::inverse (vec.hpp:137-150): adjugate divided entrywise by det.
__device__ __forceinline__ D33 m33_inverse(const D33& a) {
    const auto& m = a.m;
    const double dt = m33_det(a);
    D33 r;
    r.m[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / dt;
    r.m[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / dt;
    r.m[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / dt;
    r.m[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / dt;
    r.m[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / dt;
    r.m[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / dt;
    r.m[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / dt;
    r.m[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / dt;
    r.m[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / dt;
    return r;
}

// Mat3::sym_eigenvalues (vec.hpp:154-179): trigonometric closed form,
// ascending.
__device__ inline void m33_sym_eig(const D33& a, double ev[3]) {
    const auto& m = a.m;
    const double p1 = m[0][1] * m[0][1] + m[0][2] * m[0][2] + m[1][2] * m[1][2];
    if (p1 == 0.0) {
        double d0 = m[0][0], d1 = m[1][1], d2 = m[2][2], t;
        if (d0 > d1) { t = d0; d0 = d1; d1 = t; }
        if (d1 > d2) { t = d1; d1 = d2; d2 = t; }
        if (d0 > d1) { t = d0; d0 = d1; d1 = t; }
        ev[0] = d0; ev[1] = d1; ev[2] = d2;
        return;
    }
    const double q = (m[0][0] + m[1][1] + m[2][2]) / 3.0;
    const double p2 = (m[0][0] - q) * (m[0][0] - q) + (m[1][1] - q) * (m[1][1] - q) +
                      (m[2][2] - q) * (m[2][2] - q) + 2.0 * p1;
    const double p = sqrt(p2 / 6.0);
    const double inv_p = 1.0 / p;
    D33 B;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) B.m[i][j] = (m[i][j] - (i == j ? q : 0.0)) * inv_p;
    double r = m33_det(B) / 2.0;
    r = fmax(-1.0, fmin(1.0, r));
    const double phi = acos(r) / 3.0;
    const double e_hi = q + 2.0 * p * cos(phi);
    const double e_lo = q + 2.0 * p * cos(phi + 2.0 * 3.14159265358979323846 / 3.0);
    ev[0] = e_lo;
    ev[2] = e_hi;
    ev[1] = 3.0 * q - e_lo - e_hi;
}

// x86-64 cvttsd2si semantics for static_cast<int>(double): NaN and
// out-of-range values become INT_MIN (render.hpp:123-126 rely on it for
// non-finite centers, which then fail the bounds test and are culled).
__device__ __forceinline__ int x86_trunc_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000;
    return (int)v;
}

// quat_to_rotation (vec.hpp:183-199). Returns false for a zero / non-finite norm.
__device__ __forceinline__ bool quat_rotation(double qw, double qx, double qy, double qz, D33& r) {
    const double n = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (!(n > 0.0) || !isfinite(n)) return false;
    const double w = qw / n, x = qx / n, y = qy / n, z = qz / n;
    r.m[0][0] = 1.0 - 2.0 * (y * y + z * z);
    r.m[0][1] = 2.0 * (x * y - w * z);
    r.m[0][2] = 2.0 * (x * z + w * y);
    r.m[1][0] = 2.0 * (x * y + w * z);
    r.m[1][1] = 1.0 - 2.0 * (x * x + z * z);
    r.m[1][2] = 2.0 * (y * z - w * x);
    r.m[2][0] = 2.0 * (x * z - w * y);
    r.m[2][1] = 2.0 * (y * z + w * x);
    r.m[2][2] = 1.0 - 2.0 * (x * x + y * y);
    return true;
}

// covariance_from_scale_rotation (core.hpp:165-173): R diag((mod s)^2) R^T.
// R*diag is formed entrywise: the reference's full product only adds exact
// zeros to each entry, so the values are identical.
__device__ __forceinline__ int world_covariance(const double p[11], double mod, D33& sigma,
                                                D33& rot, D3& scale) {
    scale = {exp(p[3]), exp(p[4]), exp(p[5])};
    if (!(scale.x > 0.0) || !(scale.y > 0.0) || !(scale.z > 0.0) || !(mod > 0.0))
        return kErrInvalid;
    if (!quat_rotation(p[6], p[7], p[8], p[9], rot)) return kErrInvalid;
    const double sx = mod * scale.x, sy = mod * scale.y, sz = mod * scale.z;
    const double s2[3] = {sx * sx, sy * sy, sz * sz};
    D33 rs;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) rs.m[i][j] = rot.m[i][j] * s2[j];
    sigma = m33_mul(rs, m33_t(rot));
    return kErrNone;
}

// invert_covariance (core.hpp:184-198) with the scale-ratio shortcut above.
__device__ __forceinline__ int invert_cov(const D33& sigma, const D3& scale, double mod,
                                          D33& inv) {
    const double smax = fmax(scale.x, fmax(scale.y, scale.z));
    const double smin = fmin(scale.x, fmin(scale.y, scale.z));
    const double ratio = (smax / smin) * (smax / smin);
    const bool certainly_ok = ratio <= 1e6 && mod * smin > 1e-100 && mod * smax < 1e100;
    D33 s = sigma;
    if (!certainly_ok) {
        double ev[3];
        m33_sym_eig(sigma, ev);
        if (!(ev[0] > 0.0) || ev[2] / ev[0] > 1e12) {
            const double eps = 1e-9 * (sigma.m[0][0] + sigma.m[1][1] + sigma.m[2][2]) / 3.0;
            if (!(eps > 0.0)) return kErrDegenerate;
            for (int i = 0; i < 3; ++i) s.m[i][i] += eps;
            m33_sym_eig(s, ev);
            if (!(ev[0] > 0.0)) return kErrDegenerate;
        }
    }
    inv = m33_inverse(s);
    return kErrNone;
}

// Per-primitive state of one slice (PreparedGaussian, render.hpp:68-79).
struct Focus {
    double alpha, op, alpha_tilde, det2;
    D3 mu_c, mu_e;
    D33 A;    // Sigma_c^-1 (floored)
    D33 Se;   // Sigma_e
    double cov_a, cov_b, cov_c, cov_d;
    double con_a, con_b, con_c, con_d;
    int lo_x, hi_x, lo_y, hi_y;
};

enum FocusResult : int { kSurvive = 0, kCulled = -1 };

// prepare_gaussians body (render.hpp:91-130). Returns kSurvive, kCulled or a
// DevErr code (> 0).
__device__ __forceinline__ int focus_prepare(const double p[11], const SliceArgs& s, Focus& f) {
    f.alpha = 1.0 / (1.0 + exp(-p[10]));
    D33 sigma, rot;
    D3 scale;
    int e = world_covariance(p, s.mod, sigma, rot, scale);
    if (e) return e;
    const D3 mu = {p[0], p[1], p[2]};
    D33 sigma_c;
    if (s.identity_rot) {
        // R_c = I: R mu = mu and R Sigma R^T = Sigma exactly (only +0 terms).
        f.mu_c = {mu.x + s.t[0], mu.y + s.t[1], mu.z + s.t[2]};
        sigma_c = sigma;
    } else {
        D33 Rc;
#pragma unroll
        for (int i = 0; i < 9; ++i) Rc.m[i / 3][i % 3] = s.R[i];
        const D3 rm = m33_mulv(Rc, mu);
        f.mu_c = {rm.x + s.t[0], rm.y + s.t[1], rm.z + s.t[2]};
        sigma_c = m33_mul(m33_mul(Rc, sigma), m33_t(Rc));
    }
    e = invert_cov(sigma_c, scale, s.mod, f.A);
    if (e) return e;
    D33 b = f.A;
    b.m[2][2] += 1.0 / (s.sigma_z * s.sigma_z);
    f.Se = m33_inverse(b);
    const D3 a_mu = m33_mulv(f.A, f.mu_c);
    f.mu_e = m33_mulv(f.Se, a_mu);
    const double q = dot3(f.mu_c, a_mu) - dot3(f.mu_e, m33_mulv(b, f.mu_e));
    f.op = exp(-0.5 * q);
    if (f.alpha * f.op < s.tau) return kCulled;

    f.cov_a = f.Se.m[0][0];
    f.cov_b = f.Se.m[0][1];
    f.cov_c = f.Se.m[1][0];
    f.cov_d = f.Se.m[1][1];
    f.det2 = f.cov_a * f.cov_d - f.cov_b * f.cov_c;
    if (!(f.det2 > 0.0)) return kErrDegenerate;
    f.con_a = f.cov_d / f.det2;
    f.con_b = -f.cov_b / f.det2;
    f.con_c = -f.cov_c / f.det2;
    f.con_d = f.cov_a / f.det2;
    f.alpha_tilde = f.alpha * f.op / sqrt(f.det2);

    const double m = 0.5 * (f.cov_a + f.cov_d);
    const double r = sqrt(0.25 * (f.cov_a - f.cov_d) * (f.cov_a - f.cov_d) + f.cov_b * f.cov_b);
    const double hi_ev = m + r;
    const double radius = s.footprint * sqrt(fmax(hi_ev, 0.0));
    const double cx = f.mu_e.x / s.sx + s.ppx;
    const double cy = f.mu_e.y / s.sy + s.ppy;
    const double rx = radius / s.sx;
    const double ry = radius / s.sy;
    f.lo_x = max(0, x86_trunc_int(ceil(cx - rx)));
    f.hi_x = min(s.W - 1, x86_trunc_int(floor(cx + rx)));
    f.lo_y = max(0, x86_trunc_int(ceil(cy - ry)));
    f.hi_y = min(s.H - 1, x86_trunc_int(floor(cy + ry)));
    if (f.lo_x > f.hi_x || f.lo_y > f.hi_y) return kCulled;
    return kSurvive;
}

// ---------------------------------------------------------------------------
// Fast path: closed forms in fp32 (mu_c and mu_2d in fp64), used when the
// result provably equals the reference's decision; anything near a decision
// boundary (cull threshold, integer pixel bound) returns kAmbiguous and is
// recomputed by focus_prepare above.
//   Sigma_e = Sigma_c - u u^T / den, u = Sigma_c e3, den = sigma_z^2 + Sigma_c,zz
//   mu_e    = mu_c - u * mu_c,z / den,  q = mu_c,z^2 / den
// The reference evaluates the same quantities through two 3x3 inverses
// (render.hpp:99-106); they agree to ~1e-9 relative, far inside the margins.
// ---------------------------------------------------------------------------
enum FastResult : int { kFastSurvive = 0, kFastCulled = -1, kAmbiguous = 1 };

struct FastFocus {
    float alpha, op, det2;
    float cov_a, cov_b, cov_d;     // Sigma_2d
    float con_a, con_b, con_d;     // Sigma_2d^-1
    float u[3], den, r;            // u = Sigma_c e3, r = mu_c,z / den
    float Rc[9];                   // R_c R(q): Gaussian axes in camera frame
    float ms[3];                   // mod * scale
};

// SurvivorRecord::gidx bit 31 flags survivors decided by the reference-order
// fp64 path (their chain also runs in fp64).
constexpr uint32_t kExactFlag = 0x80000000u;

__device__ __forceinline__ bool near_integer(double v, double tol) {
    return fabs(v - rint(v)) < tol;
}

// Decision-grade fast path in fp64 closed form: no 3x3 inverses, no
// trigonometric eigenvalues, one division per quantity. Its values differ from
// the reference's two-inverse evaluation by the reference's own rounding noise
// (<= cond * 1e-16 relative), so the ambiguity bands below are ~1e-7 px /
// 1e-9 relative: the reference-order path (focus_prepare) essentially never
// runs. Fills the survivor record on kFastSurvive.
__device__ __forceinline__ int fast_decide(const float pf[11], const SliceArgs& s,
                                           SurvivorRecord& rec) {
    float sum = pf[0];
#pragma unroll
    for (int k = 1; k < 11; ++k) sum += pf[k];
    if (!isfinite(sum)) return kAmbiguous;
    const float lmax = fmaxf(pf[3], fmaxf(pf[4], pf[5])), lmin = fminf(pf[3], fminf(pf[4], pf[5]));
    if (!(lmax < 30.f && lmin > -30.f && lmax - lmin < 6.2f)) return kAmbiguous;
    if (!(s.mod > 1e-6 && s.mod < 1e6)) return kAmbiguous;
    const double q0 = pf[6], q1 = pf[7], q2 = pf[8], q3 = pf[9];
    const double qn2 = q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3;
    if (!(qn2 > 1e-20 && qn2 < 1e20)) return kAmbiguous;
    const double iqn = rsqrt(qn2);
    const double w = q0 * iqn, x = q1 * iqn, y = q2 * iqn, z = q3 * iqn;
    const double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                         2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                         2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    const double ms[3] = {s.mod * exp((double)pf[3]), s.mod * exp((double)pf[4]), s.mod * exp((double)pf[5])};
    double C[9], mc[3];
    if (s.identity_rot) {
#pragma unroll
        for (int i = 0; i < 9; ++i) C[i] = R[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) mc[i] = (double)pf[i] + s.t[i];
    } else {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                C[3 * i + j] = s.R[3 * i] * R[j] + s.R[3 * i + 1] * R[3 + j] + s.R[3 * i + 2] * R[6 + j];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            mc[i] = s.R[3 * i] * (double)pf[0] + s.R[3 * i + 1] * (double)pf[1] +
                    s.R[3 * i + 2] * (double)pf[2] + s.t[i];
    }
    const double m0 = ms[0] * ms[0], m1 = ms[1] * ms[1], m2 = ms[2] * ms[2];
    const double sxx = C[0] * C[0] * m0 + C[1] * C[1] * m1 + C[2] * C[2] * m2;
    const double sxy = C[0] * C[3] * m0 + C[1] * C[4] * m1 + C[2] * C[5] * m2;
    const double syy = C[3] * C[3] * m0 + C[4] * C[4] * m1 + C[5] * C[5] * m2;
    const double sxz = C[0] * C[6] * m0 + C[1] * C[7] * m1 + C[2] * C[8] * m2;
    const double syz = C[3] * C[6] * m0 + C[4] * C[7] * m1 + C[5] * C[8] * m2;
    const double szz = C[6] * C[6] * m0 + C[7] * C[7] * m1 + C[8] * C[8] * m2;
    const double den = s.sigma_z * s.sigma_z + szz;
    const double iden = 1.0 / den;
    const double r = mc[2] * iden;
    const double q = mc[2] * r;
    const double alpha = 1.0 / (1.0 + exp(-(double)pf[10]));
    const double op = exp(-0.5 * q);
    // condition number of Sigma_c (exact from the scales) bounds the
    // reference's own rounding noise in q, mu_e and Sigma_e
    const double smin = fmin(ms[0], fmin(ms[1], ms[2])), smax = fmax(ms[0], fmax(ms[1], ms[2]));
    const double ratio = smax / smin;
    const double cond = ratio * ratio;
    const double mu2 = mc[0] * mc[0] + mc[1] * mc[1] + mc[2] * mc[2];
    if (s.tau > 0.0) {  // alpha * op < tau (render.hpp:107) with a relative noise band
        const double ao = alpha * op;
        const double band = s.tau * (1e-9 + 1e-13 * (fabs(q) + mu2 / (smin * smin)));
        if (ao < s.tau - band) return kFastCulled;
        if (!(ao > s.tau + band)) return kAmbiguous;
    }
    const double cov_a = sxx - sxz * sxz * iden;
    const double cov_b = sxy - sxz * syz * iden;
    const double cov_d = syy - syz * syz * iden;
    if (!(cov_a > 1e-3 * sxx && cov_d > 1e-3 * syy)) return kAmbiguous;
    const double det2 = cov_a * cov_d - cov_b * cov_b;
    if (!(det2 > 1e-6 * cov_a * cov_d)) return kAmbiguous;
    const double mu2x = mc[0] - sxz * r, mu2y = mc[1] - syz * r;
    const double hm = 0.5 * (cov_a + cov_d);
    const double hr = sqrt(0.25 * (cov_a - cov_d) * (cov_a - cov_d) + cov_b * cov_b);
    const double radius = s.footprint * sqrt(fmax(hm + hr, 0.0));
    const double cx = mu2x * s.inv_sx + s.ppx, cy = mu2y * s.inv_sy + s.ppy;
    const double rx = radius * s.inv_sx, ry = radius * s.inv_sy;
    // bounds (render.hpp:116-126) are exact unless c +- r lies within the
    // reference's rounding noise of an integer
    const double tol = 1e-9 + 1e-14 * cond * (fabs(cx) + fabs(cy) + rx + ry + sqrt(mu2) / fmin(s.sx, s.sy));
    if (near_integer(cx - rx, tol) || near_integer(cx + rx, tol) || near_integer(cy - ry, tol) ||
        near_integer(cy + ry, tol))
        return kAmbiguous;
    if (!(fabs(cx) + rx < 1e9 && fabs(cy) + ry < 1e9)) return kAmbiguous;
    const int lo_x = max(0, (int)ceil(cx - rx)), hi_x = min(s.W - 1, (int)floor(cx + rx));
    const int lo_y = max(0, (int)ceil(cy - ry)), hi_y = min(s.H - 1, (int)floor(cy + ry));
    if (lo_x > hi_x || lo_y > hi_y) return kFastCulled;
    const double idet = 1.0 / det2;
    rec.mu2d_x = mu2x;
    rec.mu2d_y = mu2y;
    rec.conic_a = (float)(cov_d * idet);
    rec.conic_b = (float)(-cov_b * idet);
    rec.conic_d = (float)(cov_a * idet);
    rec.alpha_tilde = (float)(alpha * op * rsqrt(det2));
    rec.lo_x = (uint16_t)lo_x;
    rec.hi_x = (uint16_t)hi_x;
    rec.lo_y = (uint16_t)lo_y;
    rec.hi_y = (uint16_t)hi_y;
    return kFastSurvive;
}

// fp32 state of a fast-path survivor for the inverse-free backward (no
// decisions: K_exact already made them and flagged the record).
__device__ __forceinline__ void fast_state(const float pf[11], const SliceArgs& s, FastFocus& f) {
    const float qn2 = pf[6] * pf[6] + pf[7] * pf[7] + pf[8] * pf[8] + pf[9] * pf[9];
    const float inv = rsqrtf(qn2);
    const float w = pf[6] * inv, x = pf[7] * inv, y = pf[8] * inv, z = pf[9] * inv;
    float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                  2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                  2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
    const float mod = (float)s.mod;
    f.ms[0] = __expf(pf[3]) * mod;
    f.ms[1] = __expf(pf[4]) * mod;
    f.ms[2] = __expf(pf[5]) * mod;
    double mc[3];
    if (s.identity_rot) {
#pragma unroll
        for (int i = 0; i < 9; ++i) f.Rc[i] = R[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) mc[i] = (double)pf[i] + s.t[i];
    } else {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                f.Rc[3 * i + j] = (float)s.R[3 * i] * R[j] + (float)s.R[3 * i + 1] * R[3 + j] +
                                  (float)s.R[3 * i + 2] * R[6 + j];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            mc[i] = s.R[3 * i] * (double)pf[0] + s.R[3 * i + 1] * (double)pf[1] +
                    s.R[3 * i + 2] * (double)pf[2] + s.t[i];
    }
    // Sigma_c = Rc diag(ms^2) Rc^T (symmetric entries needed: xx, xy, yy, xz, yz, zz)
    const float m0 = f.ms[0] * f.ms[0], m1 = f.ms[1] * f.ms[1], m2 = f.ms[2] * f.ms[2];
    const float* C = f.Rc;
    const float sxx = C[0] * C[0] * m0 + C[1] * C[1] * m1 + C[2] * C[2] * m2;
    const float sxy = C[0] * C[3] * m0 + C[1] * C[4] * m1 + C[2] * C[5] * m2;
    const float syy = C[3] * C[3] * m0 + C[4] * C[4] * m1 + C[5] * C[5] * m2;
    const float sxz = C[0] * C[6] * m0 + C[1] * C[7] * m1 + C[2] * C[8] * m2;
    const float syz = C[3] * C[6] * m0 + C[4] * C[7] * m1 + C[5] * C[8] * m2;
    const float szz = C[6] * C[6] * m0 + C[7] * C[7] * m1 + C[8] * C[8] * m2;
    f.u[0] = sxz;
    f.u[1] = syz;
    f.u[2] = szz;
    f.den = (float)(s.sigma_z * s.sigma_z) + szz;
    const float mcz = (float)mc[2];
    f.r = mcz / f.den;
    const float q = mcz * f.r;
    const float raw = pf[10];
    f.alpha = 1.f / (1.f + __expf(-raw));
    f.op = __expf(-0.5f * q);
    const float id = 1.f / f.den;
    f.cov_a = sxx - sxz * sxz * id;
    f.cov_b = sxy - sxz * syz * id;
    f.cov_d = syy - syz * syz * id;
    f.det2 = f.cov_a * f.cov_d - f.cov_b * f.cov_b;
    const float idet = 1.f / f.det2;
    f.con_a = f.cov_d * idet;
    f.con_b = -f.cov_b * idet;
    f.con_d = f.cov_a * idet;
}

// Inverse-free camera-space backward for a fast-path survivor (same math as
// camera_space_backward, backward.hpp:55-89, rewritten with A Sigma_e =
// I - e3 u^T/den and A delta = e3 r, which need no matrix inverse), then the
// world chain (grad_chain.hpp:48-77). fp32 throughout.
__device__ __forceinline__ void fast_backward(const float pf[11], const FastFocus& f,
                                              const double accd[6], const SliceArgs& s,
                                              float g[11], float dl_dmu[3]) {
    const float acc[6] = {(float)accd[0], (float)accd[1], (float)accd[2],
                          (float)accd[3], (float)accd[4], (float)accd[5]};
    const float sqd = sqrtf(f.det2);
    const float d_alpha = acc[0] * f.op / sqd;
    const float d_op = acc[0] * f.alpha / sqd;
    const float d_det = acc[0] * f.alpha * f.op * (-0.5f) / (f.det2 * sqd);
    // dL/dcov2d = -conic X conic + conic (d_det det2), X = dL/dconic
    const float ca = f.con_a, cb = f.con_b, cd = f.con_d;
    const float xa = acc[3], xb = acc[4], xd = acc[5];
    const float ta = ca * xa + cb * xb, tb = ca * xb + cb * xd;
    const float tc = cb * xa + cd * xb, td = cb * xb + cd * xd;
    const float k = d_det * f.det2;
    const float g00 = -(ta * ca + tb * cb) + ca * k;
    const float g01 = -(ta * cb + tb * cd) + cb * k;
    const float g10 = -(tc * ca + td * cb) + cb * k;
    const float g11 = -(tc * cb + td * cd) + cd * k;
    const float gq = d_op * (-0.5f) * f.op;
    const float ug = (f.u[0] * acc[1] + f.u[1] * acc[2]) / f.den;
    // A Sigma_e g = g - e3 (u.g)/den ; A delta = e3 r
    const float seg[3] = {acc[1], acc[2], -ug};
    float dmc[3] = {seg[0], seg[1], seg[2] + 2.f * gq * f.r};
    // M = (A Se g)(A d)^T + gq (A d)(A d)^T - (A Se) G (A Se)^T, P = A Se
    // P rows: e0, e1, e2 - u/den ; G = [[g00,g01,0],[g10,g11,0],[0,0,0]]
    const float id = 1.f / f.den;
    const float p20 = -f.u[0] * id, p21 = -f.u[1] * id;
    // (P G): rows 0,1 = G rows; row 2 = p20*G0 + p21*G1
    const float pg[3][2] = {{g00, g01}, {g10, g11}, {p20 * g00 + p21 * g10, p20 * g01 + p21 * g11}};
    // (P G P^T)[i][j] = pg[i][0]*P[j][0] + pg[i][1]*P[j][1]; P[j] = (1,0,0),(0,1,0),(p20,p21,1)
    float T3[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        T3[i][0] = pg[i][0];
        T3[i][1] = pg[i][1];
        T3[i][2] = pg[i][0] * p20 + pg[i][1] * p21;
    }
    float M[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[i][j] = -T3[i][j];
#pragma unroll
    for (int i = 0; i < 3; ++i) M[i][2] += seg[i] * f.r;
    M[2][2] += gq * f.r * f.r;
    float dS[3][3];  // dL/dSigma_c = -sym(M)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) dS[i][j] = -0.5f * (M[i][j] + M[j][i]);
    // camera -> world
    float dW[3][3];
    if (s.identity_rot) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            dl_dmu[i] = dmc[i];
#pragma unroll
            for (int j = 0; j < 3; ++j) dW[i][j] = dS[i][j];
        }
    } else {
        float Rc[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) Rc[i] = (float)s.R[i];
#pragma unroll
        for (int i = 0; i < 3; ++i) dl_dmu[i] = Rc[i] * dmc[0] + Rc[3 + i] * dmc[1] + Rc[6 + i] * dmc[2];
        float tmp[3][3];  // Rc^T dS
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                tmp[i][j] = Rc[i] * dS[0][j] + Rc[3 + i] * dS[1][j] + Rc[6 + i] * dS[2][j];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j)
                dW[i][j] = tmp[i][0] * Rc[j] + tmp[i][1] * Rc[3 + j] + tmp[i][2] * Rc[6 + j];
    }
    // chain_world_covariance (grad_chain.hpp:48-77): M = R diag(ms), dL/dM = 2 dW M
    const float qn = sqrtf(pf[6] * pf[6] + pf[7] * pf[7] + pf[8] * pf[8] + pf[9] * pf[9]);
    const float iq = 1.f / qn;
    const float q[4] = {pf[6] * iq, pf[7] * iq, pf[8] * iq, pf[9] * iq};
    const float w = q[0], x = q[1], y = q[2], z = q[3];
    const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y)},
                           {2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x)},
                           {2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)}};
    float dM[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            dM[i][j] = 2.f * (dW[i][0] * R[0][j] + dW[i][1] * R[1][j] + dW[i][2] * R[2][j]) * f.ms[j];
    const float mod = (float)s.mod;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const float a = R[0][j] * dM[0][j] + R[1][j] * dM[1][j] + R[2][j] * dM[2][j];
        g[3 + j] = a * f.ms[j];  // = a * mod * s_j
    }
    (void)mod;
    float gr[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) gr[i][j] = dM[i][j] * f.ms[j];
    float dq[4];
    dq[0] = 2.f * (-z * gr[0][1] + y * gr[0][2] + z * gr[1][0] - x * gr[1][2] - y * gr[2][0] + x * gr[2][1]);
    dq[1] = 2.f * (y * gr[0][1] + z * gr[0][2] + y * gr[1][0] - 2.f * x * gr[1][1] - w * gr[1][2] +
                   z * gr[2][0] + w * gr[2][1] - 2.f * x * gr[2][2]);
    dq[2] = 2.f * (-2.f * y * gr[0][0] + x * gr[0][1] + w * gr[0][2] + x * gr[1][0] + z * gr[1][2] -
                   w * gr[2][0] + z * gr[2][1] - 2.f * y * gr[2][2]);
    dq[3] = 2.f * (-2.f * z * gr[0][0] - w * gr[0][1] + x * gr[0][2] + w * gr[1][0] - 2.f * z * gr[1][1] +
                   y * gr[1][2] + x * gr[2][0] + y * gr[2][1]);
    const float along = dq[0] * q[0] + dq[1] * q[1] + dq[2] * q[2] + dq[3] * q[3];
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) g[6 + kq] = (dq[kq] - q[kq] * along) * iq;
    g[0] = dl_dmu[0];
    g[1] = dl_dmu[1];
    g[2] = dl_dmu[2];
    g[10] = d_alpha * (f.alpha * (1.f - f.alpha));
}

// rotation_backward (grad_chain.hpp:27-40): dL/dq-hat for R(q-hat).
__device__ __forceinline__ void rotation_backward(const double q[4], const D33& gm, double out[4]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const auto& g = gm.m;
    out[0] = 2.0 * (-z * g[0][1] + y * g[0][2] + z * g[1][0] - x * g[1][2] - y * g[2][0] +
                    x * g[2][1]);
    out[1] = 2.0 * (y * g[0][1] + z * g[0][2] + y * g[1][0] - 2.0 * x * g[1][1] - w * g[1][2] +
                    z * g[2][0] + w * g[2][1] - 2.0 * x * g[2][2]);
    out[2] = 2.0 * (-2.0 * y * g[0][0] + x * g[0][1] + w * g[0][2] + x * g[1][0] +
                    z * g[1][2] - w * g[2][0] + z * g[2][1] - 2.0 * y * g[2][2]);
    out[3] = 2.0 * (-2.0 * z * g[0][0] - w * g[0][1] + x * g[0][2] + w * g[1][0] -
                    2.0 * z * g[1][1] + y * g[1][2] + x * g[2][0] + y * g[2][1]);
}

// chain_world_covariance (grad_chain.hpp:48-77): dL/dSigma (world) ->
// dL/d log-scale and dL/d raw quaternion (gauge-projected).
__device__ __forceinline__ void chain_world(const double p[11], const D33& dl_dsigma, double mod,
                                            double d_ls[3], double d_q[4]) {
    const double qn = sqrt(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
    const double inv_qn = 1.0 / qn;  // GaussianPrimitive::rotation(), core.hpp:42-46
    const double q[4] = {p[6] * inv_qn, p[7] * inv_qn, p[8] * inv_qn, p[9] * inv_qn};
    D33 r;
    quat_rotation(q[0], q[1], q[2], q[3], r);
    const double s[3] = {exp(p[3]), exp(p[4]), exp(p[5])};
    const double ms[3] = {mod * s[0], mod * s[1], mod * s[2]};
    const D33 sym2 = m33_add(dl_dsigma, m33_t(dl_dsigma));
    D33 mm;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) mm.m[i][j] = r.m[i][j] * ms[j];
    const D33 dl_dm = m33_mul(sym2, mm);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) acc += r.m[i][j] * dl_dm.m[i][j];
        d_ls[j] = acc * mod * s[j];
    }
    D33 dl_dr;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) dl_dr.m[i][j] = dl_dm.m[i][j] * ms[j];
    double dq[4];
    rotation_backward(q, dl_dr, dq);
    const double along = dq[0] * q[0] + dq[1] * q[1] + dq[2] * q[2] + dq[3] * q[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) d_q[k] = (dq[k] - q[k] * along) * inv_qn;
}

// camera_space_backward (backward.hpp:55-89) + world chain (:148-166).
// acc = {A-tilde sum, dmu2d.x, dmu2d.y, c_xx, c_xy, c_yy}. Writes the 11
// stored-parameter gradients and dL/dmu (world) for the screen statistics.
__device__ __forceinline__ void focus_backward(const double p[11], const Focus& f,
                                               const double acc[6], const SliceArgs& s,
                                               double g[11], D3& dl_dmu) {
    const double sqrt_det = sqrt(f.det2);
    const double d_alpha = acc[0] * f.op / sqrt_det;
    const double d_opacity = acc[0] * f.alpha / sqrt_det;
    const double d_det = acc[0] * f.alpha * f.op * (-0.5) / (f.det2 * sqrt_det);

    // cm = conic * dL/dconic * conic; dL/dcov2d = -cm + conic * (d_det * det2)
    const double ca = f.con_a, cb = f.con_b, cc = f.con_c, cd = f.con_d;
    const double xa = acc[3], xb = acc[4], xc = acc[4], xd = acc[5];
    const double t_a = ca * xa + cb * xc, t_b = ca * xb + cb * xd;
    const double t_c = cc * xa + cd * xc, t_d = cc * xb + cd * xd;
    const double cm_a = t_a * ca + t_b * cc, cm_b = t_a * cb + t_b * cd;
    const double cm_c = t_c * ca + t_d * cc, cm_d = t_c * cb + t_d * cd;
    const double k = d_det * f.det2;
    D33 gse = {};
    gse.m[0][0] = cm_a * -1.0 + ca * k;
    gse.m[0][1] = cm_b * -1.0 + cb * k;
    gse.m[1][0] = cm_c * -1.0 + cc * k;
    gse.m[1][1] = cm_d * -1.0 + cd * k;
    const D3 g_mu_e = {acc[1], acc[2], 0.0};

    const double g_q = d_opacity * (-0.5) * f.op;
    const D3 delta = {f.mu_c.x - f.mu_e.x, f.mu_c.y - f.mu_e.y, f.mu_c.z - f.mu_e.z};
    const D3 se_g = m33_mulv(f.Se, g_mu_e);
    const D3 a1 = m33_mulv(f.A, se_g);
    const D3 a2 = m33_mulv(f.A, delta);
    const D3 dl_dmu_c = {a1.x + a2.x * (2.0 * g_q), a1.y + a2.y * (2.0 * g_q),
                         a1.z + a2.z * (2.0 * g_q)};
    D33 dl_da = m33_add(outer3(se_g, delta), m33_scale(outer3(delta, delta), g_q));
    const D33 sgs = m33_mul(m33_mul(f.Se, gse), f.Se);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) dl_da.m[i][j] -= sgs.m[i][j];
    dl_da = m33_scale(m33_add(dl_da, m33_t(dl_da)), 0.5);
    const D33 dl_dsc = m33_scale(m33_mul(m33_mul(f.A, dl_da), f.A), -1.0);

    D33 dl_dsigma;
    if (s.identity_rot) {
        dl_dmu = dl_dmu_c;
        dl_dsigma = dl_dsc;
    } else {
        D33 Rc;
#pragma unroll
        for (int i = 0; i < 9; ++i) Rc.m[i / 3][i % 3] = s.R[i];
        const D33 rct = m33_t(Rc);
        dl_dmu = m33_mulv(rct, dl_dmu_c);
        dl_dsigma = m33_mul(m33_mul(rct, dl_dsc), Rc);
    }
    double d_ls[3], d_q[4];
    chain_world(p, dl_dsigma, s.mod, d_ls, d_q);
    g[0] = dl_dmu.x;
    g[1] = dl_dmu.y;
    g[2] = dl_dmu.z;
    g[3] = d_ls[0];
    g[4] = d_ls[1];
    g[5] = d_ls[2];
    g[6] = d_q[0];
    g[7] = d_q[1];
    g[8] = d_q[2];
    g[9] = d_q[3];
    g[10] = d_alpha * (f.alpha * (1.0 - f.alpha));
}

}  // namespace gpk
