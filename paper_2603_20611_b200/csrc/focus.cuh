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
