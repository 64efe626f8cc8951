// cull.cu — the streaming cull of prepare_gaussians (render.hpp:107): K_filter,
// its batched-step form over several slice poses and the training step's
// Adam + next-slice cull. fp32 throughout with conservative margins (a culled
// Gaussian is one the reference culls), so it is built with FMA contraction;
// the reference-order fp64 code lives in prep.cu (--fmad=false).
#include <algorithm>

#include "adam.cuh"
#include "common.cuh"

namespace gpk {

namespace {

// fp32 certain-cull: true only if the exact reference test alpha*op < tau
// (render.hpp:107) is guaranteed to hold.
__device__ __forceinline__ bool certainly_culled(const float p[11], const SliceArgs& s,
                                                 float log_tau, float mod_f, float sz2) {
#pragma unroll
    for (int k = 0; k < 11; ++k)
        if (!isfinite(p[k])) return false;
    if (fabsf(p[3]) > 40.f || fabsf(p[4]) > 40.f || fabsf(p[5]) > 40.f) return false;
    const float qn2 = p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9];
    if (!(qn2 > 1e-20f && qn2 < 1e20f)) return false;
    const float s0 = __expf(p[3]) * mod_f, s1 = __expf(p[4]) * mod_f, s2 = __expf(p[5]) * mod_f;
    const float smax = fmaxf(s0, fmaxf(s1, s2)), smin = fminf(s0, fminf(s1, s2));
    if (!(smax < 5e2f * smin)) return false;  // (smax/smin)^2 < 2.5e5: far inside the 1e6 guard
    const float inv = rsqrtf(qn2);
    const float w = p[6] * inv, x = p[7] * inv, y = p[8] * inv, z = p[9] * inv;
    const float r00 = 1.f - 2.f * (y * y + z * z), r01 = 2.f * (x * y - w * z), r02 = 2.f * (x * z + w * y);
    const float r10 = 2.f * (x * y + w * z), r11 = 1.f - 2.f * (x * x + z * z), r12 = 2.f * (y * z - w * x);
    const float r20 = 2.f * (x * z - w * y), r21 = 2.f * (y * z + w * x), r22 = 1.f - 2.f * (x * x + y * y);
    const float e0 = (float)s.R[6], e1 = (float)s.R[7], e2 = (float)s.R[8];
    const float pr0 = e0 * r00 + e1 * r10 + e2 * r20;
    const float pr1 = e0 * r01 + e1 * r11 + e2 * r21;
    const float pr2 = e0 * r02 + e1 * r12 + e2 * r22;
    const float var = (s0 * pr0) * (s0 * pr0) + (s1 * pr1) * (s1 * pr1) + (s2 * pr2) * (s2 * pr2);
    const double mcz = s.R[6] * (double)p[0] + s.R[7] * (double)p[1] + s.R[8] * (double)p[2] + s.t[2];
    const float mczf = (float)mcz;
    const float q = mczf * mczf / (sz2 + var);
    const float raw = p[10];
    const float log_alpha = raw >= 0.f ? -log1pf(__expf(-raw)) : raw - log1pf(__expf(raw));
    // Noise of the reference's q = mu_c^T A mu_c - mu_e^T B mu_e (render.hpp:105):
    // ~64 ulp of |mu_c|^2 * ||A||, ||A|| <= 1/(mod*smin)^2.
    const float mcx = (float)(s.R[0] * (double)p[0] + s.R[1] * (double)p[1] + s.R[2] * (double)p[2] + s.t[0]);
    const float mcy = (float)(s.R[3] * (double)p[0] + s.R[4] * (double)p[1] + s.R[5] * (double)p[2] + s.t[1]);
    const float mu2 = mcx * mcx + mcy * mcy + mczf * mczf;
    const float noise = 2e-14f * mu2 / (smin * smin);
    const float thresh = log_alpha - log_tau;
    const float margin = 2e-3f + 2e-5f * fabsf(thresh) + noise;
    return 0.5f * q > thresh + margin;
}

// Cheaper certain-cull for the common case R_c = I (every slice_pose_for_index
// pose): only the third row of R(q) is needed, mu_c,z = mu_z + t_z in fp32
// with t_z split hi/lo, and the guards avoid per-parameter checks (a single
// finiteness test of the parameter sum routes NaN/Inf to the exact path).
struct FilterConsts {
    float log_tau, mod, sz2;
    float tx, ty, tz_hi, tz_lo;
    float mod2, inv_mod2, inv_sz2;   // quick test only
};

__device__ __forceinline__ bool certainly_culled_identity(const float p[11], const FilterConsts& c) {
    float sum = p[0];
#pragma unroll
    for (int k = 1; k < 11; ++k) sum += p[k];
    if (!isfinite(sum)) return false;
    const float lmax = fmaxf(p[3], fmaxf(p[4], p[5])), lmin = fminf(p[3], fminf(p[4], p[5]));
    // |log-scale| <= 40 and (smax/smin) < e^6.2 ~ 490: the exact path's inverse
    // is unfloored there (focus.cuh invert_cov guard 1e3 ratio)
    if (!(lmax < 40.f && lmin > -40.f && lmax - lmin < 6.2f)) return false;
    const float qn2 = p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9];
    if (!(qn2 > 1e-20f && qn2 < 1e20f)) return false;
    const float inv = rsqrtf(qn2);
    const float w = p[6] * inv, x = p[7] * inv, y = p[8] * inv, z = p[9] * inv;
    // third row of R(q): Sigma_c,zz = sum_k (mod s_k)^2 R_2k^2
    const float r0 = 2.f * (x * z - w * y), r1 = 2.f * (y * z + w * x), r2 = 1.f - 2.f * (x * x + y * y);
    const float s0 = __expf(p[3]) * c.mod, s1 = __expf(p[4]) * c.mod, s2 = __expf(p[5]) * c.mod;
    const float var = (s0 * r0) * (s0 * r0) + (s1 * r1) * (s1 * r1) + (s2 * r2) * (s2 * r2);
    const float mcz = (p[2] + c.tz_hi) + c.tz_lo;
    const float den = c.sz2 + var;
    const float q = mcz * mcz / den;
    const float raw = p[10];
    const float log_alpha = raw >= 0.f ? -__logf(1.f + __expf(-raw)) : raw - __logf(1.f + __expf(raw));
    const float mcx = p[0] + c.tx, mcy = p[1] + c.ty;
    const float smin = __expf(lmin) * c.mod;
    const float mu2 = mcx * mcx + mcy * mcy + mcz * mcz;
    // reference cancellation noise (render.hpp:105) + fp32 rounding of mu_c,z
    const float noise = 2e-14f * mu2 / (smin * smin) +
                        4.f * fabsf(mcz) * 1.2e-7f * (fabsf(p[2]) + fabsf(c.tz_hi)) / den;
    const float thresh = log_alpha - c.log_tau;
    const float margin = 2e-3f + 2e-5f * fabsf(thresh) + noise;
    return 0.5f * q > thresh + margin;
}


// Cheapest certain-cull for R_c = I, division-free: lower-bounds q by replacing
// the projected variance Sigma_c,zz with its maximum (mod * s_max)^2, upper-
// bounds the threshold by log alpha <= min(raw, 0) and the margin's noise
// terms by their values at Sigma_c,zz = 0 / s_min. Returns true only if the
// full fp32 test (certainly_culled_identity) culls too:
//   0.5 q > T + M   with q = mcz^2 / den, 0 < sz2 <= den <= den_hi
//   <=  0.5 mcz^2 > X_up * (X_up >= 0 ? den_hi : sz2),  X_up >= T + M.
// Undecided items take the full test, compacted, so the warp does not pay it
// for every Gaussian.
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ bool quick_culled_identity(const float p[11], const FilterConsts& c) {
    // Branch-free (the four items of a lane interleave): the guards are folded
    // into the result with bitwise ANDs instead of early returns.
    // NaN/Inf guard: log-scales (fmaxf/fminf drop NaN), mu_z and alpha_raw
    // (fminf drops NaN) explicitly; mu_x/y propagate into the final compare
    // (false -> not culled) and the quaternion fails the norm range test.
    const bool fin = isfinite(((p[2] + p[3]) + (p[4] + p[5])) + p[10]);
    const float lmax = fmaxf(p[3], fmaxf(p[4], p[5])), lmin = fminf(p[3], fminf(p[4], p[5]));
    const bool scales_ok = (lmax < 40.f) & (lmin > -40.f) & (lmax - lmin < 6.2f);
    const float qn2 = __fmaf_rn(p[6], p[6], __fmaf_rn(p[7], p[7], __fmaf_rn(p[8], p[8], p[9] * p[9])));
    const bool quat_ok = (qn2 > 1e-20f) & (qn2 < 1e20f);
    const float mcz = (p[2] + c.tz_hi) + c.tz_lo;
    const float mcx = p[0] + c.tx, mcy = p[1] + c.ty;
    const float mu2 = __fmaf_rn(mcx, mcx, __fmaf_rn(mcy, mcy, mcz * mcz));
    // e^(2 lmax) mod^2 = (mod s_max)^2 ; e^(-2 lmin) / mod^2 = 1 / (mod s_min)^2
    // (the clamps only keep the exponentials finite where the guards reject)
    // (MUFU.EX2 with flush-to-zero: the arguments stay within +-116, so no
    // denormal range fix-up is needed; ~2 ulp, inside the 2e-4 factor)
    const float den_hi = __fmaf_rn(ex2_ftz(fminf(lmax, 40.f) * 2.8853900817779268f) * c.mod2, 1.0002f, c.sz2);
    const float inv_smin2 = ex2_ftz(fmaxf(lmin, -40.f) * -2.8853900817779268f) * c.inv_mod2 * 1.0002f;
    const float thresh_hi = fminf(p[10], 0.f) - c.log_tau;
    const float noise = __fmaf_rn(2e-14f * mu2, inv_smin2,
                                  4.8e-7f * fabsf(mcz) * (fabsf(p[2]) + fabsf(c.tz_hi)) * c.inv_sz2 * 1.0002f);
    const float x = thresh_hi + (2e-3f + __fmaf_rn(2e-5f, fabsf(thresh_hi) + 0.7f, noise));
    const float x_up = __fmaf_rn(1e-3f, fabsf(x) + noise, x) + 1e-6f;
    const bool culled = 0.5f * mcz * mcz > x_up * (x_up >= 0.f ? den_hi : c.sz2);
    return fin & scales_ok & quat_ok & culled;
}

// ---- lazy training steps: the cull from stale parameters --------------------------
// K_filter of a lazy step (LazyAdam, common.cuh) sees each Gaussian's stored
// parameters, current at t_done <= t, and |true - stored| <= the drift bound of
// the kLazyWindow - 1 last steps per parameter group (position, log-scale, raw
// alpha, quaternion). quick_culled_drift is quick_culled_identity with every
// input at its worst case inside that box, so it culls only what the quick
// test would cull at the true parameters (and so the reference too); the rest
// is brought up to date (replayed, lazy_materialize) and decided exactly as
// the eager K_filter decides it.
struct LazyView {
    LazyAdam L;
    uint64_t cap;
    long long t;             // AdamState::step: the steps the true parameters have seen
    float dmu, dls, dal;     // drift bounds: position, log-scale, raw alpha
    bool all;                // no usable bound (bad state / missing constants): replay everything
};

__device__ __forceinline__ bool quick_culled_drift(const float p[11], const FilterConsts& c, const LazyView& z) {
    const bool fin = isfinite(((p[2] + p[3]) + (p[4] + p[5])) + p[10]) & isfinite(p[0] + p[1]);
    const float lmax = fmaxf(p[3], fmaxf(p[4], p[5])) + z.dls, lmin = fminf(p[3], fminf(p[4], p[5])) - z.dls;
    const bool scales_ok = (lmax < 40.f) & (lmin > -40.f) & (lmax - lmin < 6.2f);
    // renormalised every step: a stored norm near 1 stays away from the guards
    const float qn2 = __fmaf_rn(p[6], p[6], __fmaf_rn(p[7], p[7], __fmaf_rn(p[8], p[8], p[9] * p[9])));
    const bool quat_ok = (qn2 > 0.25f) & (qn2 < 4.f);
    const float az = fabsf((p[2] + c.tz_hi) + c.tz_lo);
    const float dz = __fmaf_rn(2.4e-7f, fabsf(p[2]) + fabsf(c.tz_hi), z.dmu);
    const float mcz_lo = fmaxf(az - dz, 0.f), mcz_hi = az + dz;
    const float mcx = fabsf(p[0] + c.tx) + z.dmu, mcy = fabsf(p[1] + c.ty) + z.dmu;
    const float mu2 = __fmaf_rn(mcx, mcx, __fmaf_rn(mcy, mcy, mcz_hi * mcz_hi)) * 1.0001f;
    const float den_hi = __fmaf_rn(ex2_ftz(fminf(lmax, 40.f) * 2.8853900817779268f) * c.mod2, 1.0003f, c.sz2);
    const float inv_smin2 = ex2_ftz(fmaxf(lmin, -40.f) * -2.8853900817779268f) * c.inv_mod2 * 1.0003f;
    const float thresh_hi = fminf(p[10] + z.dal, 0.f) - c.log_tau;
    const float noise = __fmaf_rn(2e-14f * mu2, inv_smin2,
                                  4.8e-7f * mcz_hi * (fabsf(p[2]) + dz + fabsf(c.tz_hi)) * c.inv_sz2 * 1.0003f);
    const float x = thresh_hi + (2e-3f + __fmaf_rn(2e-5f, fabsf(thresh_hi) + 0.7f, noise));
    const float x_up = __fmaf_rn(1e-3f, fabsf(x) + noise, x) + 2e-6f;
    const float rhs = x_up >= 0.f ? x_up * den_hi * 1.0001f : x_up * c.sz2 * 0.9999f;
    const bool culled = 0.5f * mcz_lo * mcz_lo > rhs;
    return fin & scales_ok & quat_ok & culled;
}

// Gaussian i's true parameters (p: its stored ones in, the replayed ones out).
__device__ __noinline__ void lazy_materialize(const LazyView z, uint32_t i, float p[11]) {
    const LazyAdam& L = z.L;
    const long long td = L.t_done[i];
    if (td >= z.t) return;
    float m[11], v[11];
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        m[k] = L.m[(uint64_t)k * z.cap + i];
        v[k] = L.v[(uint64_t)k * z.cap + i];
    }
    lazy_replay(L, td + 1, z.t, p, m, v);
}

// The drift bounds of the pending steps (one thread; k_adam_consts summed them
// per step into the ring entry of the last step done).
__device__ __forceinline__ LazyView lazy_view(const PrepLaunch& a) {
    LazyView z;
    z.L = a.lazy;
    z.cap = a.cap;
    z.t = *a.lazy.step;
    z.dmu = z.dls = z.dal = 0.f;
    z.all = *a.lazy.bad != 0;
    if (z.t > 0) {
        const AdamConsts& e = a.lazy.ring[z.t % kLazyRing];
        if (e.step != z.t) {
            z.all = true;
        } else {
            z.dmu = e.cum[0];
            z.dal = e.cum[1];
            z.dls = e.cum[2];
            // the quaternion guard of quick_culled_drift needs the renormalised
            // quaternion to stay renormalisable (|delta q| per step well below 1)
            z.all |= !(e.cum[0] < 1e30f && e.cum[1] < 1e30f && e.cum[2] < 1e30f && e.cum[3] < 0.25f);
        }
    }
    return z;
}

// quick_culled_identity split for several poses that differ only in t_z
// (slice_pose_for_index stacks: same R = I, t_x, t_y, PSF, tau, mod): the
// pose-invariant terms once per Gaussian, then a few FMAs per pose. Same
// arithmetic, same verdicts as quick_culled_identity.
struct QuickInv {
    float p2, ap2, mcx, mcy, den_hi, inv_smin2, thr;  // thr = fminf(raw alpha, 0) - log tau
    bool ok;
};
__device__ __forceinline__ QuickInv quick_invariant(const float p[11], const FilterConsts& c) {
    QuickInv q;
    const bool fin = isfinite(((p[2] + p[3]) + (p[4] + p[5])) + p[10]);
    const float lmax = fmaxf(p[3], fmaxf(p[4], p[5])), lmin = fminf(p[3], fminf(p[4], p[5]));
    const bool scales_ok = (lmax < 40.f) & (lmin > -40.f) & (lmax - lmin < 6.2f);
    const float qn2 = __fmaf_rn(p[6], p[6], __fmaf_rn(p[7], p[7], __fmaf_rn(p[8], p[8], p[9] * p[9])));
    const bool quat_ok = (qn2 > 1e-20f) & (qn2 < 1e20f);
    const float mcx = p[0] + c.tx, mcy = p[1] + c.ty;
    q.p2 = p[2];
    q.ap2 = fabsf(p[2]);
    q.mcx = mcx;  // NaN in mu_x/y propagates into the compare (not culled)
    q.mcy = mcy;
    q.den_hi = __fmaf_rn(ex2_ftz(fminf(lmax, 40.f) * 2.8853900817779268f) * c.mod2, 1.0002f, c.sz2);
    q.inv_smin2 = ex2_ftz(fmaxf(lmin, -40.f) * -2.8853900817779268f) * c.inv_mod2 * 1.0002f;
    q.thr = fminf(p[10], 0.f) - c.log_tau;
    q.ok = fin & scales_ok & quat_ok;
    return q;
}
__device__ __forceinline__ bool quick_culled_pose(const QuickInv& q, const FilterConsts& c) {
    const float mcz = (q.p2 + c.tz_hi) + c.tz_lo;
    const float mu2 = __fmaf_rn(q.mcx, q.mcx, __fmaf_rn(q.mcy, q.mcy, mcz * mcz));
    const float noise = __fmaf_rn(2e-14f * mu2, q.inv_smin2,
                                  4.8e-7f * fabsf(mcz) * (q.ap2 + fabsf(c.tz_hi)) * c.inv_sz2 * 1.0002f);
    const float x = q.thr + (2e-3f + __fmaf_rn(2e-5f, fabsf(q.thr) + 0.7f, noise));
    const float x_up = __fmaf_rn(1e-3f, fabsf(x) + noise, x) + 1e-6f;
    const bool culled = 0.5f * mcz * mcz > x_up * (x_up >= 0.f ? q.den_hi : c.sz2);
    return q.ok & culled;
}

// The quick bound for every pose of the step at once (a conservative "culled
// by every pose", so the union test runs only near the poses): the noise term
// bounded with the largest |mu_c,z| over the poses (at the smallest or the
// largest t_z), x_up with it (x_up grows with the noise), and the smallest
// |mu_c,z| by the hull [mu_c,z(t_z min), mu_c,z(t_z max)] (0 inside it).
__device__ __forceinline__ bool quick_culled_all(const QuickInv& q, const FilterConsts& c, const FilterConsts& lo,
                                                 const FilterConsts& hi, float tz_abs_max) {
    const float z0 = (q.p2 + lo.tz_hi) + lo.tz_lo, z1 = (q.p2 + hi.tz_hi) + hi.tz_lo;
    const float mz = fmaxf(fabsf(z0), fabsf(z1)) * 1.00001f;
    const float dmin = (z0 <= 0.f && z1 >= 0.f) ? 0.f : fminf(fabsf(z0), fabsf(z1)) * 0.99999f;
    const float mu2 = __fmaf_rn(q.mcx, q.mcx, __fmaf_rn(q.mcy, q.mcy, mz * mz));
    const float noise = __fmaf_rn(2e-14f * mu2, q.inv_smin2,
                                  4.8e-7f * mz * (q.ap2 + tz_abs_max) * c.inv_sz2 * 1.0002f);
    const float x = q.thr + (2e-3f + __fmaf_rn(2e-5f, fabsf(q.thr) + 0.7f, noise));
    const float x_up = __fmaf_rn(1e-3f, fabsf(x) + noise, x) + 1e-6f;
    const bool culled = 0.5f * dmin * dmin * 0.9999f > x_up * (x_up >= 0.f ? q.den_hi : c.sz2);
    return q.ok & culled;
}

// Data-parallel union over the step's poses when they share R = I, t_x,
// t_y, PSF, tau and mod (MultiPrep::shared_quick): a superset of every pose's
// candidates (the complement of certainly_culled_identity) from ONE evaluation
// per Gaussian. Only the cancellation-noise term of the margin depends on the
// pose (through mu_c,z); with |mu_c,z| bounded by its largest value over the
// poses, margin_k <= margin_max, so pose k's candidate test implies
//   mu_c,z,k^2 <= Q = 2 (sigma_z^2 + Sigma_c,zz) (thresh + margin_max)
// (relative slack 1e-4 for the fp32 roundings), and the union is "some pose's
// mu_c,z within sqrt(Q)". Identical on every rank (same parameters, same poses).
__device__ __forceinline__ bool union_candidate(const float p[11], const FilterConsts& c,
                                                const FilterConsts* fcs, int nb, float tz_abs_max) {
    float sum = p[0];
#pragma unroll
    for (int k = 1; k < 11; ++k) sum += p[k];
    if (!isfinite(sum)) return true;
    const float lmax = fmaxf(p[3], fmaxf(p[4], p[5])), lmin = fminf(p[3], fminf(p[4], p[5]));
    if (!(lmax < 40.f && lmin > -40.f && lmax - lmin < 6.2f)) return true;
    const float qn2 = p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9];
    if (!(qn2 > 1e-20f && qn2 < 1e20f)) return true;
    const float inv = rsqrtf(qn2);
    const float w = p[6] * inv, x = p[7] * inv, y = p[8] * inv, z = p[9] * inv;
    const float r0 = 2.f * (x * z - w * y), r1 = 2.f * (y * z + w * x), r2 = 1.f - 2.f * (x * x + y * y);
    const float s0 = __expf(p[3]) * c.mod, s1 = __expf(p[4]) * c.mod, s2 = __expf(p[5]) * c.mod;
    const float var = (s0 * r0) * (s0 * r0) + (s1 * r1) * (s1 * r1) + (s2 * r2) * (s2 * r2);
    const float den = c.sz2 + var;
    const float raw = p[10];
    const float log_alpha = raw >= 0.f ? -__logf(1.f + __expf(-raw)) : raw - __logf(1.f + __expf(raw));
    float mz = 0.f;
    for (int k = 0; k < nb; ++k) mz = fmaxf(mz, fabsf((p[2] + fcs[k].tz_hi) + fcs[k].tz_lo));
    const float mcx = p[0] + c.tx, mcy = p[1] + c.ty;
    const float smin = __expf(lmin) * c.mod;
    const float mu2 = mcx * mcx + mcy * mcy + mz * mz;
    const float noise = 2e-14f * mu2 / (smin * smin) + 4.f * mz * 1.2e-7f * (fabsf(p[2]) + tz_abs_max) / den;
    const float thresh = log_alpha - c.log_tau;
    const float R = thresh + (2e-3f + 2e-5f * fabsf(thresh) + noise);
    if (!(R >= 0.f)) return !(R < 0.f);  // every pose culls it (NaN: keep)
    const float Q = 2.f * den * R * 1.0001f + 1e-30f;
    for (int k = 0; k < nb; ++k) {
        const float mcz = (p[2] + fcs[k].tz_hi) + fcs[k].tz_lo;
        if (mcz * mcz <= Q) return true;
    }
    return false;
}

// ---- K_filter ------------------------------------------------------------------
// prepare_gaussians' cull (render.hpp:107) as a streaming pass with no block
// barriers. Warps walk 128-Gaussian chunks grid-stride; each lane owns four
// consecutive Gaussians and loads their 11 parameters with one 16 B vector
// load per plane straight into registers (many warps per SM keep the HBM pipe
// full). Per chunk:
//   1. division-free fp32 quick bound; lanes whose Gaussians it cannot decide
//      run the full closed-form test (q = mu_cz^2 / (sigma_z^2 + Sigma_c,zz),
//      SURVEY.md §7.3.2) — both conservative: a culled Gaussian is one the
//      reference culls too;
//   2. candidates compacted in set order (warp scan) into 48 B CandParams
//      records at chunk-major slots [b*128, b*128 + count_b), count_b stored.
// Gradient clearing (dense output contract, grad_chain.hpp:12-22): the previous
// survivors' entries (sparse), or the chunk's planes when anything else wrote
// them. No fp64 and no cross-warp waiting here.
constexpr int kFilterThreads = 256;

// Housekeeping shared by the cull kernels: clear the per-sort-tile digit
// histograms the previous radix sort used (its passes only) before this
// prepare / the radix passes refill them.
__device__ __forceinline__ void clear_prev_sort_rows(const PrepLaunch& a, unsigned gtid, unsigned gthreads) {
    const unsigned pt = a.prev_sort_words[0], pnb = a.prev_sort_words[1], pp = a.prev_sort_words[2];
    const unsigned tile_words = pt * pnb;
    const unsigned used = tile_words + (unsigned)sort_supers_cap(pt) * pnb;  // per pass
    for (unsigned ps = 0; ps < pp; ++ps) {
        unsigned* region = a.tile_hist_all + (uint64_t)ps * a.hist_region;
        unsigned* super = sort_super_row(region, a.sort_tiles_cap, pnb, 0);
        for (unsigned w = gtid; w < used; w += gthreads) (w < tile_words ? region : super - tile_words)[w] = 0u;
    }
}

__device__ __forceinline__ FilterConsts filter_consts(const SliceArgs& sl, float log_tau) {
    FilterConsts fc;
    fc.log_tau = log_tau;
    fc.mod = (float)sl.mod;
    fc.sz2 = (float)(sl.sigma_z * sl.sigma_z);
    fc.tx = (float)sl.t[0];
    fc.ty = (float)sl.t[1];
    fc.tz_hi = (float)sl.t[2];
    fc.tz_lo = (float)(sl.t[2] - (double)fc.tz_hi);
    fc.mod2 = (float)(sl.mod * sl.mod);
    fc.inv_mod2 = (float)(1.0 / (sl.mod * sl.mod));
    fc.inv_sz2 = (float)(1.0 / (sl.sigma_z * sl.sigma_z));
    return fc;
}

// Per-warp scratch of cull_chunk: the undecided Gaussians (lane*4 + item) and
// the full test's verdicts (one ballot word per 32); register-fed callers also
// copy the undecided parameters here (plane-major).
struct CullIdx {
    uint8_t idx[kFilterBlock];
    unsigned res[kFilterBlock / 32];
};
struct CullScratch {
    CullIdx x;
    float p[11][kFilterBlock];
};

// Cull one warp chunk (128 consecutive Gaussians, 4 per lane in v[]) and
// compact its candidates in set order (lanes in order, each lane's 4 in order)
// into 48 B CandParams records at slots [b*128, b*128 + count_b). Whole warp.
// The quick test runs on all 128; the Gaussians it leaves undecided (about 1
// in 10 at C2) are compacted so the full test runs in ceil(U/32) warp rounds
// instead of once per lane item. `staged` (plane-major [11][128], the chunk in
// shared memory) supplies their parameters; else they are copied to sc.p.
// qmask_given >= 0: the quick test's verdicts of the lane's items, computed by
// the caller (the multi-pose filter shares its pose-invariant part).
// Returns the lane's candidate mask; write = false: verdicts only (the union
// of a data-parallel step's other poses), nothing stored.
__device__ __forceinline__ unsigned cull_chunk(const PrepLaunch& a, const FilterConsts& fc, float log_tau,
                                               int filter_on, unsigned b, uint32_t i0, const float4 v[11],
                                               CullIdx& sx, float (*sp)[kFilterBlock], const float* staged,
                                               int qmask_given = -1, bool write = true,
                                               const LazyView* lz = nullptr) {
    const int lane = threadIdx.x & 31;
    const bool ident = a.slice.identity_rot != 0;
    // items inside the set: all candidates with the cull off, else undecided
    // unless the quick test culls them (identity poses only)
    const unsigned inset = i0 >= a.n ? 0u : (a.n - i0 >= kFilterItems ? (1u << kFilterItems) - 1 : (1u << (a.n - i0)) - 1);
    unsigned cmask = filter_on ? 0u : inset, umask = filter_on ? inset : 0u;
    if (lz) {
        // lazy step: everything the drift-widened quick test cannot cull is
        // brought up to date below and takes the exact test (staged != nullptr)
        cmask = 0u;
        umask = inset;
        if (filter_on && ident && !lz->all) {
            unsigned lmask = 0;
#pragma unroll
            for (int k = 0; k < kFilterItems; ++k) {
                float p[11];
#pragma unroll
                for (int q = 0; q < 11; ++q) p[q] = (&v[q].x)[k];
                lmask |= (quick_culled_drift(p, fc, *lz) ? 1u : 0u) << k;
            }
            umask &= ~lmask;
        }
    } else if (filter_on && ident && qmask_given >= 0) {
        umask &= ~(unsigned)qmask_given;
    } else if (filter_on && ident) {
        unsigned qmask = 0;
#pragma unroll
        for (int k = 0; k < kFilterItems; ++k) {
            float p[11];
#pragma unroll
            for (int q = 0; q < 11; ++q) p[q] = (&v[q].x)[k];
            qmask |= (quick_culled_identity(p, fc) ? 1u : 0u) << k;
        }
        umask &= ~qmask;
    }
    const unsigned nu = __popc(umask);
    unsigned uincl = nu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, uincl, o);
        if (lane >= o) uincl += u;
    }
    const unsigned U = __shfl_sync(0xffffffffu, uincl, 31);
    if (U) {
        unsigned pos = uincl - nu;
#pragma unroll
        for (int k = 0; k < kFilterItems; ++k)
            if (umask & (1u << k)) {
                if (staged) {
                    sx.idx[pos] = (uint8_t)(lane * kFilterItems + k);
                } else {
#pragma unroll
                    for (int q = 0; q < 11; ++q) sp[q][pos] = (&v[q].x)[k];
                }
                ++pos;
            }
        __syncwarp();
        for (unsigned r = 0; r * 32 < U; ++r) {
            const unsigned e = r * 32 + lane;
            bool cand = false;
            if (e < U) {
                float p[11];
                if (staged) {
                    const unsigned j = sx.idx[e];
#pragma unroll
                    for (int q = 0; q < 11; ++q) p[q] = staged[q * kFilterBlock + j];
                    if (lz) {  // the true parameters, back into the stage for the emission
                        lazy_materialize(*lz, b * kFilterBlock + j, p);
                        float* stw = const_cast<float*>(staged);
#pragma unroll
                        for (int q = 0; q < 11; ++q) stw[q * kFilterBlock + j] = p[q];
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 11; ++q) p[q] = sp[q][e];
                }
                cand = !filter_on || (ident ? !certainly_culled_identity(p, fc)
                                            : !certainly_culled(p, a.slice, log_tau, fc.mod, fc.sz2));
            }
            const unsigned bal = __ballot_sync(0xffffffffu, cand);
            if (lane == 0) sx.res[r] = bal;
        }
        __syncwarp();
        pos = uincl - nu;
#pragma unroll
        for (int k = 0; k < kFilterItems; ++k)
            if (umask & (1u << k)) {
                if ((sx.res[pos >> 5] >> (pos & 31)) & 1u) cmask |= 1u << k;
                ++pos;
            }
        __syncwarp();  // the scratch is reused by the warp's next chunk
    }
    if (!write) return cmask;
    const unsigned nc = __popc(cmask);
    unsigned incl = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) a.cand_count[b] = incl;
    if (cmask) {
        CandParams* out = a.cand + (uint64_t)b * kFilterBlock + (incl - nc);
#pragma unroll
        for (int k = 0; k < kFilterItems; ++k)
            if (cmask & (1u << k)) {
                float p[11];
#pragma unroll
                for (int q = 0; q < 11; ++q)
                    p[q] = lz ? staged[q * kFilterBlock + (threadIdx.x & 31) * kFilterItems + k] : (&v[q].x)[k];
                store_cand(out++, p, i0 + k);
            }
    }
    return cmask;
}

// cp.async (16 B, L1 bypass) staging of K_filter chunks: each lane copies its
// own 4 Gaussians' 11 plane slices; one commit group per chunk. With an L2
// eviction-priority hint (the parameter planes are read again by the same
// training step's Adam: keep them in L2 until then)
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, unsigned long long policy) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

constexpr int kFilterStages = 2;
constexpr size_t kFilterStageFloats = 11 * kFilterBlock;  // one warp chunk, plane-major
constexpr size_t kFilterSmem =
    (size_t)(kFilterThreads / 32) * (kFilterStages * kFilterStageFloats * 4 + sizeof(CullIdx));

// Each warp streams its chunks (grid-stride) through a 2-stage cp.async ring:
// chunk b+1's 5.6 KB is in flight while chunk b is culled, so HBM never waits
// for the cull arithmetic (a register-fed loop leaves the memory idle between
// its load bursts: ~2 chunks per warp at C2).
template <bool kZeroGrads, bool kLazy>
__global__ void __launch_bounds__(kFilterThreads, 2) k_filter(const PrepLaunch a, float log_tau, int filter_on) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    extern __shared__ __align__(16) float s_filter[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* ring = s_filter + (size_t)warp * kFilterStages * kFilterStageFloats;
    CullIdx& sx = reinterpret_cast<CullIdx*>(s_filter + (size_t)(kFilterThreads / 32) * kFilterStages *
                                                             kFilterStageFloats)[warp];
    const unsigned nchunks = a.nfilter;
    const unsigned gthreads = gridDim.x * kFilterThreads;
    const unsigned gtid = blockIdx.x * kFilterThreads + tid;
    const unsigned gwarps = gthreads / 32;
    const unsigned long long keep = l2_evict_last_policy();
    auto prefetch = [&](unsigned b, int stage) {
        // cap is a multiple of kParamAlign: the chunk never leaves the plane
        const float* src = a.params + (uint64_t)b * kFilterBlock + lane * kFilterItems;
        float* dst = ring + stage * kFilterStageFloats + lane * kFilterItems;
#pragma unroll
        for (int q = 0; q < 11; ++q) cp_async16_hint(dst + q * kFilterBlock, src + (uint64_t)q * a.cap, keep);
    };
    unsigned b = gtid / 32;
    if (b < nchunks) prefetch(b, 0);
    cp_async_commit();

    const unsigned dirty = kZeroGrads ? *a.grads_dirty : 0u;
    const bool dense_zero = kZeroGrads && dirty == kGradsDense;
    if (a.head)  // the prepare's control head (no separate memset)
        for (unsigned w = gtid; w < a.head_words; w += gthreads) a.head[w] = 0u;
    clear_prev_sort_rows(a, gtid, gthreads);
    if constexpr (kZeroGrads) {
        if (!dense_zero)  // the previous survivors' gradients (sparse mode)
            for (unsigned e = gtid; e < dirty; e += gthreads) {
                const uint32_t i = a.dirty_idx[e];
#pragma unroll
                for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = 0.f;
            }
    }
    const FilterConsts fc = filter_consts(a.slice, log_tau);
    __shared__ LazyView s_lz;
    if (kLazy) {
        if (tid == 0) s_lz = lazy_view(a);
        __syncthreads();
    }
    const LazyView lz = kLazy ? s_lz : LazyView{};

    for (int it = 0; b < nchunks; ++it, b += gwarps) {
        if (b + gwarps < nchunks) prefetch(b + gwarps, (it + 1) & 1);
        cp_async_commit();
        cp_async_wait1();  // this lane's copies of chunk b landed
        __syncwarp();      // ... and every lane's (the full test reads other lanes' Gaussians)
        const float* st = ring + (it & 1) * kFilterStageFloats;
        const uint32_t i0 = b * kFilterBlock + lane * kFilterItems;  // this lane's first Gaussian
        float4 v[11];
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = *reinterpret_cast<const float4*>(st + q * kFilterBlock + lane * kFilterItems);
        if (dense_zero)
#pragma unroll
            for (int q = 0; q < 11; ++q)
                *reinterpret_cast<float4*>(a.grads + (uint64_t)q * a.cap + i0) = make_float4(0.f, 0.f, 0.f, 0.f);
        cull_chunk(a, fc, log_tau, filter_on, b, i0, v, sx, nullptr, st, -1, true, kLazy ? &lz : nullptr);
        __syncwarp();  // stage (it & 1) is refilled by the next iteration's prefetch
    }
}

// ---- K_filter over several slice poses (batched steps) ---------------------------
// The parameters are streamed ONCE for the B slices of a batched step: each
// warp chunk is culled against every slice's pose in turn (cull_chunk with that
// slice's PrepLaunch), each slice's candidates compacted into its own context's
// buffers. Per-slice housekeeping (control head, previous sort rows) as
// K_filter's. Gradients are not touched (batched steps keep slot gradients).
struct MultiPrep {
    PrepLaunch p[kMaxBatch];
    float log_tau[kMaxBatch];
    int filter_on[kMaxBatch];
    int nb;
    int shared_quick;  // every pose R = I with the same t_x, t_y, PSF, tau, mod: split quick test
    // data-parallel step: only pose `own` stores candidates (the others give
    // verdicts); union_words[4 b + k] bit l = item 4 l + k of chunk b is a
    // candidate of some pose (nullptr: batched step, every pose stores)
    int own;
    unsigned* union_words;
};

__global__ void __launch_bounds__(kFilterThreads, 2) k_filter_multi(const __grid_constant__ MultiPrep m) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    extern __shared__ __align__(16) float s_filter[];
    const PrepLaunch& a0 = m.p[0];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* ring = s_filter + (size_t)warp * kFilterStages * kFilterStageFloats;
    CullIdx& sx = reinterpret_cast<CullIdx*>(s_filter + (size_t)(kFilterThreads / 32) * kFilterStages *
                                                             kFilterStageFloats)[warp];
    const unsigned nchunks = a0.nfilter;
    const unsigned gthreads = gridDim.x * kFilterThreads;
    const unsigned gtid = blockIdx.x * kFilterThreads + tid;
    const unsigned gwarps = gthreads / 32;
    const unsigned long long keep = l2_evict_last_policy();
    auto prefetch = [&](unsigned b, int stage) {
        const float* src = a0.params + (uint64_t)b * kFilterBlock + lane * kFilterItems;
        float* dst = ring + stage * kFilterStageFloats + lane * kFilterItems;
#pragma unroll
        for (int q = 0; q < 11; ++q) cp_async16_hint(dst + q * kFilterBlock, src + (uint64_t)q * a0.cap, keep);
    };
    __shared__ FilterConsts s_fc[kMaxBatch];
    unsigned b = gtid / 32;
    if (b < nchunks) prefetch(b, 0);
    cp_async_commit();
    __shared__ float s_tzmax;
    __shared__ int s_kmin, s_kmax;  // the poses with the smallest / largest t_z (the hull of mu_c,z)
    if (tid < m.nb) s_fc[tid] = filter_consts(m.p[tid].slice, m.log_tau[tid]);
    if (tid == 0) {
        float t = 0.f;
        int kmin = 0, kmax = 0;
        for (int k = 0; k < m.nb; ++k) {
            t = fmaxf(t, fabsf((float)m.p[k].slice.t[2]));
            if (m.p[k].slice.t[2] < m.p[kmin].slice.t[2]) kmin = k;
            if (m.p[k].slice.t[2] > m.p[kmax].slice.t[2]) kmax = k;
        }
        s_tzmax = t;
        s_kmin = kmin;
        s_kmax = kmax;
    }
    for (int k = 0; k < m.nb; ++k) {
        if (m.union_words && k != m.own) continue;  // verdict-only poses own no buffers
        const PrepLaunch& a = m.p[k];
        for (unsigned w = gtid; w < a.head_words; w += gthreads) a.head[w] = 0u;
        clear_prev_sort_rows(a, gtid, gthreads);
    }
    __syncthreads();  // s_fc
    for (int it = 0; b < nchunks; ++it, b += gwarps) {
        if (b + gwarps < nchunks) prefetch(b + gwarps, (it + 1) & 1);
        cp_async_commit();
        cp_async_wait1();
        __syncwarp();
        const float* st = ring + (it & 1) * kFilterStageFloats;
        const uint32_t i0 = b * kFilterBlock + lane * kFilterItems;
        float4 v[11];
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = *reinterpret_cast<const float4*>(st + q * kFilterBlock + lane * kFilterItems);
        unsigned umask = 0;
        if (m.union_words && m.shared_quick) {
            // the union in one evaluation per Gaussian; only the rank's own
            // pose runs the cull with its candidate emission
            // (one pose: the union is the pose's own candidates)
            const FilterConsts& fo = s_fc[m.own];
            unsigned qmask = 0, need = 0;
#pragma unroll
            for (int it2 = 0; it2 < kFilterItems; ++it2) {
                float p[11];
#pragma unroll
                for (int q = 0; q < 11; ++q) p[q] = (&v[q].x)[it2];
                const QuickInv qi = quick_invariant(p, fo);
                qmask |= (quick_culled_pose(qi, fo) ? 1u : 0u) << it2;
                if (m.nb > 1 && i0 + it2 < a0.n && !quick_culled_all(qi, fo, s_fc[s_kmin], s_fc[s_kmax], s_tzmax))
                    need |= 1u << it2;
            }
            if (m.nb > 1) {
                // the items the all-pose quick bound cannot cull take the union
                // test compacted across the warp (a few per chunk: one round of
                // 32 instead of every item slot of every lane)
                const unsigned nn = __popc(need);
                unsigned incl = nn;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                const unsigned U = __shfl_sync(0xffffffffu, incl, 31);
                if (U) {
                    unsigned pos = incl - nn;
#pragma unroll
                    for (int it2 = 0; it2 < kFilterItems; ++it2)
                        if (need & (1u << it2)) sx.idx[pos++] = (uint8_t)(lane * kFilterItems + it2);
                    __syncwarp();
                    for (unsigned r = 0; r * 32 < U; ++r) {
                        const unsigned e = r * 32 + lane;
                        bool in = false;
                        if (e < U) {
                            const unsigned j = sx.idx[e];
                            float p[11];
#pragma unroll
                            for (int q = 0; q < 11; ++q) p[q] = st[q * kFilterBlock + j];
                            in = union_candidate(p, fo, s_fc, m.nb, s_tzmax);
                        }
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        if (lane == 0) sx.res[r] = bal;
                    }
                    __syncwarp();
                    pos = incl - nn;
#pragma unroll
                    for (int it2 = 0; it2 < kFilterItems; ++it2)
                        if (need & (1u << it2)) {
                            if ((sx.res[pos >> 5] >> (pos & 31)) & 1u) umask |= 1u << it2;
                            ++pos;
                        }
                    __syncwarp();  // the scratch is reused by the cull below
                }
            }
            const unsigned own = cull_chunk(m.p[m.own], fo, m.log_tau[m.own], m.filter_on[m.own], b, i0, v, sx,
                                            nullptr, st, (int)qmask, true);
            if (m.nb == 1) umask = own;
        } else if (m.shared_quick) {
            QuickInv qi[kFilterItems];
#pragma unroll
            for (int it2 = 0; it2 < kFilterItems; ++it2) {
                float p[11];
#pragma unroll
                for (int q = 0; q < 11; ++q) p[q] = (&v[q].x)[it2];
                qi[it2] = quick_invariant(p, s_fc[0]);
            }
#pragma unroll 1
            for (int k = 0; k < m.nb; ++k) {
                unsigned qmask = 0;
#pragma unroll
                for (int it2 = 0; it2 < kFilterItems; ++it2) qmask |= (quick_culled_pose(qi[it2], s_fc[k]) ? 1u : 0u) << it2;
                umask |= cull_chunk(m.p[k], s_fc[k], m.log_tau[k], m.filter_on[k], b, i0, v, sx, nullptr, st, (int)qmask,
                                    !m.union_words || k == m.own);
            }
        } else {
#pragma unroll 1
            for (int k = 0; k < m.nb; ++k)
                umask |= cull_chunk(m.p[k], s_fc[k], m.log_tau[k], m.filter_on[k], b, i0, v, sx, nullptr, st, -1,
                                    !m.union_words || k == m.own);
        }
        if (m.union_words) {
#pragma unroll
            for (int it2 = 0; it2 < kFilterItems; ++it2) {
                const unsigned w = __ballot_sync(0xffffffffu, (umask >> it2) & 1u);
                if (lane == 0) m.union_words[(uint64_t)b * kFilterItems + it2] = w;
            }
        }
        __syncwarp();
    }
}

// ---- K_adam_cull -----------------------------------------------------------------
// Training step: adam_step (optimize.hpp:195-221) fused with the NEXT slice's
// K_filter. Both stream every parameter once; fused, the next step starts at
// K_decide and the parameters cross HBM once per step instead of twice. Each
// thread updates 4 consecutive primitives (adam.cuh: the same bits as the
// stand-alone Adam kernel; dense or slot gradients), leaves the dense gradient
// planes zero, then its warp culls the 128 updated primitives against the next
// pose (cull_chunk).
template <int kMinB>
__global__ void __launch_bounds__(256, kMinB) k_adam_cull(const AdamLaunch a, const PrepLaunch f, float log_tau,
                                                      int filter_on) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ CullScratch s_cull[8];
    const bool adam_on = !(a.ctrl && a.ctrl->pair_overflow);  // the slice overflowed: no update
    const bool slots = a.slot_grads != nullptr;
    const AdamConsts c = *a.consts;  // k_adam_consts ran before
    if (adam_on) adam_advance_step(a, c);
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
    clear_prev_sort_rows(f, gtid, gthreads);
    // K_filter's gradient duty. Dense gradients: the Adam below zeroes every
    // non-zero entry it consumes. Slot gradients: the dense planes are not
    // consumed, so the pending clear of the last dense backward happens here
    // (the next K_decide resets the state word).
    unsigned dirty = 0;
    if (!slots) {
        if (gtid == 0) *f.grads_dirty = 0u;
    } else {
        dirty = *f.grads_dirty;
        if (dirty != kGradsDense)
            for (unsigned e = gtid; e < dirty; e += gthreads) {
                const uint32_t i = f.dirty_idx[e];
#pragma unroll
                for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = 0.f;
            }
    }
    const uint32_t i0 = gtid * kFilterItems;
    float4 p[11];
    if (i0 < a.n) {
        unsigned nz = 0;
        if (adam_on) {
            Pack<kFilterItems> q[11];
            uint32_t gslot[kFilterItems];
            const bool any = slots && adam_slots<kFilterItems>(a, i0, gslot);
            // (software-pipelined planes, as k_adam: the same bits)
            adam_update_pipe<kFilterItems>(
                a, c, i0, [&](int k) { return adam_grad<kFilterItems>(a, k, i0, slots ? gslot : nullptr); }, q, nz);
            adam_store<kFilterItems>(a, i0, q);
            if (any) adam_slots_clear<kFilterItems>(a, i0);
#pragma unroll
            for (int d = 0; d < 11; ++d) p[d] = make_float4(q[d].v[0], q[d].v[1], q[d].v[2], q[d].v[3]);
        } else {
            if (slots) adam_slots_clear<kFilterItems>(a, i0);
#pragma unroll
            for (int d = 0; d < 11; ++d) p[d] = *reinterpret_cast<const float4*>(a.params + (uint64_t)d * a.cap + i0);
        }
        if (slots ? dirty == kGradsDense : nz != 0)
#pragma unroll
            for (int d = 0; d < 11; ++d)
                *reinterpret_cast<float4*>(a.grads + (uint64_t)d * a.cap + i0) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
#pragma unroll
        for (int d = 0; d < 11; ++d) p[d] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const unsigned b = i0 / kFilterBlock;  // the warp's chunk
    if (b < f.nfilter) {
        CullScratch& sc = s_cull[threadIdx.x >> 5];
        cull_chunk(f, filter_consts(f.slice, log_tau), log_tau, filter_on, b, i0, p, sc.x, sc.p, nullptr);
    }
}

}  // namespace

void launch_prep(const PrepLaunch& a, int num_sms, cudaStream_t st) {
    if (a.n == 0) return;
    const bool filter_on = a.slice.tau > 0.0 && a.slice.mod > 1e-10 && a.slice.mod < 1e10 &&
                           a.slice.sigma_z > 1e-10 && a.slice.sigma_z < 1e10;
    const float log_tau = filter_on ? (float)log(a.slice.tau) : 0.f;
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(k_filter<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaFuncSetAttribute(k_filter<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaFuncSetAttribute(k_filter<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaFuncSetAttribute(k_filter<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_filter<true, false>, kFilterThreads, kFilterSmem);
        if (per_sm < 1) per_sm = 1;
    }
    const uint64_t need = ((uint64_t)a.nfilter * 32 + kFilterThreads - 1) / kFilterThreads;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms * per_sm));
    const int fo = filter_on ? 1 : 0;
    if (a.lazy_on) {
        if (a.grads) launch_pdl(k_filter<true, true>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, fo);
        else launch_pdl(k_filter<false, true>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, fo);
    } else {
        if (a.grads) launch_pdl(k_filter<true, false>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, fo);
        else launch_pdl(k_filter<false, false>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, fo);
    }
}

void launch_prep_multi(const PrepLaunch* pl, int nb, int num_sms, cudaStream_t st, int own, unsigned* union_words) {
    if (nb < 1 || pl[0].n == 0) return;
    MultiPrep m;
    m.nb = nb;
    m.own = own;
    m.union_words = union_words;
    m.shared_quick = 1;
    for (int k = 0; k < nb; ++k) {
        m.p[k] = pl[k];
        const SliceArgs& sl = pl[k].slice;
        const bool on = sl.tau > 0.0 && sl.mod > 1e-10 && sl.mod < 1e10 && sl.sigma_z > 1e-10 && sl.sigma_z < 1e10;
        m.filter_on[k] = on ? 1 : 0;
        m.log_tau[k] = on ? (float)log(sl.tau) : 0.f;
        const SliceArgs& s0 = pl[0].slice;
        if (!on || !sl.identity_rot || sl.t[0] != s0.t[0] || sl.t[1] != s0.t[1] || sl.sigma_z != s0.sigma_z ||
            sl.tau != s0.tau || sl.mod != s0.mod)
            m.shared_quick = 0;
    }
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(k_filter_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_filter_multi, kFilterThreads, kFilterSmem);
        if (per_sm < 1) per_sm = 1;
    }
    const uint64_t need = ((uint64_t)pl[0].nfilter * 32 + kFilterThreads - 1) / kFilterThreads;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms * per_sm));
    launch_pdl(k_filter_multi, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, m);
}

void launch_adam_cull(const AdamLaunch& a, const PrepLaunch& f, cudaStream_t st) {
    const bool filter_on = f.slice.tau > 0.0 && f.slice.mod > 1e-10 && f.slice.mod < 1e10 &&
                           f.slice.sigma_z > 1e-10 && f.slice.sigma_z < 1e10;
    const float log_tau = filter_on ? (float)log(f.slice.tau) : 0.f;
    const unsigned threads = (unsigned)std::max<uint64_t>((uint64_t)f.nfilter * 32, (a.n + kFilterItems - 1) / kFilterItems);
    const unsigned grid = (threads + 255) / 256;
    if (!grid) return;
    // (2 CTAs/SM without spills measured the same as 3 with a 48 B spill)
    launch_pdl(k_adam_cull<3>, dim3(grid), dim3(256), 0, st, a, f, log_tau, filter_on ? 1 : 0);
}

}  // namespace gpk
