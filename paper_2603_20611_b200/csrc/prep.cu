// prep.cu — per-slice preprocessing (prepare_gaussians, render.hpp:83-138, and
// the TileGrid build, render.hpp:142-160) and the backward chain
// (backward.hpp:148-185). Built with --fmad=false so the fp64 focus algebra
// rounds like the reference (see focus.cuh).
//
// Two kernels replace prepare_gaussians + TileGrid:
//   K_filter  one thread per Gaussian (8 per thread), coalesced SoA loads, an
//             fp32 CERTAIN-CULL test in closed form (q = mu_cz^2 /
//             (sigma_z^2 + Sigma_c,zz)) with a margin
//             covering fp32 error and the reference's own cancellation noise.
//             Certainly-culled primitives get their dense gradient zero-filled
//             here (the gradient plane is written exactly once per slice); the
//             rest become candidates, compacted in set order inside the block
//             and published with a plain per-block count — no cross-block
//             waiting. This is the HBM-bound kernel (44 B read + 44 B written
//             per Gaussian) and runs at full occupancy.
//   K_exact   persistent CTAs take 256-candidate chunks in order (each CTA
//             locates its candidates from the per-block counts), run the
//             reference's fp64 computation (focus_prepare) densely, decide the
//             exact cull, write 48 B survivor records and — through a wait-free
//             ordered prefix over chunk aggregates — survivor slots and (tile,
//             candidate) pairs in (candidate, tile) order: the order a stable
//             sort on the tile key needs to reproduce the reference lists.
//             Global and per-sort-tile digit histograms for the first radix
//             pass are accumulated on the way.
#include "adam.cuh"
#include "common.cuh"
#include "focus.cuh"

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

__device__ __forceinline__ void load_params(const float* __restrict__ params, uint64_t cap,
                                            uint32_t i, float p[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) p[k] = __ldg(params + (uint64_t)k * cap + i);
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
    const unsigned used = tile_words + ((pt + kSuperTiles - 1) / kSuperTiles) * pnb;  // per pass
    for (unsigned ps = 0; ps < pp; ++ps) {
        unsigned* region = a.tile_hist_all + (uint64_t)ps * a.hist_region;
        unsigned* super = region + a.sort_tiles_cap * pnb - tile_words;
        for (unsigned w = gtid; w < used; w += gthreads) (w < tile_words ? region : super)[w] = 0u;
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
__device__ __forceinline__ void cull_chunk(const PrepLaunch& a, const FilterConsts& fc, float log_tau, int filter_on,
                                           unsigned b, uint32_t i0, const float4 v[11], CullIdx& sx,
                                           float (*sp)[kFilterBlock], const float* staged) {
    const int lane = threadIdx.x & 31;
    const bool ident = a.slice.identity_rot != 0;
    // items inside the set: all candidates with the cull off, else undecided
    // unless the quick test culls them (identity poses only)
    const unsigned inset = i0 >= a.n ? 0u : (a.n - i0 >= kFilterItems ? (1u << kFilterItems) - 1 : (1u << (a.n - i0)) - 1);
    unsigned cmask = filter_on ? 0u : inset, umask = filter_on ? inset : 0u;
    if (filter_on && ident) {
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
                } else {
#pragma unroll
                    for (int q = 0; q < 11; ++q) p[q] = sp[q][e];
                }
                cand = ident ? !certainly_culled_identity(p, fc)
                             : !certainly_culled(p, a.slice, log_tau, fc.mod, fc.sz2);
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
                for (int q = 0; q < 11; ++q) p[q] = (&v[q].x)[k];
                store_cand(out++, p, i0 + k);
            }
    }
}

// cp.async (16 B, L1 bypass) staging of K_filter chunks: each lane copies its
// own 4 Gaussians' 11 plane slices; one commit group per chunk.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// ... with an L2 eviction-priority hint (the parameter planes are read again
// by the same training step's Adam: keep them in L2 until then)
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
template <bool kZeroGrads>
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
    if (kZeroGrads && !dense_zero)  // the previous survivors' gradients (sparse mode)
        for (unsigned e = gtid; e < dirty; e += gthreads) {
            const uint32_t i = a.dirty_idx[e];
#pragma unroll
            for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = 0.f;
        }
    const FilterConsts fc = filter_consts(a.slice, log_tau);

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
        cull_chunk(a, fc, log_tau, filter_on, b, i0, v, sx, nullptr, st);
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
    unsigned b = gtid / 32;
    if (b < nchunks) prefetch(b, 0);
    cp_async_commit();
    for (int k = 0; k < m.nb; ++k) {
        const PrepLaunch& a = m.p[k];
        for (unsigned w = gtid; w < a.head_words; w += gthreads) a.head[w] = 0u;
        clear_prev_sort_rows(a, gtid, gthreads);
    }
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
#pragma unroll 1
        for (int k = 0; k < m.nb; ++k) {
            const PrepLaunch& a = m.p[k];
            cull_chunk(a, filter_consts(a.slice, m.log_tau[k]), m.log_tau[k], m.filter_on[k], b, i0, v, sx, nullptr,
                       st);
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
__global__ void __launch_bounds__(256, 3) k_adam_cull(const AdamLaunch a, const PrepLaunch f, float log_tau,
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
            adam_update<kFilterItems>(a, c, i0, slots ? gslot : nullptr, q, nz);
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

// ---- K_decide ------------------------------------------------------------------
// The rest of prepare_gaussians + the TileGrid pair list (render.hpp:91-160),
// one CTA per kDecideChunks consecutive K_filter chunks (a "group"; few enough
// groups that all CTAs are resident together), groups taken in ticket order:
//   1. each candidate gets the decision-grade fp64 closed form (fast_decide)
//      and, within ~1e-9 of a decision boundary, the reference's own fp64
//      evaluation (focus_prepare): survivors and pixel bounds — therefore tile
//      pairs — are the reference's bit for bit. Survivors are compacted in set
//      order: 48 B record + 48 B params at group-major survivor slots.
//   2. group aggregate (survivors, pairs) through a wait-free ordered prefix
//      over group words (predecessors hold earlier tickets: they are running
//      or done and publish before they wait).
//   3. survivor slots, and (tile, survivor slot) pairs in (survivor, tile)
//      order — the order a stable sort on the tile key needs to reproduce the
//      reference's ascending per-tile lists — with the first radix pass's
//      digit histograms (global, per sort tile, per super-tile).
constexpr int kDecideThreads = 256;
constexpr int kDecideGroup = kDecideGroupSize;

__global__ void __launch_bounds__(kDecideThreads) k_decide(const PrepLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    extern __shared__ unsigned s_dyn_u[];
    unsigned* s_incl = s_dyn_u;                                              // kDecideGroup
    uint16_t(*s_rect)[3] = reinterpret_cast<uint16_t(*)[3]>(s_dyn_u + kDecideGroup);  // kDecideGroup x 3
    __shared__ unsigned s_hist[kMaxSortPasses][kMaxBuckets];
    __shared__ unsigned s_cnt[2][kDecideThreads / 32];
    __shared__ unsigned s_cpre[kDecideChunks + 1];
    __shared__ unsigned s_grp, s_nsurv, s_nexact;
    __shared__ unsigned long long s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned dmask = (1u << a.digit_bits) - 1;
    const unsigned nb = dmask + 1;
    const int tiles_x = a.slice.tiles_x;
    const unsigned ngroups = gridDim.x;
    for (int k = tid; k < a.passes * kMaxBuckets; k += kDecideThreads) (&s_hist[0][0])[k] = 0;
    if (tid == 0) {
        s_grp = blockIdx.x;
        s_nsurv = 0;
        s_nexact = 0;
    }
    __syncthreads();
    if (warp < kDecideChunks / 32) {  // exclusive prefix of the group's chunk counts
        const unsigned c = s_grp * kDecideChunks + tid;
        const unsigned v = c < a.nfilter ? __ldcg(&a.cand_count[c]) : 0u;
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        s_cpre[tid] = incl - v;
        if (lane == 31) s_cnt[0][warp] = incl;
    }
    __syncthreads();
    if (tid < kDecideChunks && warp > 0)
        for (int w = 0; w < warp; ++w) s_cpre[tid] += s_cnt[0][w];
    if (tid == 0) {
        unsigned tot = 0;
        for (int w = 0; w < kDecideChunks / 32; ++w) tot += s_cnt[0][w];
        s_cpre[kDecideChunks] = tot;
    }
    __syncthreads();
    const unsigned g = s_grp;
    // the preceding K_filter / fused Adam + cull cleared the dense gradient
    // planes as the state word said (the dense chain sets it again)
    if (a.grads && blockIdx.x == 0 && tid == 0) *a.grads_dirty = 0u;
    const uint32_t base = g * kDecideGroup;
    const unsigned nc = s_cpre[kDecideChunks];

    // ---- 1. exact decision, survivors compacted in order -------------------------
    for (unsigned j0 = 0, r = 0; j0 < nc; j0 += kDecideThreads, r ^= 1) {
        const unsigned j = j0 + tid;
        SurvivorRecord rec;
        float pf[11];
        uint32_t i = 0;
        bool survive = false;
        if (j < nc) {
            int q = 0;  // chunk of candidate j: last q with s_cpre[q] <= j
#pragma unroll
            for (int step = kDecideChunks / 2; step > 0; step >>= 1)
                if (s_cpre[q + step] <= j) q += step;
            load_cand(a.cand + (uint64_t)base + q * kFilterBlock + (j - s_cpre[q]), pf, i);
            uint32_t flag = 0;
            const int fr = fast_decide(pf, a.slice, rec);
            if (fr == kFastSurvive) {
                survive = true;
            } else if (fr == kAmbiguous) {
                flag = kExactFlag;
                // near a decision boundary: the reference's own fp64 evaluation
                double pd[11];
#pragma unroll
                for (int t = 0; t < 11; ++t) pd[t] = (double)pf[t];
                Focus f;
                const int res = focus_prepare(pd, a.slice, f);
                if (res == kSurvive) {
                    survive = true;
                    rec.mu2d_x = f.mu_e.x;
                    rec.mu2d_y = f.mu_e.y;
                    rec.conic_a = (float)f.con_a;
                    rec.conic_b = (float)f.con_b;
                    rec.conic_d = (float)f.con_d;
                    rec.alpha_tilde = (float)f.alpha_tilde;
                    rec.lo_x = (uint16_t)f.lo_x;
                    rec.hi_x = (uint16_t)f.hi_x;
                    rec.lo_y = (uint16_t)f.lo_y;
                    rec.hi_y = (uint16_t)f.hi_y;
                } else if (res > 0) {
                    record_error(a.err, res, i);
                }
            }
            rec.gidx = i | flag;
            rec.pair_base = 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, survive);
        const unsigned mx = __ballot_sync(0xffffffffu, survive && (rec.gidx & kExactFlag));
        if (lane == 0) {
            s_cnt[r][warp] = __popc(m);
            if (mx) atomicAdd(&s_nexact, (unsigned)__popc(mx));
        }
        __syncthreads();
        unsigned rank = s_nsurv + __popc(m & lanemask_lt());
        for (int w = 0; w < warp; ++w) rank += s_cnt[r][w];
        if (survive) {
            a.records[base + rank] = rec;
            store_cand(a.surv_params + base + rank, pf, i);
            a.survivor_list[base + rank] = i;
            // fp64-decided survivors take the fp64 chain (K_chain_exact, which
            // runs beside K_chain once the backward is done)
            if (rec.gidx & kExactFlag) a.exact_list[atomicAdd(&a.ctrl->chain_exact, 1u)] = base + rank;
            const unsigned tx0 = rec.lo_x / kTile, ty0 = rec.lo_y / kTile;
            const unsigned ntx = rec.hi_x / kTile - tx0 + 1, nty = rec.hi_y / kTile - ty0 + 1;
            s_rect[rank][0] = (uint16_t)tx0;
            s_rect[rank][1] = (uint16_t)ty0;
            s_rect[rank][2] = (uint16_t)ntx;
            s_incl[rank] = ntx * nty;
        }
        __syncthreads();
        if (tid == 0) {
            unsigned t = 0;
            for (int w = 0; w < kDecideThreads / 32; ++w) t += s_cnt[r][w];
            s_nsurv += t;
        }
    }
    __syncthreads();
    const unsigned S = s_nsurv;
    if (tid == 0) {  // statistics (gpk_prepare_stats)
        if (nc) atomicAdd(&a.ctrl->candidates, nc);
        if (s_nexact) atomicAdd(&a.ctrl->exact_decided, s_nexact);
    }

    // ---- 2. inclusive scan of the pair counts, ordered group prefix -------------
    {
        constexpr int kPer = kDecideGroup / kDecideThreads;  // consecutive survivors per thread
        const unsigned j0 = tid * kPer;
        unsigned run = 0;
        for (int q = 0; q < kPer; ++q) run += (j0 + q < S) ? s_incl[j0 + q] : 0u;
        unsigned incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_cnt[0][warp] = incl;
        __syncthreads();
        unsigned ex = incl - run;
        for (int w = 0; w < warp; ++w) ex += s_cnt[0][w];
        for (int q = 0; q < kPer && j0 + q < S; ++q) {
            ex += s_incl[j0 + q];
            s_incl[j0 + q] = ex;
        }
    }
    __syncthreads();
    const unsigned Pb = S ? s_incl[S - 1] : 0u;
    // ---- 2. reserve the group's pair range (no ordering between groups here:
    // the radix pass orders pairs of equal tile by group index, i.e. by slot)
    if (tid == 0) {
        const unsigned P0 = atomicAdd(&a.ctrl->pairs, Pb);
        if (S) atomicAdd(&a.ctrl->survivors, S);
        if ((unsigned long long)P0 + Pb > a.pair_cap) a.ctrl->pair_overflow = 1u;
        a.grp_pairs[g] = make_uint2(P0, Pb);
        a.grp_surv[g] = S;
        s_excl = P0;
    }
    __syncthreads();

    // ---- 3. pair bases and pair emission ------------------------------------------
    const unsigned P0 = (unsigned)s_excl;
    for (unsigned j = tid; j < S; j += kDecideThreads) a.records[base + j].pair_base = P0 + (j ? s_incl[j - 1] : 0u);
    // tile of the group's k-th pair (pairs in (survivor, tile-in-rect) order)
    auto pair_tile = [&](unsigned k, unsigned& surv) {
        unsigned lo = 0, hi = S - 1;
        while (lo < hi) {
            const unsigned mid = (lo + hi) >> 1;
            if (s_incl[mid] > k) hi = mid; else lo = mid + 1;
        }
        surv = lo;
        const unsigned local = k - (lo ? s_incl[lo - 1] : 0u);
        const unsigned ntx = s_rect[lo][2];
        return (s_rect[lo][1] + local / ntx) * (unsigned)tiles_x + s_rect[lo][0] + local % ntx;
    };
    if (a.bucket_tab) {
        // single-pass slice (every tile is one digit): bucket the group's pairs
        // by tile — counts, bucket starts (published for k_gather), then slots
        // into their buckets. Order inside a bucket is restored by k_gather.
        for (unsigned k = tid; k < Pb; k += kDecideThreads) {
            unsigned j;
            atomicAdd(&s_hist[0][pair_tile(k, j)], 1u);
        }
        __syncthreads();
        unsigned* s_start = &s_hist[1][0];
        {
            constexpr int kPer = kMaxBuckets / kDecideThreads;
            const unsigned d0 = tid * kPer;
            unsigned v[kPer], run = 0;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                v[q] = s_hist[0][d0 + q];
                run += v[q];
                if (v[q]) atomicAdd(&a.hist[d0 + q], v[q]);
            }
            unsigned incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) s_cnt[0][warp] = incl;
            __syncthreads();
            unsigned ex = incl - run;
            for (int w = 0; w < warp; ++w) ex += s_cnt[0][w];
            // the group's row of bucket starts (+ end), coalesced
            unsigned* trow = a.bucket_tab + (uint64_t)g * (nb + 1);
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                s_start[d0 + q] = ex;
                if (d0 + q < nb) trow[d0 + q] = P0 + ex;
                s_hist[0][d0 + q] = 0;  // becomes the fill counter
                ex += v[q];
            }
            if (tid == 0) trow[nb] = P0 + Pb;
        }
        __syncthreads();
        // stable fill: each bucket receives its pairs in pair order (= ascending
        // slot, one pair per survivor and tile), so the gather is a plain
        // concatenation. Rounds of 1024 pairs; warp w ranks its 128 with
        // __match_any_sync against its own per-tile counters, then a per-tile
        // prefix over the warps (on top of the running bucket fill) places them.
        uint16_t(*s_w16)[kMaxBuckets] = reinterpret_cast<uint16_t(*)[kMaxBuckets]>(s_dyn_u + kDecideGroup + kDecideGroup * 3 / 2);
        constexpr int kSub = 4;  // 32-pair rounds per warp per round
        for (unsigned r0 = 0; r0 < Pb; r0 += kDecideThreads * kSub) {
            for (unsigned w = tid; w < 8u * (nb / 2); w += kDecideThreads)
                reinterpret_cast<unsigned*>(&s_w16[0][0])[(w / (nb / 2)) * (kMaxBuckets / 2) + w % (nb / 2)] = 0u;
            __syncthreads();
            unsigned tl[kSub], jj[kSub], rk[kSub];
#pragma unroll
            for (int q = 0; q < kSub; ++q) {
                const unsigned k = r0 + (unsigned)(warp * kSub + q) * 32 + lane;
                const bool valid = k < Pb;
                tl[q] = valid ? pair_tile(k, jj[q]) : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, tl[q]);
                const unsigned prior = valid ? s_w16[warp][tl[q]] : 0u;
                __syncwarp();
                if (valid && (__ffs(peers) - 1) == lane) s_w16[warp][tl[q]] = (uint16_t)(prior + __popc(peers));
                __syncwarp();
                rk[q] = prior + __popc(peers & lanemask_lt());
            }
            __syncthreads();
            for (unsigned d = tid; d < nb; d += kDecideThreads) {
                unsigned run = s_hist[0][d];
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    const unsigned c = s_w16[w][d];
                    s_w16[w][d] = (uint16_t)run;  // bucket fill <= survivors of the group <= 4096
                    run += c;
                }
                s_hist[0][d] = run;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kSub; ++q)
                if (tl[q] != 0xffffffffu) {
                    const unsigned long long pos = (unsigned long long)P0 + s_start[tl[q]] + s_w16[warp][tl[q]] + rk[q];
                    if (pos < a.pair_cap) a.vals[pos] = base + jj[q];
                }
            __syncthreads();  // the next round clears the warp tables
        }
        // the last group to finish turns the per-tile counts into list starts
        // (one scan, instead of every gather CTA re-reading the same counts)
        __syncthreads();
        __shared__ bool s_last;
        if (tid == 0) s_last = ticket_acq_rel(&a.ctrl->decide_done) == ngroups - 1;
        __syncthreads();
        if (!s_last) return;
        {
            constexpr int kPer = kMaxBuckets / kDecideThreads;
            const unsigned d0 = tid * kPer;
            const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
            unsigned v[kPer], run = 0;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                v[q] = d0 + q < nb ? __ldcg(&a.hist[d0 + q]) : 0u;
                run += v[q];
            }
            unsigned incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            __syncthreads();
            if (lane == 31) s_cnt[1][warp] = incl;
            __syncthreads();
            unsigned ex = incl - run;
            for (int w = 0; w < warp; ++w) ex += s_cnt[1][w];
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                if (d0 + q < nb) a.tile_begin[d0 + q] = min(ex, P);
                ex += v[q];
            }
            if (tid == kDecideThreads - 1) a.tile_begin[nb] = min(ex, P);
        }
        return;
    }
    for (unsigned k = tid; k < Pb; k += kDecideThreads) {
        unsigned lo;
        const unsigned tile = pair_tile(k, lo);
        const unsigned long long pos = (unsigned long long)P0 + k;
        if (pos < a.pair_cap) {
            a.keys[pos] = tile;
            a.vals[pos] = base + lo;
            for (int ps = 0; ps < a.passes; ++ps)
                atomicAdd(&s_hist[ps][(tile >> (a.digit_bits * ps)) & dmask], 1u);
        }
    }
    __syncthreads();
    // first radix pass: this group's digit-count row (plain stores, every digit),
    // its super-row and the global counts of every pass
    unsigned* row = a.tile_hist0 + (uint64_t)g * nb;
    unsigned* super = a.tile_hist0 + (a.sort_tiles_cap + g / kSuperTiles) * nb;
    for (unsigned d = tid; d <= dmask; d += kDecideThreads) {
        const unsigned v = s_hist[0][d];
        row[d] = v;
        if (v) atomicAdd(&super[d], v);
    }
    for (int ps = 0; ps < a.passes; ++ps)
        for (unsigned d = tid; d <= dmask; d += kDecideThreads) {
            const unsigned v = s_hist[ps][d];
            if (v) atomicAdd(&a.hist[ps * kMaxBuckets + d], v);
        }
}

// Stage-2 merge of one survivor's per-tile sums in tile order (backward.hpp:141-145).
__device__ __forceinline__ void merge_partials(const ChainLaunch& a, const SurvivorRecord& rec,
                                               double acc[6]) {
    const unsigned ntx = rec.hi_x / kTile - rec.lo_x / kTile + 1;
    const unsigned nty = rec.hi_y / kTile - rec.lo_y / kTile + 1;
    const unsigned np = ntx * nty;
#pragma unroll
    for (int j = 0; j < 6; ++j) acc[j] = 0.0;
    const float2* part = reinterpret_cast<const float2*>(a.partials + 6ull * rec.pair_base);
    for (unsigned k = 0; k < np; ++k) {
        const float2 p0 = part[3 * k], p1 = part[3 * k + 1], p2 = part[3 * k + 2];
        acc[0] += (double)p0.x;
        acc[1] += (double)p0.y;
        acc[2] += (double)p1.x;
        acc[3] += (double)p1.y;
        acc[4] += (double)p2.x;
        acc[5] += (double)p2.y;
    }
}

// Gradient of set index i (survivor slot cid): the dense planes, or the slot
// planes in slot-gradient mode (coalesced: a CTA's survivors are consecutive).
__device__ __forceinline__ void store_chain(const ChainLaunch& a, uint32_t i, uint32_t cid, const float g[11],
                                            const float dmu[3], const double acc[6]) {
    const bool finite = isfinite(g[10]) && isfinite(g[0] + g[1] + g[2]) &&
                        isfinite(g[3] + g[4] + g[5]) && isfinite(g[6] + g[7] + g[8] + g[9]);
    if (!finite) record_error(a.err, kErrNumeric, i);  // backward.hpp:175-185
    float* dst = a.slot_grads ? a.slot_grads + cid : a.grads + i;
#pragma unroll
    for (int k = 0; k < 11; ++k) dst[(uint64_t)k * a.cap] = g[k];
    if (a.slot_grads) a.gmap[i] = (uint16_t)(cid % kDecideGroupSize + 1);
    if (a.stat_norm) a.stat_norm[i] = (float)sqrt(acc[1] * acc[1] + acc[2] * acc[2]);
    if (a.stat_observed) a.stat_observed[i] = 1;
    if (a.stat_world) {
        a.stat_world[3ull * i + 0] = dmu[0];
        a.stat_world[3ull * i + 1] = dmu[1];
        a.stat_world[3ull * i + 2] = dmu[2];
    }
    if (a.acc_obs && !a.ctrl->pair_overflow) {  // DensifyAccum::add (optimize.hpp:238-245); one survivor per thread; an overflowed slice is replayed
        a.acc_norm[i] += sqrt(acc[1] * acc[1] + acc[2] * acc[2]);
        a.acc_obs[i] += 1;
        a.acc_world[3ull * i + 0] += (double)dmu[0];
        a.acc_world[3ull * i + 1] += (double)dmu[1];
        a.acc_world[3ull * i + 2] += (double)dmu[2];
    }
}

// K_chain: one thread per survivor (backward.hpp:148-185). Survivors that
// fast_prepare resolves (the same decision K_exact made: identical code and
// inputs) take the inverse-free fp32 chain; the rest are deferred to
// K_chain_exact so this kernel stays small in registers.
__global__ void __launch_bounds__(256) k_chain(const ChainLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    // CTA per K_decide group: its survivors sit at slots [g*4096, g*4096 + S_g)
    const unsigned g = blockIdx.x;
    const unsigned S = a.grp_surv[g];
    const bool dense = a.slot_grads == nullptr;  // dense planes: keep the sparse-clear list
    if (dense && g == 0 && threadIdx.x == 0) *a.grads_dirty = a.ctrl->survivors;
    for (unsigned j = threadIdx.x; j < S; j += blockDim.x) {
        const uint32_t cid = g * kDecideGroupSize + j;
        const SurvivorRecord rec = a.records[cid];
        if (dense) a.dirty_idx[atomicAdd(a.dirty_ctr, 1u)] = rec.gidx & ~kExactFlag;
        if (rec.gidx & kExactFlag) continue;  // K_chain_exact (listed by K_decide)
        float pf[11];
        uint32_t i;
        load_cand(a.sparams + cid, pf, i);
        FastFocus ff;
        fast_state(pf, a.slice, ff);
        double acc[6];
        merge_partials(a, rec, acc);
        float g11[11], dmu[3];
        fast_backward(pf, ff, acc, a.slice, g11, dmu);
        store_chain(a, i, cid, g11, dmu, acc);
    }
}

// K_chain_exact: the reference's fp64 chain for the deferred survivors.
__global__ void __launch_bounds__(128) k_chain_exact(const ChainLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned E = *a.exact_count;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const uint32_t cid = a.exact_list[e];  // record slot
        const SurvivorRecord rec = a.records[cid];
        float pf[11];
        uint32_t i;
        load_cand(a.sparams + cid, pf, i);
        double acc[6];
        merge_partials(a, rec, acc);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        Focus f;
        focus_prepare(pd, a.slice, f);
        double gd[11];
        D3 dl_dmu;
        focus_backward(pd, f, acc, a.slice, gd, dl_dmu);
        float g[11], dmu[3] = {(float)dl_dmu.x, (float)dl_dmu.y, (float)dl_dmu.z};
#pragma unroll
        for (int k = 0; k < 11; ++k) g[k] = (float)gd[k];
        store_chain(a, i, cid, g, dmu, acc);
    }
}

// ---- PreparedGaussian in full (render.hpp:68-79) ----------------------------------
// For the survivors listed by slot (set order), every field the reference's
// prepare_gaussians fills, in the reference's own fp64 operation order
// (focus_prepare; this TU is built --fmad=false): alpha, opacity_r,
// alpha_tilde, mu_c, mu_e, sigma_c, sigma_c_inv, sigma_e, mu_2d, cov2d,
// conic, det2 — 47 doubles per survivor (include/gpile_b200.h). Read-out only:
// the pixel kernels use the 48 B SurvivorRecord.
__global__ void __launch_bounds__(128) k_prepared_full(const CandParams* __restrict__ sparams,
                                                       const uint32_t* __restrict__ slots, unsigned S,
                                                       const SliceArgs s, double* __restrict__ out) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    float pf[11];
    uint32_t idx;
    load_cand(sparams + slots[k], pf, idx);
    double pd[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) pd[t] = (double)pf[t];
    Focus f;
    focus_prepare(pd, s, f);
    D33 sigma, rot, sc;
    D3 scale;
    world_covariance(pd, s.mod, sigma, rot, scale);
    if (s.identity_rot) {
        sc = sigma;
    } else {
        D33 Rc;
#pragma unroll
        for (int i = 0; i < 9; ++i) Rc.m[i / 3][i % 3] = s.R[i];
        sc = m33_mul(m33_mul(Rc, sigma), m33_t(Rc));
    }
    double* o = out + 47ull * k;
    o[0] = f.alpha;
    o[1] = f.op;
    o[2] = f.alpha_tilde;
    o[3] = f.mu_c.x, o[4] = f.mu_c.y, o[5] = f.mu_c.z;
    o[6] = f.mu_e.x, o[7] = f.mu_e.y, o[8] = f.mu_e.z;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        o[9 + i] = sc.m[i / 3][i % 3];
        o[18 + i] = f.A.m[i / 3][i % 3];
        o[27 + i] = f.Se.m[i / 3][i % 3];
    }
    o[36] = f.mu_e.x, o[37] = f.mu_e.y;  // mu_2d (render.hpp:53-56)
    o[38] = f.cov_a, o[39] = f.cov_b, o[40] = f.cov_c, o[41] = f.cov_d;
    o[42] = f.con_a, o[43] = f.con_b, o[44] = f.con_c, o[45] = f.con_d;
    o[46] = f.det2;
}

// ---- voxelizer: prepare_voxel_prims + VoxelTiles (voxelize.hpp:52-105) ---------
// Persistent CTAs take 256-primitive chunks in set order. Per primitive: the
// world covariance and its inverse in the reference's fp64 order (support
// bounds must reproduce the reference's integer voxel ranges exactly,
// voxelize.hpp:66-74; invert_covariance raises the same errors), a 64 B record
// for the evaluation kernel, and (8^3-tile, primitive) pairs emitted in
// (primitive, tile) order through the same wait-free ordered prefix as K_exact.
__global__ void __launch_bounds__(256) k_vprep(const VoxPrepLaunch a) {
    __shared__ unsigned s_chunk;
    __shared__ unsigned long long s_incl[256];
    __shared__ uint16_t s_t0[256][3];
    __shared__ uint16_t s_nt[256][2];  // tiles along x and y of the primitive's box
    __shared__ unsigned long long s_warp[8];
    __shared__ unsigned long long s_excl;
    __shared__ unsigned s_hist[kMaxSortPasses][kMaxBuckets];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = tid; k < kMaxSortPasses * kMaxBuckets; k += 256) (&s_hist[0][0])[k] = 0;
    const unsigned dmask = (1u << a.digit_bits) - 1;
    const unsigned nchunks = (a.n + 255) / 256;
    const VoxArgs& v = a.v;
    constexpr float kK = -0.72134752044448170368f;  // -0.5 * log2(e)

    while (true) {
        __syncthreads();
        if (tid == 0) s_chunk = atomicAdd(&a.ctrl->exact_chunk_ctr, 1u);
        __syncthreads();
        const unsigned chunk = s_chunk;
        if (chunk >= nchunks) break;
        const uint32_t i = chunk * 256 + tid;
        unsigned long long val = 0;
        if (i < a.n) {
            float pf[11];
            load_params(a.params, a.cap, i, pf);
            double pd[11];
#pragma unroll
            for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
            D33 sigma, rot, inv;
            D3 scale;
            int e = world_covariance(pd, v.mod, sigma, rot, scale);
            if (!e) e = invert_cov(sigma, scale, v.mod, inv);
            if (e) {
                record_error(a.err, e, i);
            } else {
                const double alpha = 1.0 / (1.0 + exp(-pd[10]));
                int lo[3], hi[3];
                bool inside = true;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double half = v.support * sqrt(sigma.m[d][d]);
                    const double lo_w = pd[d] - half, hi_w = pd[d] + half;
                    lo[d] = max(0, x86_trunc_int(ceil((lo_w - v.origin[d]) / v.spacing[d])));
                    hi[d] = min(v.dims[d] - 1, x86_trunc_int(floor((hi_w - v.origin[d]) / v.spacing[d])));
                    if (lo[d] > hi[d]) inside = false;
                }
                if (inside) {
                    unsigned np = 1;
                    unsigned nt[3];
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const int t0 = lo[d] / v.tile[d];
                        nt[d] = (unsigned)(hi[d] / v.tile[d] - t0 + 1);
                        np *= nt[d];
                        s_t0[tid][d] = (uint16_t)t0;
                    }
                    s_nt[tid][0] = (uint16_t)nt[0];
                    s_nt[tid][1] = (uint16_t)nt[1];
                    val = (1ull << 32) | np;
                    VoxRecord rec;
                    rec.mu[0] = pf[0];
                    rec.mu[1] = pf[1];
                    rec.mu[2] = pf[2];
                    rec.log2a = (float)log2(alpha);
                    rec.a[0] = (float)inv.m[0][0] * kK;
                    rec.a[1] = (float)inv.m[1][1] * kK;
                    rec.a[2] = (float)inv.m[2][2] * kK;
                    rec.a[3] = (float)(inv.m[0][1] + inv.m[1][0]) * kK;
                    rec.a[4] = (float)(inv.m[0][2] + inv.m[2][0]) * kK;
                    rec.a[5] = (float)(inv.m[1][2] + inv.m[2][1]) * kK;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        rec.lo[d] = (uint16_t)lo[d];
                        rec.hi[d] = (uint16_t)hi[d];
                    }
                    rec.gidx = i;
                    rec.pair_base = 0;
                    rec.pad = 0;
                    a.records[i] = rec;
                }
            }
        }
        unsigned long long incl = val;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        unsigned long long add = 0;
        for (int w = 0; w < warp; ++w) add += s_warp[w];
        incl += add;
        s_incl[tid] = incl;
        __syncthreads();
        const unsigned long long agg = s_incl[255];
        if (warp == 0) {
            const unsigned long long excl = warp_prefix_aggregates(a.chunk_words, chunk, agg);
            if (lane == 0) {
                s_excl = excl;
                if (chunk == nchunks - 1) {
                    const unsigned long long tot = excl + agg;
                    const unsigned P = (unsigned)(tot & 0xffffffffull);
                    a.ctrl->survivors = (unsigned)(tot >> 32);
                    a.ctrl->pairs = P;
                    a.ctrl->pair_overflow = (P > a.pair_cap) ? 1u : 0u;
                }
            }
        }
        __syncthreads();
        const unsigned S0 = (unsigned)(s_excl >> 32);
        const unsigned P0 = (unsigned)(s_excl & 0xffffffffull);
        {
            const unsigned long long prev = tid ? s_incl[tid - 1] : 0ull;
            if ((s_incl[tid] >> 32) != (prev >> 32)) {
                a.survivor_list[S0 + (unsigned)(prev >> 32)] = i;
                a.records[i].pair_base = P0 + (unsigned)(prev & 0xffffffffull);
            }
        }
        const unsigned Pb = (unsigned)(agg & 0xffffffffull);
        for (unsigned k = tid; k < Pb; k += 256) {
            unsigned lo = 0, hi = 255;
            while (lo < hi) {
                const unsigned mid = (lo + hi) >> 1;
                if ((unsigned)(s_incl[mid] & 0xffffffffull) > k) hi = mid; else lo = mid + 1;
            }
            const unsigned before = lo ? (unsigned)(s_incl[lo - 1] & 0xffffffffull) : 0u;
            const unsigned local = k - before;
            const unsigned ntx = s_nt[lo][0], nty = s_nt[lo][1];
            const unsigned dx = local % ntx, rest = local / ntx;
            const unsigned dy = rest % nty, dz = rest / nty;
            // z-major tile index (voxelize.hpp:98-101): ((tz * ny) + ty) * nx + tx
            const unsigned tile = ((s_t0[lo][2] + dz) * (unsigned)v.ntiles[1] + (s_t0[lo][1] + dy)) *
                                      (unsigned)v.ntiles[0] + (s_t0[lo][0] + dx);
            const unsigned long long pos = (unsigned long long)P0 + k;
            if (pos < a.pair_cap) {
                a.keys[pos] = tile;
                a.vals[pos] = chunk * 256 + lo;
                if (a.passes > 0) {
                    const uint64_t st = pos / kSortTile;
                    atomicAdd(&a.tile_hist0[st * (dmask + 1) + (tile & dmask)], 1u);
                    atomicAdd(&a.tile_hist0[(a.sort_tiles_cap + st / kSuperTiles) * (dmask + 1) + (tile & dmask)], 1u);
                }
                for (int ps = 0; ps < a.passes; ++ps)
                    atomicAdd(&s_hist[ps][(tile >> (a.digit_bits * ps)) & dmask], 1u);
            }
        }
    }
    __syncthreads();
    for (int ps = 0; ps < a.passes; ++ps)
        for (unsigned d = tid; d <= dmask; d += 256) {
            const unsigned c = s_hist[ps][d];
            if (c) atomicAdd(&a.hist[ps * kMaxBuckets + d], c);
        }
}

// voxelize_backward stage 3 (voxelize.hpp:217-232): merge per-tile sums in
// tile order, dL/dSigma = sym(-Sigma^-1 dL/dSigma^-1 Sigma^-1), world chain.
__global__ void __launch_bounds__(128) k_vchain(const VoxChainLaunch a) {
    const unsigned S = a.ctrl->survivors;
    for (unsigned slot = blockIdx.x * blockDim.x + threadIdx.x; slot < S;
         slot += gridDim.x * blockDim.x) {
        const uint32_t i = a.survivor_list[slot];
        const VoxRecord rec = a.records[i];
        unsigned np = 1;
#pragma unroll
        for (int d = 0; d < 3; ++d) np *= (unsigned)(rec.hi[d] / a.v.tile[d] - rec.lo[d] / a.v.tile[d] + 1);
        double acc[10];
#pragma unroll
        for (int j = 0; j < 10; ++j) acc[j] = 0.0;
        const float* part = a.partials + 10ull * rec.pair_base;
        for (unsigned k = 0; k < np; ++k)
#pragma unroll
            for (int j = 0; j < 10; ++j) acc[j] += (double)part[10 * k + j];
        float pf[11];
        load_params(a.params, a.cap, i, pf);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        D33 sigma, rot, inv;
        D3 scale;
        world_covariance(pd, a.v.mod, sigma, rot, scale);
        invert_cov(sigma, scale, a.v.mod, inv);
        D33 dA;
        dA.m[0][0] = acc[4];
        dA.m[1][1] = acc[5];
        dA.m[2][2] = acc[6];
        dA.m[0][1] = dA.m[1][0] = acc[7];
        dA.m[0][2] = dA.m[2][0] = acc[8];
        dA.m[1][2] = dA.m[2][1] = acc[9];
        D33 ds = m33_scale(m33_mul(m33_mul(inv, dA), inv), -1.0);
        ds = m33_scale(m33_add(ds, m33_t(ds)), 0.5);
        double d_ls[3], d_q[4];
        chain_world(pd, ds, a.v.mod, d_ls, d_q);
        const double alpha = 1.0 / (1.0 + exp(-pd[10]));
        float g[11] = {(float)acc[1], (float)acc[2], (float)acc[3], (float)d_ls[0], (float)d_ls[1],
                       (float)d_ls[2], (float)d_q[0], (float)d_q[1], (float)d_q[2], (float)d_q[3],
                       (float)(acc[0] * (alpha * (1.0 - alpha)))};
        if (!isfinite(g[10] + g[0] + g[3] + g[6])) record_error(a.err, kErrNumeric, i);  // voxelize.hpp:234-238
#pragma unroll
        for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = g[k];
    }
}

}  // namespace

void launch_prepared_full(const CandParams* sparams, const uint32_t* slots, unsigned S, const SliceArgs& s,
                          double* out, cudaStream_t st) {
    if (S) k_prepared_full<<<(S + 127) / 128, 128, 0, st>>>(sparams, slots, S, s, out);
}

void launch_vox_prep(const VoxPrepLaunch& a, cudaStream_t st) {
    if (a.n) k_vprep<<<a.grid, 256, 0, st>>>(a);
}

void launch_vox_chain(const VoxChainLaunch& a, int grid, cudaStream_t st) {
    k_vchain<<<grid, 128, 0, st>>>(a);
}

void launch_prep(const PrepLaunch& a, int num_sms, cudaStream_t st) {
    if (a.n == 0) return;
    const bool filter_on = a.slice.tau > 0.0 && a.slice.mod > 1e-10 && a.slice.mod < 1e10 &&
                           a.slice.sigma_z > 1e-10 && a.slice.sigma_z < 1e10;
    const float log_tau = filter_on ? (float)log(a.slice.tau) : 0.f;
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(k_filter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaFuncSetAttribute(k_filter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFilterSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_filter<true>, kFilterThreads, kFilterSmem);
        if (per_sm < 1) per_sm = 1;
    }
    const uint64_t need = ((uint64_t)a.nfilter * 32 + kFilterThreads - 1) / kFilterThreads;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, (uint64_t)num_sms * per_sm));
    if (a.grads)
        launch_pdl(k_filter<true>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, filter_on ? 1 : 0);
    else
        launch_pdl(k_filter<false>, dim3(grid), dim3(kFilterThreads), kFilterSmem, st, a, log_tau, filter_on ? 1 : 0);
}

void launch_prep_multi(const PrepLaunch* pl, int nb, int num_sms, cudaStream_t st) {
    if (nb < 1 || pl[0].n == 0) return;
    MultiPrep m;
    m.nb = nb;
    for (int k = 0; k < nb; ++k) {
        m.p[k] = pl[k];
        const SliceArgs& sl = pl[k].slice;
        const bool on = sl.tau > 0.0 && sl.mod > 1e-10 && sl.mod < 1e10 && sl.sigma_z > 1e-10 && sl.sigma_z < 1e10;
        m.filter_on[k] = on ? 1 : 0;
        m.log_tau[k] = on ? (float)log(sl.tau) : 0.f;
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
    launch_pdl(k_adam_cull, dim3(grid), dim3(256), 0, st, a, f, log_tau, filter_on ? 1 : 0);
}

void launch_bin(const PrepLaunch& a, cudaStream_t st) {
    if (!a.n) return;
    const int smem = kDecideGroup * (4 + 6) + 8 * kMaxBuckets * 2;  // + the stable fill's warp tables
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const unsigned groups = (a.nfilter + kDecideChunks - 1) / kDecideChunks;
    launch_pdl(k_decide, dim3(groups), dim3(kDecideThreads), smem, st, a);
}

void launch_chain(const ChainLaunch& a, int grid, cudaStream_t st) {
    launch_pdl(k_chain, dim3(grid), dim3(256), 0, st, a);
}

void launch_chain_exact(const ChainLaunch& a, int grid, cudaStream_t st) {
    launch_pdl(k_chain_exact, dim3(std::max(1, grid / 8)), dim3(128), 0, st, a);
}

}  // namespace gpk
