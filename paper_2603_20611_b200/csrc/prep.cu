// prep.cu — K_prep (preprocess + cull + bounds + pair emission) and K_chain
// (backward chain to world parameters). Built with --fmad=false so the fp64
// focus algebra rounds like the reference (see focus.cuh).
//
// K_prep replaces prepare_gaussians (render.hpp:83-138) + the TileGrid build
// (render.hpp:142-160) for one slice:
//   1. one thread per Gaussian, coalesced SoA loads; an fp32 CERTAIN-CULL test
//      in closed form (q = mu_cz^2 / (sigma_z^2 + Sigma_c,zz))
//      with a safety margin that covers fp32 error and the reference's own
//      cancellation noise; everything not certainly culled is a candidate.
//      Dense gradients of certainly-culled primitives are zero-filled here
//      (grad_chain.hpp:12-22 exact zeros) so the gradient plane is written once.
//   2. order-preserving block compaction of candidates, then the exact fp64
//      reference computation (focus_prepare) on the dense candidate list.
//   3. a decoupled-lookback chained scan over blocks yields, in set order, the
//      survivor slots and each survivor's first pair position; pairs
//      (tile key, candidate id) are emitted in (id, tile) order — the order a
//      stable sort on the tile key needs to reproduce the reference lists.
//   4. per-block digit histograms for the radix passes.
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
    // columns of R(q)
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

__device__ __forceinline__ void load_params(const float* __restrict__ params, uint64_t cap,
                                            uint32_t i, float p[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) p[k] = __ldg(params + (uint64_t)k * cap + i);
}

__device__ __forceinline__ void zero_grads(float* grads, uint64_t cap, uint32_t i) {
#pragma unroll
    for (int k = 0; k < 11; ++k) grads[(uint64_t)k * cap + i] = 0.f;
}

// Block-wide inclusive scan of one 64-bit value per thread (256 threads).
__device__ __forceinline__ unsigned long long block_incl_scan64(unsigned long long v,
                                                                unsigned long long* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    unsigned long long add = 0;
    for (int w = 0; w < warp; ++w) add += s_warp[w];
    __syncthreads();
    return v + add;
}

template <bool kZeroGrads>
__global__ void __launch_bounds__(kPrepThreads) k_prep(const PrepLaunch a, float log_tau,
                                                       int filter_on, unsigned nblocks) {
    __shared__ unsigned s_bid;
    __shared__ unsigned s_wcnt[kPrepItems * 8];
    __shared__ unsigned s_ncand;
    __shared__ uint32_t s_cand[kPrepBlock];
    __shared__ unsigned long long s_incl[kPrepBlock];   // (survivors << 32) | pairs, inclusive
    __shared__ uint16_t s_rect[kPrepBlock][3];           // tx0, ty0, ntx
    __shared__ unsigned long long s_warp[8];
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned s_hist[kMaxSortPasses][256];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_bid = atomicAdd(&a.ctrl->prep_block_ctr, 1u);
        if (s_bid == 0) atomicAdd(a.epoch, 1u);  // new epoch for this prepare's sort passes
    }
    for (int k = tid; k < kMaxSortPasses * 256; k += kPrepThreads) (&s_hist[0][0])[k] = 0;
    __syncthreads();
    const unsigned b = s_bid;
    const uint32_t base = b * kPrepBlock;
    const float mod_f = (float)a.slice.mod;
    const float sz2 = (float)(a.slice.sigma_z * a.slice.sigma_z);

    // ---- phase 1: certain-cull filter, zero-fill, candidate flags ----------
    unsigned ballots[kPrepItems];
#pragma unroll
    for (int k = 0; k < kPrepItems; ++k) {
        const uint32_t i = base + k * kPrepThreads + tid;
        bool cand = false;
        if (i < a.n) {
            cand = true;
            if (filter_on) {
                float p[11];
                load_params(a.params, a.cap, i, p);
                cand = !certainly_culled(p, a.slice, log_tau, mod_f, sz2);
            }
            if (kZeroGrads && !cand) zero_grads(a.grads, a.cap, i);
        }
        ballots[k] = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) s_wcnt[k * 8 + warp] = __popc(ballots[k]);
    }
    __syncthreads();
    if (warp == 0) {
        const unsigned v = s_wcnt[lane];
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        s_wcnt[lane] = incl - v;
        if (lane == 31) s_ncand = incl;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPrepItems; ++k) {
        if (ballots[k] & (1u << lane)) {
            const unsigned pos = s_wcnt[k * 8 + warp] + __popc(ballots[k] & lanemask_lt());
            s_cand[pos] = base + k * kPrepThreads + tid;
        }
    }
    __syncthreads();
    const unsigned nc = s_ncand;

    // ---- phase 2: exact fp64 reference path on the dense candidate list ----
    for (unsigned c = tid; c < nc; c += kPrepThreads) {
        const uint32_t i = s_cand[c];
        float pf[11];
        load_params(a.params, a.cap, i, pf);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        Focus f;
        const int r = focus_prepare(pd, a.slice, f);
        unsigned long long v = 0;
        if (r == kSurvive) {
            const int tx0 = f.lo_x / kTile, tx1 = f.hi_x / kTile;
            const int ty0 = f.lo_y / kTile, ty1 = f.hi_y / kTile;
            const unsigned ntx = tx1 - tx0 + 1, nty = ty1 - ty0 + 1;
            v = (1ull << 32) | (unsigned long long)(ntx * nty);
            s_rect[c][0] = (uint16_t)tx0;
            s_rect[c][1] = (uint16_t)ty0;
            s_rect[c][2] = (uint16_t)ntx;
            SurvivorRecord rec;
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
            rec.gidx = i;
            rec.pair_base = 0;
            a.records[base + c] = rec;
        } else {
            if (r > 0) record_error(a.err, r, i);
            if (kZeroGrads) zero_grads(a.grads, a.cap, i);
        }
        s_incl[c] = v;
    }
    __syncthreads();

    // ---- phase 3: block scan of (survivor, pairs) over candidates ----------
    // Each thread owns 4 consecutive candidates.
    {
        unsigned long long loc[kPrepItems];
        unsigned long long run = 0;
#pragma unroll
        for (int k = 0; k < kPrepItems; ++k) {
            const unsigned c = tid * kPrepItems + k;
            run += (c < nc) ? s_incl[c] : 0ull;
            loc[k] = run;
        }
        const unsigned long long incl = block_incl_scan64(run, s_warp);
        const unsigned long long excl = incl - run;
#pragma unroll
        for (int k = 0; k < kPrepItems; ++k) {
            const unsigned c = tid * kPrepItems + k;
            if (c < nc) s_incl[c] = excl + loc[k];
        }
    }
    __syncthreads();
    const unsigned long long agg = nc ? s_incl[nc - 1] : 0ull;

    // ---- phase 4: decoupled look-back across blocks --------------------------
    if (warp == 0) {
        unsigned long long excl = 0;
        if (b == 0) {
            if (lane == 0) {
                a.prep_incl[0] = agg;
                st_release_u32(&a.prep_flags[0], 2u);
            }
        } else {
            if (lane == 0) {
                a.prep_agg[b] = agg;
                st_release_u32(&a.prep_flags[b], 1u);
            }
            int j = (int)b - 1;
            while (true) {
                const int idx = j - lane;
                unsigned f = 2u;
                unsigned long long val = 0;
                if (idx >= 0) {
                    do {
                        f = ld_acquire_u32(&a.prep_flags[idx]);
                    } while (f == 0u);
                    val = (f == 2u) ? ld_relaxed_u64(&a.prep_incl[idx])
                                    : ld_relaxed_u64(&a.prep_agg[idx]);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, f == 2u);
                if (pm) {
                    const int first = __ffs(pm) - 1;
                    unsigned long long part = (lane <= first) ? val : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                    excl += part;
                    break;
                }
                unsigned long long part = val;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                j -= 32;
            }
            if (lane == 0) {
                a.prep_incl[b] = excl + agg;
                st_release_u32(&a.prep_flags[b], 2u);
            }
        }
        if (lane == 0) {
            s_prefix = excl;
            if (b == nblocks - 1) {
                const unsigned long long tot = excl + agg;
                const unsigned S = (unsigned)(tot >> 32), P = (unsigned)(tot & 0xffffffffull);
                a.ctrl->survivors = S;
                a.ctrl->pairs = P;
                a.ctrl->pair_overflow = (P > a.pair_cap) ? 1u : 0u;
            }
        }
    }
    __syncthreads();
    const unsigned S0 = (unsigned)(s_prefix >> 32);
    const unsigned P0 = (unsigned)(s_prefix & 0xffffffffull);

    // ---- phase 5: survivor slots, pair bases, cooperative pair emission -----
    for (unsigned c = tid; c < nc; c += kPrepThreads) {
        const unsigned long long inc = s_incl[c];
        const unsigned long long prev = c ? s_incl[c - 1] : 0ull;
        if ((inc >> 32) != (prev >> 32)) {
            const unsigned slot = S0 + (unsigned)(prev >> 32);
            a.survivor_list[slot] = base + c;
            a.records[base + c].pair_base = P0 + (unsigned)(prev & 0xffffffffull);
        }
    }
    const unsigned Pb = (unsigned)(agg & 0xffffffffull);
    const int tiles_x = a.slice.tiles_x;
    for (unsigned k = tid; k < Pb; k += kPrepThreads) {
        // candidate c = first with inclusive pair count > k
        unsigned lo = 0, hi = nc - 1;
        while (lo < hi) {
            const unsigned mid = (lo + hi) >> 1;
            if ((unsigned)(s_incl[mid] & 0xffffffffull) > k) hi = mid; else lo = mid + 1;
        }
        const unsigned c = lo;
        const unsigned before = c ? (unsigned)(s_incl[c - 1] & 0xffffffffull) : 0u;
        const unsigned local = k - before;
        const unsigned ntx = s_rect[c][2];
        const unsigned ty = s_rect[c][1] + local / ntx;
        const unsigned tx = s_rect[c][0] + local % ntx;
        const unsigned tile = ty * (unsigned)tiles_x + tx;
        const unsigned long long pos = (unsigned long long)P0 + k;
        if (pos < a.pair_cap) {
            a.keys[pos] = tile;
            a.vals[pos] = base + c;
            for (int ps = 0; ps < a.passes; ++ps) atomicAdd(&s_hist[ps][(tile >> (8 * ps)) & 255u], 1u);
        }
    }
    __syncthreads();
    for (int ps = 0; ps < a.passes; ++ps) {
        const unsigned v = s_hist[ps][tid];
        if (v) atomicAdd(&a.hist[ps * 256 + tid], v);
    }
}

// K_chain: one thread per survivor (backward.hpp:148-185).
__global__ void __launch_bounds__(128) k_chain(const ChainLaunch a) {
    const unsigned S = a.ctrl->survivors;
    for (unsigned slot = blockIdx.x * blockDim.x + threadIdx.x; slot < S;
         slot += gridDim.x * blockDim.x) {
        const uint32_t cid = a.survivor_list[slot];
        const SurvivorRecord rec = a.records[cid];
        const uint32_t i = rec.gidx;
        float pf[11];
        load_params(a.params, a.cap, i, pf);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        Focus f;
        focus_prepare(pd, a.slice, f);  // deterministic: same state as K_prep
        const unsigned ntx = rec.hi_x / kTile - rec.lo_x / kTile + 1;
        const unsigned nty = rec.hi_y / kTile - rec.lo_y / kTile + 1;
        const unsigned np = ntx * nty;
        // stage-2 merge in tile order (backward.hpp:141-145)
        double acc[6] = {0, 0, 0, 0, 0, 0};
        const float* part = a.partials + 6ull * rec.pair_base;
        for (unsigned k = 0; k < np; ++k) {
#pragma unroll
            for (int j = 0; j < 6; ++j) acc[j] += (double)part[6 * k + j];
        }
        double g[11];
        D3 dl_dmu;
        focus_backward(pd, f, acc, a.slice, g, dl_dmu);
        const bool finite = isfinite(g[10]) && isfinite(g[0] + g[1] + g[2]) &&
                            isfinite(g[3] + g[4] + g[5]) && isfinite(g[6] + g[7] + g[8] + g[9]);
        if (!finite) record_error(a.err, kErrNumeric, i);
#pragma unroll
        for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = (float)g[k];
        if (a.stat_norm) a.stat_norm[i] = (float)sqrt(acc[1] * acc[1] + acc[2] * acc[2]);
        if (a.stat_observed) a.stat_observed[i] = 1;
        if (a.stat_world) {
            a.stat_world[3ull * i + 0] = (float)dl_dmu.x;
            a.stat_world[3ull * i + 1] = (float)dl_dmu.y;
            a.stat_world[3ull * i + 2] = (float)dl_dmu.z;
        }
    }
}

}  // namespace

void launch_prep(const PrepLaunch& a, cudaStream_t st) {
    if (a.n == 0) return;
    const unsigned nblocks = (a.n + kPrepBlock - 1) / kPrepBlock;
    const bool filter_on = a.slice.tau > 0.0 && a.slice.mod > 1e-10 && a.slice.mod < 1e10 &&
                           a.slice.sigma_z > 1e-10 && a.slice.sigma_z < 1e10;
    const float log_tau = filter_on ? (float)log(a.slice.tau) : 0.f;
    if (a.grads)
        k_prep<true><<<nblocks, kPrepThreads, 0, st>>>(a, log_tau, filter_on ? 1 : 0, nblocks);
    else
        k_prep<false><<<nblocks, kPrepThreads, 0, st>>>(a, log_tau, filter_on ? 1 : 0, nblocks);
}

void launch_chain(const ChainLaunch& a, int grid, cudaStream_t st) {
    k_chain<<<grid, 128, 0, st>>>(a);
}

}  // namespace gpk
