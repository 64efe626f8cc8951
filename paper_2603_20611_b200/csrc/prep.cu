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

__device__ __forceinline__ void load_params(const float* __restrict__ params, uint64_t cap,
                                            uint32_t i, float p[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) p[k] = __ldg(params + (uint64_t)k * cap + i);
}

__device__ __forceinline__ void zero_grads(float* grads, uint64_t cap, uint32_t i) {
#pragma unroll
    for (int k = 0; k < 11; ++k) grads[(uint64_t)k * cap + i] = 0.f;
}

// ---- K_filter ------------------------------------------------------------------
template <bool kZeroGrads>
__global__ void __launch_bounds__(kPrepThreads) k_filter(const PrepLaunch a, float log_tau,
                                                         int filter_on) {
    constexpr int kSlots = kFilterItems * 8;  // (item, warp) counts, in set order
    __shared__ unsigned s_off[kSlots];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned b = blockIdx.x;
    const uint32_t base = b * kFilterBlock;
    const float mod_f = (float)a.slice.mod;
    const float sz2 = (float)(a.slice.sigma_z * a.slice.sigma_z);

    // Housekeeping: clear the per-sort-tile digit histograms the previous
    // prepare used (all passes) before K_exact / the radix passes refill them.
    {
        const uint64_t row = a.sort_tiles_cap * 256;
        const uint64_t used = (uint64_t)(*a.prev_sort_tiles) * 256;
        const uint64_t total = (uint64_t)a.passes * used;
        if (used)
            for (uint64_t w = (uint64_t)b * kPrepThreads + tid; w < total;
                 w += (uint64_t)gridDim.x * kPrepThreads)
                a.tile_hist_all[(w / used) * row + (w % used)] = 0u;
    }

    unsigned ballots[kFilterItems];
#pragma unroll
    for (int k = 0; k < kFilterItems; ++k) {
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
        if (lane == 0) s_off[k * 8 + warp] = __popc(ballots[k]);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 64 slots, two per lane
        const unsigned c0 = s_off[2 * lane], c1 = s_off[2 * lane + 1];
        unsigned incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const unsigned ex = incl - c0 - c1;
        __syncwarp();
        s_off[2 * lane] = ex;
        s_off[2 * lane + 1] = ex + c0;
        if (lane == 31) a.filter_counts[b] = incl;
    }
    __syncthreads();
    uint32_t* out = a.cand_local + (uint64_t)b * kFilterBlock;
#pragma unroll
    for (int k = 0; k < kFilterItems; ++k) {
        if (ballots[k] & (1u << lane))
            out[s_off[k * 8 + warp] + __popc(ballots[k] & lanemask_lt())] = base + k * kPrepThreads + tid;
    }
}

// ---- K_exact -------------------------------------------------------------------
template <bool kZeroGrads>
__global__ void __launch_bounds__(kExactChunk) k_exact(const PrepLaunch a) {
    extern __shared__ unsigned s_bpre[];                 // exclusive prefix of filter counts (nfilter+1)
    __shared__ unsigned s_chunk;
    __shared__ unsigned long long s_incl[kExactChunk];   // (survivors << 32) | pairs, inclusive
    __shared__ uint16_t s_rect[kExactChunk][3];          // tx0, ty0, ntx
    __shared__ unsigned long long s_warp[kExactChunk / 32];
    __shared__ unsigned long long s_excl;
    __shared__ unsigned s_hist[kMaxSortPasses][256];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = tid; k < kMaxSortPasses * 256; k += kExactChunk) (&s_hist[0][0])[k] = 0;
    // candidate layout: exclusive prefix over the K_filter blocks' counts
    {
        const unsigned nb = a.nfilter;
        unsigned carry = 0;
        for (unsigned base = 0; base < nb; base += kExactChunk) {
            const unsigned j = base + tid;
            const unsigned v = j < nb ? a.filter_counts[j] : 0u;
            unsigned incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) s_warp[warp] = incl;
            __syncthreads();
            unsigned add = carry;
            for (int w = 0; w < warp; ++w) add += (unsigned)s_warp[w];
            if (j < nb) s_bpre[j] = add + incl - v;
            unsigned tot = 0;
            for (int w = 0; w < kExactChunk / 32; ++w) tot += (unsigned)s_warp[w];
            carry += tot;
            __syncthreads();
        }
        if (tid == 0) s_bpre[nb] = carry;
        __syncthreads();
    }
    const unsigned C = s_bpre[a.nfilter];
    const unsigned nchunks = (C + kExactChunk - 1) / kExactChunk;
    const int tiles_x = a.slice.tiles_x;

    while (true) {
        __syncthreads();
        if (tid == 0) s_chunk = atomicAdd(&a.ctrl->exact_chunk_ctr, 1u);
        __syncthreads();
        const unsigned chunk = s_chunk;
        if (chunk >= nchunks) break;
        const unsigned c = chunk * kExactChunk + tid;
        unsigned long long v = 0;
        if (c < C) {
            // filter block holding candidate c: last b with s_bpre[b] <= c
            unsigned lo = 0, hi = a.nfilter - 1;
            while (lo < hi) {
                const unsigned mid = (lo + hi + 1) >> 1;
                if (s_bpre[mid] <= c) lo = mid; else hi = mid - 1;
            }
            const uint32_t i = a.cand_local[(uint64_t)lo * kFilterBlock + (c - s_bpre[lo])];
            float pf[11];
            load_params(a.params, a.cap, i, pf);
            double pd[11];
#pragma unroll
            for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
            Focus f;
            const int r = focus_prepare(pd, a.slice, f);
            if (r == kSurvive) {
                const int tx0 = f.lo_x / kTile, tx1 = f.hi_x / kTile;
                const int ty0 = f.lo_y / kTile, ty1 = f.hi_y / kTile;
                const unsigned ntx = tx1 - tx0 + 1, nty = ty1 - ty0 + 1;
                v = (1ull << 32) | (unsigned long long)(ntx * nty);
                s_rect[tid][0] = (uint16_t)tx0;
                s_rect[tid][1] = (uint16_t)ty0;
                s_rect[tid][2] = (uint16_t)ntx;
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
                a.records[c] = rec;
            } else {
                if (r > 0) record_error(a.err, r, i);
                if (kZeroGrads) zero_grads(a.grads, a.cap, i);
            }
        }
        // block inclusive scan of (survivor, pairs)
        unsigned long long incl = v;
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
        const unsigned long long agg = s_incl[kExactChunk - 1];
        if (warp == 0) {
            const unsigned long long excl = warp_prefix_aggregates(a.exact_words, chunk, agg);
            if (lane == 0) {
                s_excl = excl;
                if (chunk == nchunks - 1) {
                    const unsigned long long tot = excl + agg;
                    const unsigned S = (unsigned)(tot >> 32), P = (unsigned)(tot & 0xffffffffull);
                    a.ctrl->survivors = S;
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
                a.survivor_list[S0 + (unsigned)(prev >> 32)] = c;
                a.records[c].pair_base = P0 + (unsigned)(prev & 0xffffffffull);
            }
        }
        // cooperative, balanced pair emission in (candidate, tile) order
        const unsigned Pb = (unsigned)(agg & 0xffffffffull);
        for (unsigned k = tid; k < Pb; k += kExactChunk) {
            unsigned lo = 0, hi = kExactChunk - 1;
            while (lo < hi) {
                const unsigned mid = (lo + hi) >> 1;
                if ((unsigned)(s_incl[mid] & 0xffffffffull) > k) hi = mid; else lo = mid + 1;
            }
            const unsigned before = lo ? (unsigned)(s_incl[lo - 1] & 0xffffffffull) : 0u;
            const unsigned local = k - before;
            const unsigned ntx = s_rect[lo][2];
            const unsigned ty = s_rect[lo][1] + local / ntx;
            const unsigned tx = s_rect[lo][0] + local % ntx;
            const unsigned tile = ty * (unsigned)tiles_x + tx;
            const unsigned long long pos = (unsigned long long)P0 + k;
            if (pos < a.pair_cap) {
                a.keys[pos] = tile;
                a.vals[pos] = chunk * kExactChunk + lo;
                if (a.passes > 0)
                    atomicAdd(&a.tile_hist0[(pos / kSortTile) * 256 + (tile & 255u)], 1u);
                for (int ps = 0; ps < a.passes; ++ps)
                    atomicAdd(&s_hist[ps][(tile >> (8 * ps)) & 255u], 1u);
            }
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
        focus_prepare(pd, a.slice, f);  // deterministic: same state as K_exact
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

int exact_blocks_per_sm(size_t dyn_smem) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_exact<true>, kExactChunk, dyn_smem);
    return nb > 0 ? nb : 1;
}

size_t exact_dyn_smem(unsigned nfilter) { return (size_t)(nfilter + 1) * sizeof(unsigned); }

void launch_filter(const PrepLaunch& a, cudaStream_t st) {
    if (a.n == 0) return;
    const bool filter_on = a.slice.tau > 0.0 && a.slice.mod > 1e-10 && a.slice.mod < 1e10 &&
                           a.slice.sigma_z > 1e-10 && a.slice.sigma_z < 1e10;
    const float log_tau = filter_on ? (float)log(a.slice.tau) : 0.f;
    if (a.grads)
        k_filter<true><<<a.nfilter, kPrepThreads, 0, st>>>(a, log_tau, filter_on ? 1 : 0);
    else
        k_filter<false><<<a.nfilter, kPrepThreads, 0, st>>>(a, log_tau, filter_on ? 1 : 0);
}

void launch_exact(const PrepLaunch& a, cudaStream_t st) {
    if (a.n == 0) return;
    const size_t smem = exact_dyn_smem(a.nfilter);
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_exact<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_exact<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    if (a.grads)
        k_exact<true><<<a.exact_grid, kExactChunk, smem, st>>>(a);
    else
        k_exact<false><<<a.exact_grid, kExactChunk, smem, st>>>(a);
}

void launch_chain(const ChainLaunch& a, int grid, cudaStream_t st) {
    k_chain<<<grid, 128, 0, st>>>(a);
}

}  // namespace gpk
