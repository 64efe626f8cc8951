// densify.cu — adaptive density control on the device: densify_and_prune
// (optimize.hpp:228-344) over the session-resident SoA planes.
//
// The reference walks the set in index order and builds
//   next = [kept primitives (incl. the originals of clones), in index order]
//        ++ [born primitives: a clone's copy, or a split's two children, in
//            the index order of their parents]                      (:300-322)
// with Adam moments copied for the kept and zero for the born (:324-340).
// Here that order is two exclusive scans: K_dens_classify decides each
// primitive's fate (prune / keep / clone / split, :262-289) and reduces the
// per-block counts of kept, born and split primitives; K_dens_scan turns the
// block counts into block offsets (one CTA); K_dens_emit re-derives the
// in-block ranks with a block scan and writes the new planes (params, m, v)
// at their final positions. The split children's normals (Rng::normal drawn
// sequentially in parent order, :310) are drawn on the host between the scan
// and the emit — the host knows the split count from the scan's totals.
//
// Decisions are fp64 from the stored fp32 parameters with the reference's
// expressions (alpha_activation core.hpp:21, scale() core.hpp:39-41, mean
// screen gradient :271-272); this file is built with --fmad=false so the
// clone / split arithmetic rounds like the reference's x86-64 build before
// the final fp32 store.
//
// Bytes per primitive: read 33 f32 (params, m, v) + 40 B accumulators, write
// ≤ 33 f32 (+ 33 per born primitive); a densify event runs every
// densify_interval (100) iterations, so it is far off the step's critical path.
#include "common.cuh"
#include "focus.cuh"

namespace gpk {

namespace {

constexpr int kDensThreads = 256;
constexpr int kDensItems = 4;
constexpr int kDensBlock = kDensThreads * kDensItems;

enum : uint8_t { kPrune = 0, kKeep = 1, kClone = 2, kSplit = 3 };

__device__ __forceinline__ uint8_t classify(const DensifyLaunch& a, uint64_t i) {
    const double raw = (double)a.params[10 * a.cap + i];
    const double alpha = 1.0 / (1.0 + exp(-raw));  // alpha_activation (core.hpp:21)
    const int obs = a.acc_obs[i];
    if (alpha < a.tau || obs == 0) return kPrune;  // optimize.hpp:263
    const double mean_grad = obs > 0 ? a.acc_norm[i] / obs : 0.0;
    if (mean_grad <= a.grad_threshold) return kKeep;  // :268
    const double sx = exp((double)a.params[3 * a.cap + i]);
    const double sy = exp((double)a.params[4 * a.cap + i]);
    const double sz = exp((double)a.params[5 * a.cap + i]);
    const double max_scale = fmax(sx, fmax(sy, sz));
    return max_scale <= a.split_threshold ? kClone : kSplit;  // :275
}

// counts of (kept, born, split) for one class
__device__ __forceinline__ uint3 class_counts(uint8_t c) {
    return make_uint3(c == kKeep || c == kClone, c == kClone ? 1u : c == kSplit ? 2u : 0u, c == kSplit);
}

__device__ __forceinline__ uint3 add3(uint3 x, uint3 y) { return make_uint3(x.x + y.x, x.y + y.y, x.z + y.z); }

__device__ __forceinline__ uint3 warp_incl_scan3(uint3 v) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned x = __shfl_up_sync(0xffffffffu, v.x, o);
        const unsigned y = __shfl_up_sync(0xffffffffu, v.y, o);
        const unsigned z = __shfl_up_sync(0xffffffffu, v.z, o);
        if (lane >= (unsigned)o) v = add3(v, make_uint3(x, y, z));
    }
    return v;
}

// Block-wide exclusive scan of per-thread triples; returns the thread's
// exclusive prefix and (in *total) the block total.
__device__ __forceinline__ uint3 block_excl_scan3(uint3 v, uint3* total) {
    __shared__ uint3 warp_tot[kDensThreads / 32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint3 inc = warp_incl_scan3(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    uint3 off = make_uint3(0, 0, 0), tot = make_uint3(0, 0, 0);
#pragma unroll
    for (unsigned w = 0; w < kDensThreads / 32; ++w) {
        if (w < warp) off = add3(off, warp_tot[w]);
        tot = add3(tot, warp_tot[w]);
    }
    *total = tot;
    return make_uint3(off.x + inc.x - v.x, off.y + inc.y - v.y, off.z + inc.z - v.z);
}

__global__ void __launch_bounds__(kDensThreads) k_dens_classify(const DensifyLaunch a) {
    const uint64_t base = (uint64_t)blockIdx.x * kDensBlock + (uint64_t)threadIdx.x * kDensItems;
    uint3 cnt = make_uint3(0, 0, 0);
#pragma unroll
    for (int k = 0; k < kDensItems; ++k) {
        const uint64_t i = base + k;
        if (i >= a.n) break;
        const uint8_t c = classify(a, i);
        a.cls[i] = c;
        cnt = add3(cnt, class_counts(c));
    }
    uint3 tot;
    block_excl_scan3(cnt, &tot);
    if (threadIdx.x == 0) {
        a.block_sums[3ull * blockIdx.x + 0] = tot.x;
        a.block_sums[3ull * blockIdx.x + 1] = tot.y;
        a.block_sums[3ull * blockIdx.x + 2] = tot.z;
    }
}

// One CTA: exclusive scan of the block counts in place; totals[0..2] = sums.
__global__ void __launch_bounds__(kDensThreads) k_dens_scan(const DensifyLaunch a, unsigned nblocks) {
    __shared__ uint3 carry;
    if (threadIdx.x == 0) carry = make_uint3(0, 0, 0);
    __syncthreads();
    for (unsigned b0 = 0; b0 < nblocks; b0 += kDensThreads) {
        const unsigned b = b0 + threadIdx.x;
        uint3 v = make_uint3(0, 0, 0);
        if (b < nblocks) v = make_uint3(a.block_sums[3ull * b], a.block_sums[3ull * b + 1], a.block_sums[3ull * b + 2]);
        uint3 tot;
        const uint3 ex = block_excl_scan3(v, &tot);
        const uint3 c = carry;
        if (b < nblocks) {
            a.block_sums[3ull * b + 0] = c.x + ex.x;
            a.block_sums[3ull * b + 1] = c.y + ex.y;
            a.block_sums[3ull * b + 2] = c.z + ex.z;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry = add3(c, tot);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.totals[0] = carry.x;
        a.totals[1] = carry.y;
        a.totals[2] = carry.z;
    }
}

__device__ __forceinline__ void copy_primitive(const DensifyLaunch& a, uint64_t i, uint64_t dst) {
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        a.out_params[k * a.cap_out + dst] = a.params[k * a.cap + i];
        a.out_m[k * a.cap_out + dst] = a.m[k * a.cap + i];
        a.out_v[k * a.cap_out + dst] = a.v[k * a.cap + i];
    }
}

__device__ __forceinline__ double clamp_axis(double p, double lo, double hi) { return fmin(hi, fmax(lo, p)); }

// A born primitive (moments stay zero: the output planes were cleared).
__device__ __forceinline__ void store_born(const DensifyLaunch& a, uint64_t dst, const double mu[3],
                                           const double ls[3], uint64_t src) {
    for (int d = 0; d < 3; ++d) {
        a.out_params[d * a.cap_out + dst] = (float)mu[d];
        a.out_params[(3 + d) * a.cap_out + dst] = (float)ls[d];
    }
    for (int k = 6; k < 11; ++k) a.out_params[k * a.cap_out + dst] = a.params[k * a.cap + src];
}

__global__ void __launch_bounds__(kDensThreads) k_dens_emit(const DensifyLaunch a) {
    const uint64_t base = (uint64_t)blockIdx.x * kDensBlock + (uint64_t)threadIdx.x * kDensItems;
    uint8_t cls[kDensItems];
    uint3 cnt = make_uint3(0, 0, 0);
#pragma unroll
    for (int k = 0; k < kDensItems; ++k) {
        const uint64_t i = base + k;
        cls[k] = i < a.n ? a.cls[i] : kPrune;
        cnt = add3(cnt, class_counts(cls[k]));
    }
    uint3 tot;
    uint3 r = block_excl_scan3(cnt, &tot);
    r.x += a.block_sums[3ull * blockIdx.x + 0];
    r.y += a.block_sums[3ull * blockIdx.x + 1];
    r.z += a.block_sums[3ull * blockIdx.x + 2];
    const uint64_t kept_total = a.totals[0];
#pragma unroll 1
    for (int k = 0; k < kDensItems; ++k) {
        const uint64_t i = base + k;
        const uint8_t c = cls[k];
        if (c == kPrune) continue;
        if (c != kSplit) copy_primitive(a, i, r.x);  // keep, or a clone's original
        double mu[3], ls[3];
        for (int d = 0; d < 3; ++d) {
            mu[d] = (double)a.params[d * a.cap + i];
            ls[d] = (double)a.params[(3 + d) * a.cap + i];
        }
        if (c == kClone) {
            // offset along the accumulated world gradient, by the scale (:279-286)
            double dir[3] = {a.acc_world[3 * i], a.acc_world[3 * i + 1], a.acc_world[3 * i + 2]};
            const double dn = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
            double out[3] = {mu[0], mu[1], mu[2]};
            if (dn > 0.0) {
                const double inv = 1.0 / dn;
                for (int d = 0; d < 3; ++d) {
                    const double s = exp(ls[d]);
                    out[d] = clamp_axis(mu[d] + (dir[d] * inv) * s, a.bmin[d], a.bmax[d]);
                }
            }
            store_born(a, kept_total + r.y, out, ls, i);
        } else if (c == kSplit) {
            // two children drawn from the parent, scales shrunk (:290-300)
            D33 rot;
            quat_rotation((double)a.params[6 * a.cap + i], (double)a.params[7 * a.cap + i],
                          (double)a.params[8 * a.cap + i], (double)a.params[9 * a.cap + i], rot);
            const double s[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
            for (int child = 0; child < 2; ++child) {
                const double* xi = a.normals + 6ull * r.z + 3 * child;
                const double v[3] = {s[0] * xi[0] * a.mod, s[1] * xi[1] * a.mod, s[2] * xi[2] * a.mod};
                double out[3], cls_ls[3];
                for (int d = 0; d < 3; ++d) {
                    const double off = rot.m[d][0] * v[0] + rot.m[d][1] * v[1] + rot.m[d][2] * v[2];
                    out[d] = clamp_axis(mu[d] + off, a.bmin[d], a.bmax[d]);
                    cls_ls[d] = ls[d] - a.shrink;
                }
                store_born(a, kept_total + r.y + child, out, cls_ls, i);
            }
        }
        const uint3 cc = class_counts(c);
        r = add3(r, cc);
    }
}

}  // namespace

unsigned densify_blocks(uint64_t n) { return (unsigned)((n + kDensBlock - 1) / kDensBlock); }

void launch_densify_classify(const DensifyLaunch& a, cudaStream_t st) {
    const unsigned nb = densify_blocks(a.n);
    if (nb) k_dens_classify<<<nb, kDensThreads, 0, st>>>(a);
    k_dens_scan<<<1, kDensThreads, 0, st>>>(a, nb);
}

void launch_densify_emit(const DensifyLaunch& a, cudaStream_t st) {
    const unsigned nb = densify_blocks(a.n);
    if (nb) k_dens_emit<<<nb, kDensThreads, 0, st>>>(a);
}

}  // namespace gpk
