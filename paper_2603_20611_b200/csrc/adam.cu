// adam.cu — fused Adam step over all N primitives (adam_step, optimize.hpp:195-221).
//
// k_adam_consts (one warp) evaluates the step's bias corrections and the lr_at
// schedule (optimize.hpp:71-73) in fp64 from the device step counter (the
// training step runs it on a side stream, off the critical path); the update
// kernel advances the counter, so a whole training step can be captured in a
// CUDA graph and the update kernel needs no CTA barrier. k_adam: each thread walks the 11
// parameter planes of 2 consecutive primitives with 8 B accesses, storing each
// plane as soon as it is final (few live registers: 6 CTAs per SM keep enough
// requests in flight). Bytes: read p, g, m, v and write p, m, v = 308 B per
// primitive; in slot-gradient mode (the training step, see AdamLaunch) the
// gradient comes from the survivors' slots: 266 B per primitive + 44 B per
// survivor. The reference's order is kept: position update then bbox clamp
// (:212), log-scale, raw alpha, quaternion update then renormalisation when
// the norm is > 0 (:216-217).
#include <algorithm>
#include <cmath>

#include <cstdlib>

#include "adam.cuh"

namespace gpk {

namespace {

constexpr int kAdamItems = 2;

__global__ void k_adam_consts(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    AdamConsts c;
    adam_consts(a, c);
    const int lane = threadIdx.x & 31;
    AdamConsts* ring = a.lazy.ring;  // lazy training steps only (else nullptr)
    if (ring) {
        // LazyAdam drift bound of this step: |delta p| = lr/bc1 |m| / (sqrt(v/bc2) + eps)
        // <= lr (|m| / sqrt(v)) sqrt(bc2) / bc1 <= lr 1.03 K sqrt(bc2) / bc1, and
        // lr/bc1 1e-18 / eps when v underflowed (lazy_state_ok's absolute term)
        const double b1 = a.beta1, b2 = a.beta2, eps = a.eps;
        const double gam = b1 * b1 / b2;
        const double K = (b1 >= 0.0 && b1 < 1.0 && b2 > 0.0 && b2 < 1.0 && gam < 1.0)
                             ? (1.0 - b1) / sqrt((1.0 - b2) * (1.0 - gam)) : (double)INFINITY;
        const double bc1 = 1.0 / (double)c.ibc1, bc2 = 1.0 / ((double)c.isbc2 * (double)c.isbc2);
        const double B = 1.03 * K * sqrt(bc2) / bc1 + (eps > 0.0 ? 1e-18 / (bc1 * eps) : (double)INFINITY);
        c.kratio = (float)(1.02 * K);
        // lane j (1 .. kLazyWindow - 2) holds step - j's entry, the warp sums
        const long long sj = c.step - lane;
        const bool use = lane >= 1 && lane <= kLazyWindow - 2 && sj >= 1;
        const AdamConsts* e = use ? &ring[sj % kLazyRing] : nullptr;
        const bool ok = !use || e->step == sj;
        for (int k = 0; k < 4; ++k) {
            c.drift[k] = (float)((double)c.lr[k] * B * 1.0001);
            double d = lane == 0 ? (double)c.drift[k] : use ? (ok ? (double)e->drift[k] : (double)INFINITY) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            c.cum[k] = (float)(d * 1.0001);
        }
    }
    if (lane != 0) return;
    *a.consts = c;
    if (ring) ring[c.step % kLazyRing] = c;
}

// (plain: 6 CTAs/SM, 40 registers; 7-8 CTAs/SM spill and measured slower.
// Pipelined: 5 CTAs/SM, two planes of loads in flight per thread)
template <bool kSlots, int kMinB, bool kPipe = false>
__global__ void __launch_bounds__(256, kMinB) k_adam(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const uint32_t i0 = a.lo + (blockIdx.x * blockDim.x + threadIdx.x) * kAdamItems;
    if (i0 >= a.n) return;  // the capacity is a multiple of 512: vector accesses stay in the plane
    bool overflow = a.ctrl && a.ctrl->pair_overflow;  // a slice overflowed: no update
    for (int s = 0; s < a.nsrc; ++s) overflow |= a.src_ctrl[s]->pair_overflow != 0;  // (batched step)
    if (a.uctrl) overflow |= a.uctrl[1] != 0;  // (data-parallel union rows beyond the capacity)
    if (overflow) {
        if (kSlots && !a.umap) adam_slots_clear<kAdamItems>(a, i0);
        return;
    }
    // read in place (L1) where used: the constants would otherwise hold 12
    // registers for the whole kernel
    const AdamConsts& c = *a.consts;
    adam_advance_step(a, c);
    uint32_t gslot[kAdamItems];
    const bool any = kSlots && adam_slots<kAdamItems>(a, i0, gslot);
    if (kPipe)
        adam_update_store_pipe<kAdamItems>(a, c, i0,
                                           [&](int k) { return adam_grad<kAdamItems>(a, k, i0, kSlots ? gslot : nullptr); });
    else
        adam_update_store<kAdamItems>(a, c, i0, kSlots ? gslot : nullptr);
    if (any) adam_slots_clear<kAdamItems>(a, i0);
}

// ---- Adam split around the render (single-GPU training step) ---------------------
// A Gaussian that did not survive the slice's cull has an exactly zero
// gradient, known as soon as K_decide has run; its update does not depend on
// the render. k_adam_rest updates them on a side stream while the slice
// renders (grid-stride, a bounded number of CTAs, launched at the lowest
// priority so the latency-bound slice kernels keep the SMs), k_adam_final
// the survivors from their slot gradients after the chain. Per Gaussian the
// same operations as k_adam: the same bits.
__device__ __forceinline__ bool adam_overflow(const AdamLaunch& a) { return a.ctrl && a.ctrl->pair_overflow; }

__global__ void __launch_bounds__(256, 6) k_adam_rest(const AdamLaunch a, const unsigned* __restrict__ surv_bits) {
    if (adam_overflow(a)) return;
    const AdamConsts& c = *a.consts;
    const auto zero2 = [](int) { Pack<2> g; g.v[0] = g.v[1] = 0.f; return g; };
    const auto zero1 = [](int) { Pack<1> g; g.v[0] = 0.f; return g; };
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 2; i0 < a.n; i0 += gridDim.x * blockDim.x * 2) {
        const unsigned bits = (__ldg(&surv_bits[i0 >> 5]) >> (i0 & 31)) & 3u;  // i0 even: one word
        if (bits == 0) {
            adam_update_store_g<2>(a, c, i0, zero2);
        } else if (bits != 3) {
            adam_update_store_g<1>(a, c, i0 + (bits == 1 ? 1u : 0u), zero1);
        }
    }
}

// CTA per K_decide group: its survivors (slots g*4096 + [0, S_g)); CTA 0
// advances the step counter; the chain's map entries are cleared.
__global__ void __launch_bounds__(256) k_adam_final(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned g = blockIdx.x;
    const unsigned S = a.grp_surv[g];
    const bool skip = adam_overflow(a);
    const AdamConsts& c = *a.consts;
    if (!skip) adam_advance_step(a, c);
    for (unsigned j = threadIdx.x; j < S; j += blockDim.x) {
        const uint32_t slot = g * kDecideGroupSize + j, i = a.surv_gidx[slot];
        if (!skip)
            adam_update_store_g<1>(a, c, i, [&](int k) {
                Pack<1> gr;
                gr.v[0] = __ldcs(a.slot_grads + (uint64_t)k * a.cap + slot);
                return gr;
            });
        a.gmap[i] = 0;
    }
}

// ---- lazy training steps (LazyAdam, common.cuh) ----------------------------------
__device__ __forceinline__ void lazy_load(const AdamLaunch& a, uint32_t i, float p[11], float m[11], float v[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        const uint64_t o = (uint64_t)k * a.cap + i;
        p[k] = a.params[o];
        m[k] = a.m[o];
        v[k] = a.v[o];
    }
}
__device__ __forceinline__ void lazy_store(const AdamLaunch& a, uint32_t i, const float p[11], const float m[11],
                                           const float v[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        const uint64_t o = (uint64_t)k * a.cap + i;
        a.params[o] = p[k];
        a.m[o] = m[k];
        a.v[o] = v[k];
    }
}

// The survivors of the step (CTA per K_decide group, as k_adam_final): pending
// zero-gradient steps replayed, then this step with the slot gradient; the map
// entries cleared; CTA 0 advances the step counter.
__global__ void __launch_bounds__(256) k_lazy_survivors(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned g = blockIdx.x;
    const unsigned S = a.grp_surv[g];
    const bool skip = adam_overflow(a);
    const AdamConsts& c = *a.consts;
    const long long t = c.step;
    if (!skip) adam_advance_step(a, c);
    bool ok = true;
    for (unsigned j = threadIdx.x; j < S; j += blockDim.x) {
        const uint32_t slot = g * kDecideGroupSize + j, i = a.surv_gidx[slot];
        if (!skip) {
            float p[11], m[11], v[11], gr[11];
            lazy_load(a, i, p, m, v);
            lazy_replay(a.lazy, (long long)a.lazy.t_done[i] + 1, t - 1, p, m, v);
#pragma unroll
            for (int k = 0; k < 11; ++k) gr[k] = __ldcs(a.slot_grads + (uint64_t)k * a.cap + slot);
            adam_gauss_step(c, a.bbox_min, a.bbox_max, p, m, v, gr);
            lazy_store(a, i, p, m, v);
            a.lazy.t_done[i] = (uint32_t)t;
            ok &= lazy_state_ok(c.kratio, m, v);
        }
        a.gmap[i] = 0;
    }
    if (!ok) atomicOr(a.lazy.bad, 1u);
}

// The step's window: Gaussians [w W, (w + 1) W), w = step mod kLazyWindow,
// brought up to date through this step (survivors were, by k_lazy_survivors).
__global__ void __launch_bounds__(256) k_lazy_window(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    if (adam_overflow(a)) return;
    const AdamConsts& c = *a.consts;
    const long long t = c.step;
    const uint32_t W = (uint32_t)(((uint64_t)a.n + kLazyWindow - 1) / kLazyWindow);
    const uint32_t lo = (uint32_t)(t % kLazyWindow) * W;
    const uint32_t hi = min(a.n, lo + W);
    bool ok = true;
    for (uint32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
        const long long td = a.lazy.t_done[i];
        if (td >= t) continue;
        float p[11], m[11], v[11];
        lazy_load(a, i, p, m, v);
        lazy_replay(a.lazy, td + 1, t, p, m, v);
        lazy_store(a, i, p, m, v);
        a.lazy.t_done[i] = (uint32_t)t;
        ok &= lazy_state_ok(c.kratio, m, v);
    }
    if (!ok) atomicOr(a.lazy.bad, 1u);
}

// Every Gaussian up to date through AdamState::step (before anything reads or
// writes the parameters or moments directly).
__global__ void __launch_bounds__(256) k_lazy_flush(const AdamLaunch a) {
    const long long t = *a.lazy.step;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const long long td = a.lazy.t_done[i];
        if (td >= t) continue;
        float p[11], m[11], v[11];
        lazy_load(a, i, p, m, v);
        lazy_replay(a.lazy, td + 1, t, p, m, v);
        lazy_store(a, i, p, m, v);
        a.lazy.t_done[i] = (uint32_t)t;
    }
}

// Lazy mode starts from current values: t_done = step for every Gaussian, and
// every moment state checked against the drift bound (kratio from the host:
// the training step's betas).
__global__ void __launch_bounds__(256) k_lazy_begin(const AdamLaunch a, float kratio) {
    const long long t = *a.lazy.step;
    bool ok = true;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        a.lazy.t_done[i] = (uint32_t)t;
        float m[11], v[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            m[k] = a.m[(uint64_t)k * a.cap + i];
            v[k] = a.v[(uint64_t)k * a.cap + i];
        }
        ok &= lazy_state_ok(kratio, m, v);
    }
    if (!ok) atomicOr(a.lazy.bad, 1u);
}

// Batched step, before its Adam: the B slices' slot gradients summed per
// primitive in slice order into the dense planes — every entry written (zero
// where no slice kept the primitive), every map read cleared. The dense Adam
// (k_adam) then updates from them: the sum is formed once, in a streaming
// pass, instead of B scattered reads per plane inside the latency-bound update.
__global__ void __launch_bounds__(256) k_sum_slots(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * kAdamItems;
    if (i0 >= a.n) return;
    unsigned pm[kMaxBatch];
    const bool any = adam_slots_multi(a, i0, pm);
    if (!any) {
#pragma unroll
        for (int k = 0; k < 11; ++k) stp<kAdamItems>(a.grads + (uint64_t)k * a.cap + i0, Pack<kAdamItems>{});
        return;
    }
#pragma unroll
    for (int k = 0; k < 11; ++k) stp<kAdamItems>(a.grads + (uint64_t)k * a.cap + i0, adam_grad_multi(a, k, i0, pm));
    adam_slots_multi_clear(a, i0, pm);
}

// Slot gradients -> dense planes, by survivor slot (CTA per K_decide group):
// kScatterSet writes a survivor's gradient, kScatterAdd adds it (a batched
// step's slices, one launch per slice in slice order: the same fp32 sums as
// its Adam), kScatterClearMap zeroes the survivor's map entry (a slot
// backward no Adam consumed).
__global__ void __launch_bounds__(256) k_scatter_slots(const AdamLaunch a, int mode) {
    const unsigned g = blockIdx.x;
    const unsigned S = a.grp_surv[g];
    for (unsigned j = threadIdx.x; j < S; j += blockDim.x) {
        const uint32_t slot = g * kDecideGroupSize + j, i = a.surv_gidx[slot];
        if (mode & (kScatterSet | kScatterAdd))
#pragma unroll
            for (int k = 0; k < 11; ++k) {
                float* d = a.grads + (uint64_t)k * a.cap + i;
                const float v = a.slot_grads[(uint64_t)k * a.cap + slot];
                *d = (mode & kScatterAdd) ? __fadd_rn(*d, v) : v;
            }
        if (mode & kScatterClearMap) a.gmap[i] = 0;
    }
}

}  // namespace

void launch_scatter_slot_grads(const AdamLaunch& a, unsigned ngroups, int mode, cudaStream_t st) {
    if (ngroups) k_scatter_slots<<<ngroups, 256, 0, st>>>(a, mode);
}

void launch_sum_slots(const AdamLaunch& a, cudaStream_t st) {
    const unsigned grid = (a.n + 256 * kAdamItems - 1) / (256 * kAdamItems);
    if (grid) launch_pdl(k_sum_slots, dim3(grid), dim3(256), 0, st, a);
}

void launch_adam_rest(const AdamLaunch& a, const unsigned* surv_bits, int ctas, cudaStream_t st) {
    const unsigned need = (a.n + 511) / 512;
    const unsigned grid = ctas > 0 ? std::min<unsigned>((unsigned)ctas, need) : need;
    if (grid) k_adam_rest<<<grid, 256, 0, st>>>(a, surv_bits);
}

void launch_adam_final(const AdamLaunch& a, unsigned ngroups, cudaStream_t st) {
    if (ngroups) launch_pdl(k_adam_final, dim3(ngroups), dim3(256), 0, st, a);
}

void launch_lazy_survivors(const AdamLaunch& a, unsigned ngroups, cudaStream_t st) {
    if (ngroups) launch_pdl(k_lazy_survivors, dim3(ngroups), dim3(256), 0, st, a);
}

void launch_lazy_window(const AdamLaunch& a, cudaStream_t st) {
    const uint32_t W = (uint32_t)(((uint64_t)a.n + kLazyWindow - 1) / kLazyWindow);
    if (W) launch_pdl(k_lazy_window, dim3((W + 255) / 256), dim3(256), 0, st, a);
}

void launch_lazy_flush(const AdamLaunch& a, cudaStream_t st) {
    if (a.n) k_lazy_flush<<<(a.n + 255) / 256, 256, 0, st>>>(a);
}

void launch_lazy_begin(const AdamLaunch& a, cudaStream_t st) {
    const double b1 = a.beta1, b2 = a.beta2, gam = b1 * b1 / b2;
    const double K = (b1 >= 0.0 && b1 < 1.0 && b2 > 0.0 && b2 < 1.0 && gam < 1.0)
                         ? (1.0 - b1) / std::sqrt((1.0 - b2) * (1.0 - gam)) : HUGE_VAL;
    if (a.n) k_lazy_begin<<<(a.n + 255) / 256, 256, 0, st>>>(a, (float)(1.02 * K));
}

void launch_adam_consts(const AdamLaunch& a, cudaStream_t st) {
    launch_pdl(k_adam_consts, dim3(1), dim3(32), 0, st, a);
}

void launch_adam(const AdamLaunch& a, cudaStream_t st) {
    // 2 primitives per thread, registers capped for 6 CTAs per SM: measured
    // best on B200 among 1/2/4 items per thread, persistent grid or not
    const unsigned grid = (a.n - a.lo + 256 * kAdamItems - 1) / (256 * kAdamItems);
    if (!grid || a.n <= a.lo) return;
    // software-pipelined at 5 CTAs/SM (measured: 46.9 -> 43.0 us at C2, 95 %
    // of the copy peak); GPK_ADAM_PIPE=0 selects the one-plane-at-a-time form
    static const int pipe = [] {
        const char* e = getenv("GPK_ADAM_PIPE");
        return e ? atoi(e) : 1;
    }();
    if (pipe) {
        if (a.slot_grads) launch_pdl(k_adam<true, 5, true>, dim3(grid), dim3(256), 0, st, a);
        else launch_pdl(k_adam<false, 5, true>, dim3(grid), dim3(256), 0, st, a);
    } else {
        if (a.slot_grads) launch_pdl(k_adam<true, 6>, dim3(grid), dim3(256), 0, st, a);
        else launch_pdl(k_adam<false, 6>, dim3(grid), dim3(256), 0, st, a);
    }
}

}  // namespace gpk
