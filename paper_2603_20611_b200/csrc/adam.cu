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

#include "adam.cuh"

namespace gpk {

namespace {

constexpr int kAdamItems = 2;

__global__ void k_adam_consts(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    AdamConsts c;
    adam_consts(a, c);
    if (threadIdx.x == 0) *a.consts = c;
}

// (6 CTAs/SM: 40 registers; 7-8 CTAs/SM spill and measured slower)
template <bool kSlots, int kMinB>
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

void launch_adam_consts(const AdamLaunch& a, cudaStream_t st) {
    launch_pdl(k_adam_consts, dim3(1), dim3(32), 0, st, a);
}

void launch_adam(const AdamLaunch& a, cudaStream_t st) {
    // 2 primitives per thread, registers capped for 6 CTAs per SM: measured
    // best on B200 among 1/2/4 items per thread, persistent grid or not
    const unsigned grid = (a.n - a.lo + 256 * kAdamItems - 1) / (256 * kAdamItems);
    if (!grid || a.n <= a.lo) return;
    if (a.slot_grads) launch_pdl(k_adam<true, 6>, dim3(grid), dim3(256), 0, st, a);
    else launch_pdl(k_adam<false, 6>, dim3(grid), dim3(256), 0, st, a);
}

}  // namespace gpk
