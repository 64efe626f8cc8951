// adam.cu — fused Adam step over all N primitives (adam_step, optimize.hpp:195-221).
//
// One thread per 4 consecutive primitives walks the 11 parameter planes with
// 16 B accesses: read p, g, m, v and write p, m, v (308 B/primitive: the HBM
// roofline of the kernel). Order of
// the reference is kept: position update then bbox clamp (:212), log-scale,
// quaternion update then renormalisation when the norm is > 0 (:216-217),
// raw alpha. The step counter lives on the device; bias corrections and the
// lr_at schedule (optimize.hpp:71-73) are evaluated once per CTA in fp64, so
// a whole training step can be captured in a CUDA graph.
#include "adam.cuh"

#ifndef ADAM_ITEMS
#define ADAM_ITEMS 4
#endif

namespace gpk {

namespace {

constexpr int kAdamItems = ADAM_ITEMS;  // consecutive primitives per thread (one vector access per plane)

__global__ void __launch_bounds__(256) k_adam(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ AdamConsts s_c;
    if (a.ctrl && a.ctrl->pair_overflow) return;
    if (threadIdx.x == 0) adam_consts(a, s_c);
    __syncthreads();
    const AdamConsts c = s_c;
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * kAdamItems;
    if (i0 < a.n) {  // the capacity is a multiple of 512: vector accesses stay in the plane
        Pack<kAdamItems> p[11];
        unsigned nz;
        adam_update<kAdamItems>(a, c, i0, p, nz);
        adam_store<kAdamItems>(a, i0, p);
    }
    adam_finish(a);
}

}  // namespace

void launch_adam(const AdamLaunch& a, cudaStream_t st) {
    const unsigned grid = (a.n + 256 * kAdamItems - 1) / (256 * kAdamItems);
    if (grid) launch_pdl(k_adam, dim3(grid), dim3(256), 0, st, a);
}

}  // namespace gpk
