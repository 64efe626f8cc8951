// adam.cu — fused Adam step over all N primitives (adam_step, optimize.hpp:195-221).
//
// One thread per primitive walks its 11 parameter planes: read p, g, m, v and
// write p, m, v (308 B/primitive: the HBM roofline of the kernel). Order of
// the reference is kept: position update then bbox clamp (:212), log-scale,
// quaternion update then renormalisation when the norm is > 0 (:216-217),
// raw alpha. The step counter lives on the device; bias corrections and the
// lr_at schedule (optimize.hpp:71-73) are evaluated once per CTA in fp64, so
// a whole training step can be captured in a CUDA graph.
#include "common.cuh"

namespace gpk {

namespace {

__global__ void __launch_bounds__(256) k_adam(const AdamLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ float s_c[7];  // bc1, bc2, lr pos, lr opacity, lr scale, lr rot, eps
    if (a.ctrl && a.ctrl->pair_overflow) return;
    if (threadIdx.x == 0) {
        const long long step = *a.step + 1;
        const double bc1 = 1.0 - pow(a.beta1, (double)step);
        const double bc2 = 1.0 - pow(a.beta2, (double)step);
        double f = 1.0;
        if (a.scheduled) f = pow(0.1, (double)(step - 1) / (double)a.total);
        s_c[0] = (float)bc1;
        s_c[1] = (float)bc2;
        for (int k = 0; k < 4; ++k) s_c[2 + k] = (float)(a.lr[k] * f);
        s_c[6] = (float)a.eps;
    }
    __syncthreads();
    const float b1 = (float)a.beta1, b2 = (float)a.beta2;
    const float ib1 = (float)(1.0 - a.beta1), ib2 = (float)(1.0 - a.beta2);
    const float bc1 = s_c[0], bc2 = s_c[1], eps = s_c[6];
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n) {
        float p[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const uint64_t o = (uint64_t)k * a.cap + i;
            const float g = a.grads[o];
            float m = a.m[o], v = a.v[o];
            m = b1 * m + ib1 * g;
            v = b2 * v + ib2 * g * g;
            a.m[o] = m;
            a.v[o] = v;
            const float lr = k < 3 ? s_c[2] : (k < 6 ? s_c[4] : (k < 10 ? s_c[5] : s_c[3]));
            p[k] = a.params[o] - lr * (m / bc1) / (sqrtf(v / bc2) + eps);
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) p[d] = fminf(a.bbox_max[d], fmaxf(a.bbox_min[d], p[d]));
        const float qn = sqrtf(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
        if (qn > 0.f) {
            const float inv = 1.f / qn;
#pragma unroll
            for (int d = 6; d < 10; ++d) p[d] *= inv;
        }
#pragma unroll
        for (int k = 0; k < 11; ++k) a.params[(uint64_t)k * a.cap + i] = p[k];
    }
    // last CTA out advances AdamState::step
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(a.done_ctr, 1u);
        if (done == gridDim.x - 1) {
            *a.step += 1;
            *a.done_ctr = 0;
        }
    }
}

}  // namespace

void launch_adam(const AdamLaunch& a, cudaStream_t st) {
    const unsigned grid = (a.n + 255) / 256;
    if (grid) launch_pdl(k_adam, dim3(grid), dim3(256), 0, st, a);
}

}  // namespace gpk
