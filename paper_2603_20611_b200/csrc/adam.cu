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
#include "common.cuh"

namespace gpk {

namespace {

constexpr int kAdamItems = 4;  // consecutive primitives per thread: 16 B per plane access

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

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
    // lr * (m / bc1) / (sqrt(v / bc2) + eps) with the bias corrections folded
    // into per-CTA constants: lr/bc1 * m / (sqrt(v) / sqrt(bc2) + eps); sqrt and
    // the division on MUFU (relative error ~1e-7, far inside the fp32 budget)
    const float ibc1 = 1.f / s_c[0], isbc2 = 1.f / sqrtf(s_c[1]), eps = s_c[6];
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * kAdamItems;
    if (i0 < a.n) {
        // one plane, 4 primitives: moments and the bias-corrected step (the
        // reference's operation order, optimize.hpp:184-189); the capacity is a
        // multiple of 512, so the 16 B accesses never leave the plane
        auto update = [&](int k, float lr) -> float4 {
            const uint64_t o = (uint64_t)k * a.cap + i0;
            const float4 g = __ldcs(reinterpret_cast<const float4*>(a.grads + o));
            float4 m = ld4(a.m + o), v = ld4(a.v + o), p = ld4(a.params + o);
            m.x = b1 * m.x + ib1 * g.x;
            m.y = b1 * m.y + ib1 * g.y;
            m.z = b1 * m.z + ib1 * g.z;
            m.w = b1 * m.w + ib1 * g.w;
            v.x = b2 * v.x + ib2 * g.x * g.x;
            v.y = b2 * v.y + ib2 * g.y * g.y;
            v.z = b2 * v.z + ib2 * g.z * g.z;
            v.w = b2 * v.w + ib2 * g.w * g.w;
            st4(a.m + o, m);
            st4(a.v + o, v);
            const float lrc = lr * ibc1;
            auto step = [&](float mm, float vv) {
                const float sq = vv > 0.f ? vv * rsqrtf(vv) : 0.f;
                return __fdividef(lrc * mm, fmaf(sq, isbc2, eps));
            };
            p.x -= step(m.x, v.x);
            p.y -= step(m.y, v.y);
            p.z -= step(m.z, v.z);
            p.w -= step(m.w, v.w);
            return p;
        };
        // position, then the bbox clamp (optimize.hpp:212)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            float4 p = update(d, s_c[2]);
            const float lo = a.bbox_min[d], hi = a.bbox_max[d];
            p.x = fminf(hi, fmaxf(lo, p.x));
            p.y = fminf(hi, fmaxf(lo, p.y));
            p.z = fminf(hi, fmaxf(lo, p.z));
            p.w = fminf(hi, fmaxf(lo, p.w));
            st4(a.params + (uint64_t)d * a.cap + i0, p);
        }
        // log-scale, raw alpha
#pragma unroll
        for (int d = 3; d < 6; ++d) st4(a.params + (uint64_t)d * a.cap + i0, update(d, s_c[4]));
        st4(a.params + 10ull * a.cap + i0, update(10, s_c[3]));
        // quaternion, then renormalisation when the norm is > 0 (optimize.hpp:216-217)
        float4 q[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) q[d] = update(6 + d, s_c[5]);
        float* qs[4] = {&q[0].x, &q[1].x, &q[2].x, &q[3].x};
#pragma unroll
        for (int l = 0; l < kAdamItems; ++l) {
            const float w = qs[0][l], x = qs[1][l], y = qs[2][l], z = qs[3][l];
            const float qn = sqrtf(w * w + x * x + y * y + z * z);
            if (qn > 0.f) {
                const float inv = 1.f / qn;
#pragma unroll
                for (int d = 0; d < 4; ++d) qs[d][l] *= inv;
            }
        }
#pragma unroll
        for (int d = 0; d < 4; ++d) st4(a.params + (uint64_t)(6 + d) * a.cap + i0, q[d]);
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
    const unsigned grid = (a.n + 256 * kAdamItems - 1) / (256 * kAdamItems);
    if (grid) launch_pdl(k_adam, dim3(grid), dim3(256), 0, st, a);
}

}  // namespace gpk
