// adam.cuh — the Adam update of adam_step (optimize.hpp:184-221), shared by the
// stand-alone Adam kernel (adam.cu) and the training step's Adam + next-slice
// cull kernel (prep.cu). Every operation is an explicit round-to-nearest
// intrinsic, so both translation units (prep.cu is built with --fmad=false)
// produce the same bits. A thread updates N consecutive primitives with one
// N*4-byte access per plane and array.
#pragma once

#include "common.cuh"

namespace gpk {

// Per-step constants, evaluated once by k_adam_consts (fp64, then f32): bias
// corrections of step+1 and the lr_at schedule (optimize.hpp:71-73).
// Whole warp: lanes 0-2 evaluate the three fp64 powers side by side (one pow
// latency instead of three); the result is complete in lane 0.
__device__ __forceinline__ void adam_consts(const AdamLaunch& a, AdamConsts& c) {
    const int lane = threadIdx.x & 31;
    const long long step = *a.step + 1;
    const double base = lane == 0 ? a.beta1 : lane == 1 ? a.beta2 : 0.1;
    const double ex = lane == 2 ? (double)(step - 1) / (double)a.total : (double)step;
    const double pw = lane < 3 ? pow(base, ex) : 1.0;
    const double bc1 = 1.0 - __shfl_sync(0xffffffffu, pw, 0);
    const double bc2 = 1.0 - __shfl_sync(0xffffffffu, pw, 1);
    const double f = a.scheduled ? __shfl_sync(0xffffffffu, pw, 2) : 1.0;
    c.b1 = (float)a.beta1;
    c.b2 = (float)a.beta2;
    c.ib1 = (float)(1.0 - a.beta1);
    c.ib2 = (float)(1.0 - a.beta2);
    c.ibc1 = __frcp_rn((float)bc1);
    c.isbc2 = __frcp_rn(__fsqrt_rn((float)bc2));
    c.eps = (float)a.eps;
    for (int k = 0; k < 4; ++k) c.lr[k] = (float)(a.lr[k] * f);
    c.step = step;
}

// The update kernels' CTA 0 advances AdamState::step (no other CTA reads it;
// the next step's k_adam_consts runs after this kernel).
__device__ __forceinline__ void adam_advance_step(const AdamLaunch& a, const AdamConsts& c) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.step = c.step;
}

// N consecutive floats moved with one vector access.
template <int N>
struct Pack {
    float v[N];
};
template <int N>
__device__ __forceinline__ Pack<N> ldp(const float* p) {
    Pack<N> r;
    if constexpr (N == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else if constexpr (N == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        r.v[0] = t.x, r.v[1] = t.y;
    } else {
        r.v[0] = *p;
    }
    return r;
}
template <int N>
__device__ __forceinline__ Pack<N> ldp_stream(const float* p) {
    Pack<N> r;
    if constexpr (N == 4) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
        r.v[0] = t.x, r.v[1] = t.y, r.v[2] = t.z, r.v[3] = t.w;
    } else if constexpr (N == 2) {
        const float2 t = __ldcs(reinterpret_cast<const float2*>(p));
        r.v[0] = t.x, r.v[1] = t.y;
    } else {
        r.v[0] = __ldcs(p);
    }
    return r;
}
template <int N>
__device__ __forceinline__ void stp_stream(float* p, const Pack<N>& r) {
    if constexpr (N == 4)
        __stcs(reinterpret_cast<float4*>(p), make_float4(r.v[0], r.v[1], r.v[2], r.v[3]));
    else if constexpr (N == 2)
        __stcs(reinterpret_cast<float2*>(p), make_float2(r.v[0], r.v[1]));
    else
        __stcs(p, r.v[0]);
}
template <int N>
__device__ __forceinline__ void stp(float* p, const Pack<N>& r) {
    if constexpr (N == 4)
        *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    else if constexpr (N == 2)
        *reinterpret_cast<float2*>(p) = make_float2(r.v[0], r.v[1]);
    else
        *p = r.v[0];
}

// lr * (m / bc1) / (sqrt(v / bc2) + eps), bias corrections folded into the
// constants; sqrt and the division on MUFU (relative error ~1e-7).
__device__ __forceinline__ float adam_delta(const AdamConsts& c, float lrc, float m, float v) {
    const float sq = v > 0.f ? __fmul_rn(v, rsqrtf(v)) : 0.f;
    return __fdividef(__fmul_rn(lrc, m), __fmaf_rn(sq, c.isbc2, c.eps));
}

// One parameter's update (optimize.hpp:184-188): the moments, then the step.
// Every Adam path (eager, lazy, replay) goes through this: the same bits.
__device__ __forceinline__ void adam_elem(const AdamConsts& c, float lrc, float& p, float& m, float& v, float g) {
    m = __fmaf_rn(c.b1, m, __fmul_rn(c.ib1, g));
    v = __fmaf_rn(c.b2, v, __fmul_rn(__fmul_rn(c.ib2, g), g));
    p = __fsub_rn(p, adam_delta(c, lrc, m, v));
}

// The reference's quaternion renormalisation (optimize.hpp:216-217).
__device__ __forceinline__ void adam_renorm(float& w, float& x, float& y, float& z) {
    const float qn = __fsqrt_rn(__fmaf_rn(w, w, __fmaf_rn(x, x, __fmaf_rn(y, y, __fmul_rn(z, z)))));
    if (qn > 0.f) {
        const float inv = __frcp_rn(qn);
        w = __fmul_rn(w, inv);
        x = __fmul_rn(x, inv);
        y = __fmul_rn(y, inv);
        z = __fmul_rn(z, inv);
    }
}

// One whole Adam step of one Gaussian held in registers (planes in the
// reference's order, the bbox clamp after the position, the renormalisation
// after the quaternion): the per-Gaussian form of adam_update_store_g.
__device__ __forceinline__ void adam_gauss_step(const AdamConsts& c, const float bmin[3], const float bmax[3],
                                                float p[11], float m[11], float v[11], const float g[11]) {
    const float l0 = __fmul_rn(c.lr[0], c.ibc1), l1 = __fmul_rn(c.lr[1], c.ibc1);
    const float l2 = __fmul_rn(c.lr[2], c.ibc1), l3 = __fmul_rn(c.lr[3], c.ibc1);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        adam_elem(c, l0, p[d], m[d], v[d], g[d]);
        p[d] = fminf(bmax[d], fmaxf(bmin[d], p[d]));
    }
#pragma unroll
    for (int d = 3; d < 6; ++d) adam_elem(c, l2, p[d], m[d], v[d], g[d]);
    adam_elem(c, l1, p[10], m[10], v[10], g[10]);
#pragma unroll
    for (int d = 6; d < 10; ++d) adam_elem(c, l3, p[d], m[d], v[d], g[d]);
    adam_renorm(p[6], p[7], p[8], p[9]);
}

// A zero the compiler cannot see through (the eager path's zero gradients are
// loaded values: no constant folding may change a rounding or a sign here).
__device__ __forceinline__ float opaque_zero() {
    float z;
    asm volatile("mov.b32 %0, 0;" : "=f"(z));
    return z;
}

// Replays the zero-gradient steps from .. to (inclusive) of one Gaussian
// (LazyAdam): constants from the ring, the eager operations in the eager order.
__device__ __forceinline__ void lazy_replay(const LazyAdam& L, long long from, long long to, float p[11], float m[11],
                                            float v[11]) {
    if (from > to) return;
    float g[11];
    const float z = opaque_zero();
#pragma unroll
    for (int k = 0; k < 11; ++k) g[k] = z;
    for (long long s = from; s <= to; ++s) adam_gauss_step(L.ring[s % kLazyRing], L.bbox_min, L.bbox_max, p, m, v, g);
}

// The moment-state bound the lazy drift assumes (|m| <= kratio sqrt(v) per
// parameter, + 1e-18 for flushed denormals): false (NaN included) flags the
// state as outside it.
__device__ __forceinline__ bool lazy_state_ok(float kratio, const float m[11], const float v[11]) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 11; ++k) ok &= fabsf(m[k]) <= __fmaf_rn(kratio, sqrtf(fmaxf(v[k], 0.f)), 1e-18f);
    return ok;
}

// Where a thread's N gradients come from: the dense planes at i0 (gslot ==
// nullptr), or per primitive a survivor slot (kNoSlot: zero gradient).
constexpr uint32_t kNoSlot = 0xffffffffu;

template <int N>
__device__ __forceinline__ Pack<N> adam_grad(const AdamLaunch& a, int k, uint32_t i0, const uint32_t* gslot) {
    if (!gslot) return ldp_stream<N>(a.grads + (uint64_t)k * a.cap + i0);
    Pack<N> g;
#pragma unroll
    for (int l = 0; l < N; ++l)
        g.v[l] = gslot[l] != kNoSlot ? __ldcs(a.slot_grads + (uint64_t)k * a.cap + gslot[l]) : 0.f;
    return g;
}

// Slot-gradient mode (AdamLaunch::slot_grads): the survivor slots of primitives
// i0 .. i0+N-1 from the chain's map (1 + offset within the K_decide group, 0
// for a non-survivor). Returns whether any is a survivor: the caller then
// clears those map entries (adam_slots_clear) so the map is zero again.
template <int N>
__device__ __forceinline__ bool adam_slots(const AdamLaunch& a, uint32_t i0, uint32_t gslot[N]) {
    if (a.umap) {  // data-parallel union rows: the map is rebuilt every step, never cleared
        bool any = false;
#pragma unroll
        for (int l = 0; l < N; ++l) {
            const uint32_t m = a.umap[i0 + l];
            gslot[l] = m ? m - 1 : kNoSlot;
            any |= m != 0;
        }
        (void)any;
        return false;  // nothing to clear
    }
    uint16_t m[N];
    if constexpr (N == 4) {
        const uint2 t = *reinterpret_cast<const uint2*>(a.gmap + i0);
        m[0] = (uint16_t)(t.x & 0xffffu), m[1] = (uint16_t)(t.x >> 16), m[2] = (uint16_t)(t.y & 0xffffu),
        m[3] = (uint16_t)(t.y >> 16);
    } else if constexpr (N == 2) {
        const unsigned t = *reinterpret_cast<const unsigned*>(a.gmap + i0);
        m[0] = (uint16_t)(t & 0xffffu), m[1] = (uint16_t)(t >> 16);
    } else {
        m[0] = a.gmap[i0];
    }
    const uint32_t gbase = i0 / kDecideGroupSize * kDecideGroupSize;  // N divides the group size
    bool any = false;
#pragma unroll
    for (int l = 0; l < N; ++l) {
        gslot[l] = m[l] ? gbase + m[l] - 1 : kNoSlot;
        any |= m[l] != 0;
    }
    return any;
}
template <int N>
__device__ __forceinline__ void adam_slots_clear(const AdamLaunch& a, uint32_t i0) {
    if constexpr (N == 4) *reinterpret_cast<uint2*>(a.gmap + i0) = make_uint2(0u, 0u);
    else if constexpr (N == 2) *reinterpret_cast<unsigned*>(a.gmap + i0) = 0u;
    else a.gmap[i0] = 0;
}

// One parameter plane of N consecutive primitives: moments updated and stored,
// the stepped parameters returned (before clamp / renormalisation); nz collects
// which primitives had a non-zero gradient.
// Batched step: the B slices' map entries of primitives i0, i0 + 1 (one u32
// of two u16 per slice) and their gradient of plane k summed over the slices
// in slice order.
__device__ __forceinline__ bool adam_slots_multi(const AdamLaunch& a, uint32_t i0, unsigned pm[kMaxBatch]) {
    unsigned any = 0;
#pragma unroll
    for (int s = 0; s < kMaxBatch; ++s) {
        pm[s] = s <= a.nsrc ? *reinterpret_cast<const unsigned*>((s ? a.src_gmap[s - 1] : a.gmap) + i0) : 0u;
        any |= pm[s];
    }
    return any != 0;
}
__device__ __forceinline__ void adam_slots_multi_clear(const AdamLaunch& a, uint32_t i0, const unsigned pm[kMaxBatch]) {
#pragma unroll
    for (int s = 0; s < kMaxBatch; ++s)
        if (pm[s]) *reinterpret_cast<unsigned*>((s ? a.src_gmap[s - 1] : a.gmap) + i0) = 0u;
}
__device__ __forceinline__ Pack<2> adam_grad_multi(const AdamLaunch& a, int k, uint32_t i0, const unsigned pm[kMaxBatch]) {
    // Branch-free: every slice's value is requested at once (an absent entry
    // reads the plane's first slot and is discarded), then summed in slice
    // order exactly as the dense per-slice gradients add (absent = +0).
    const uint64_t off = (uint64_t)k * a.cap + i0 / kDecideGroupSize * kDecideGroupSize - 1;
    float x0[kMaxBatch], x1[kMaxBatch];
#pragma unroll
    for (int s = 0; s < kMaxBatch; ++s) {
        x0[s] = x1[s] = 0.f;
        if (s > a.nsrc) break;  // uniform: the batch size
        const float* base = (s ? a.src_slot[s - 1] : a.slot_grads) + off;
        const unsigned m0 = pm[s] & 0xffffu, m1 = pm[s] >> 16;
        // only the slices holding the primitive are read (a primitive is in
        // few of a step's slices: the absent ones' loads were most of the
        // kernel's issue and load-unit traffic)
        if (m0) x0[s] = __ldcs(base + m0);
        if (m1) x1[s] = __ldcs(base + m1);
    }
    Pack<2> g;
    g.v[0] = (pm[0] & 0xffffu) ? x0[0] : 0.f;
    g.v[1] = (pm[0] >> 16) ? x1[0] : 0.f;
#pragma unroll
    for (int s = 1; s < kMaxBatch; ++s) {
        if (s > a.nsrc) break;
        g.v[0] = __fadd_rn(g.v[0], (pm[s] & 0xffffu) ? x0[s] : 0.f);
        g.v[1] = __fadd_rn(g.v[1], (pm[s] >> 16) ? x1[s] : 0.f);
    }
    return g;
}

template <int N, typename G>
__device__ __forceinline__ Pack<N> adam_plane_g(const AdamLaunch& a, const AdamConsts& c, int k, float lr, uint32_t i0,
                                                const G& grad, unsigned& nz) {
    const uint64_t o = (uint64_t)k * a.cap + i0;
    // Everything evict-first: the moments must not push the parameters (which
    // K_filter left in L2 with evict-last priority for this read) out of L2,
    // and the parameter accesses here demote those lines again, so nothing of
    // this step stays resident into the next one. The streams are requested
    // before the gradient (whose source may take several dependent loads).
    Pack<N> m = ldp_stream<N>(a.m + o), v = ldp_stream<N>(a.v + o), p = ldp_stream<N>(a.params + o);
    const Pack<N> g = grad(k);
    const float lrc = __fmul_rn(lr, c.ibc1);
#pragma unroll
    for (int l = 0; l < N; ++l) {
        nz |= (g.v[l] != 0.f ? 1u : 0u) << l;
        adam_elem(c, lrc, p.v[l], m.v[l], v.v[l], g.v[l]);
    }
    stp_stream<N>(a.m + o, m);
    stp_stream<N>(a.v + o, v);
    return p;
}

template <int N>
__device__ __forceinline__ Pack<N> adam_plane(const AdamLaunch& a, const AdamConsts& c, int k, float lr, uint32_t i0,
                                              const uint32_t* gslot, unsigned& nz) {
    return adam_plane_g<N>(a, c, k, lr, i0, [&](int kk) { return adam_grad<N>(a, kk, i0, gslot); }, nz);
}

// All 11 planes of N consecutive primitives in the reference's order: position
// then the bbox clamp (optimize.hpp:212), log-scale, raw alpha, quaternion then
// renormalisation when the norm is > 0 (:216-217). p[k] returns the new
// parameters; nz the primitives with a non-zero gradient; gslot as adam_grad.
template <int N>
__device__ __forceinline__ void adam_update(const AdamLaunch& a, const AdamConsts& c, uint32_t i0,
                                            const uint32_t* gslot, Pack<N> p[11], unsigned& nz) {
    nz = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        p[d] = adam_plane<N>(a, c, d, c.lr[0], i0, gslot, nz);
        const float lo = a.bbox_min[d], hi = a.bbox_max[d];
#pragma unroll
        for (int l = 0; l < N; ++l) p[d].v[l] = fminf(hi, fmaxf(lo, p[d].v[l]));
    }
#pragma unroll
    for (int d = 3; d < 6; ++d) p[d] = adam_plane<N>(a, c, d, c.lr[2], i0, gslot, nz);
    p[10] = adam_plane<N>(a, c, 10, c.lr[1], i0, gslot, nz);
#pragma unroll
    for (int d = 6; d < 10; ++d) p[d] = adam_plane<N>(a, c, d, c.lr[3], i0, gslot, nz);
#pragma unroll
    for (int l = 0; l < N; ++l) adam_renorm(p[6].v[l], p[7].v[l], p[8].v[l], p[9].v[l]);
}

// As adam_update + adam_store, storing each plane's parameters as soon as they
// are final (all but the quaternion, renormalised at the end): few registers
// live, so the stand-alone kernel runs at full occupancy. Same bits.
// Software-pipelined form (GPK_ADAM_PIPE): the next plane's parameter,
// moments and gradient are requested before this plane's arithmetic, so two
// planes' loads are in flight per thread. The same operations in the same
// order per element: the same bits.
template <int N, typename G>
__device__ __forceinline__ void adam_update_store_pipe(const AdamLaunch& a, const AdamConsts& c, uint32_t i0,
                                                       const G& grad) {
    constexpr int kOrder[11] = {0, 1, 2, 3, 4, 5, 10, 6, 7, 8, 9};
    Pack<N> m[2], v[2], p[2], g[2], q[4];
    auto fetch = [&](int j, int b) {
        const uint64_t o = (uint64_t)kOrder[j] * a.cap + i0;
        m[b] = ldp_stream<N>(a.m + o);
        v[b] = ldp_stream<N>(a.v + o);
        p[b] = ldp_stream<N>(a.params + o);
        g[b] = grad(kOrder[j]);
    };
    fetch(0, 0);
#pragma unroll
    for (int j = 0; j < 11; ++j) {
        const int b = j & 1, k = kOrder[j];
        if (j + 1 < 11) fetch(j + 1, b ^ 1);
        const float lr = k < 3 ? c.lr[0] : (k < 6 ? c.lr[2] : (k == 10 ? c.lr[1] : c.lr[3]));
        const float lrc = __fmul_rn(lr, c.ibc1);
#pragma unroll
        for (int l = 0; l < N; ++l) adam_elem(c, lrc, p[b].v[l], m[b].v[l], v[b].v[l], g[b].v[l]);
        const uint64_t o = (uint64_t)k * a.cap + i0;
        stp_stream<N>(a.m + o, m[b]);
        stp_stream<N>(a.v + o, v[b]);
        if (k < 3) {
            const float lo = a.bbox_min[k], hi = a.bbox_max[k];
#pragma unroll
            for (int l = 0; l < N; ++l) p[b].v[l] = fminf(hi, fmaxf(lo, p[b].v[l]));
        }
        if (k >= 6 && k <= 9) {
            q[k - 6] = p[b];
        } else {
            stp_stream<N>(a.params + o, p[b]);
        }
    }
#pragma unroll
    for (int l = 0; l < N; ++l) adam_renorm(q[0].v[l], q[1].v[l], q[2].v[l], q[3].v[l]);
#pragma unroll
    for (int d = 0; d < 4; ++d) stp_stream<N>(a.params + (uint64_t)(6 + d) * a.cap + i0, q[d]);
}

// adam_update (all 11 planes' new parameters in p[], moments stored) with the
// software pipelining of adam_update_store_pipe: the same bits.
template <int N, typename G>
__device__ __forceinline__ void adam_update_pipe(const AdamLaunch& a, const AdamConsts& c, uint32_t i0,
                                                 const G& grad, Pack<N> out[11], unsigned& nz) {
    constexpr int kOrder[11] = {0, 1, 2, 3, 4, 5, 10, 6, 7, 8, 9};
    nz = 0;
    Pack<N> m[2], v[2], g[2];
    auto fetch = [&](int j, int b) {
        const uint64_t o = (uint64_t)kOrder[j] * a.cap + i0;
        m[b] = ldp_stream<N>(a.m + o);
        v[b] = ldp_stream<N>(a.v + o);
        out[kOrder[j]] = ldp_stream<N>(a.params + o);
        g[b] = grad(kOrder[j]);
    };
    fetch(0, 0);
#pragma unroll
    for (int j = 0; j < 11; ++j) {
        const int b = j & 1, k = kOrder[j];
        if (j + 1 < 11) fetch(j + 1, b ^ 1);
        const float lr = k < 3 ? c.lr[0] : (k < 6 ? c.lr[2] : (k == 10 ? c.lr[1] : c.lr[3]));
        const float lrc = __fmul_rn(lr, c.ibc1);
#pragma unroll
        for (int l = 0; l < N; ++l) {
            nz |= (g[b].v[l] != 0.f ? 1u : 0u) << l;
            adam_elem(c, lrc, out[k].v[l], m[b].v[l], v[b].v[l], g[b].v[l]);
        }
        const uint64_t o = (uint64_t)k * a.cap + i0;
        stp_stream<N>(a.m + o, m[b]);
        stp_stream<N>(a.v + o, v[b]);
        if (k < 3) {
            const float lo = a.bbox_min[k], hi = a.bbox_max[k];
#pragma unroll
            for (int l = 0; l < N; ++l) out[k].v[l] = fminf(hi, fmaxf(lo, out[k].v[l]));
        }
    }
#pragma unroll
    for (int l = 0; l < N; ++l) adam_renorm(out[6].v[l], out[7].v[l], out[8].v[l], out[9].v[l]);
}

template <int N, typename G>
__device__ __forceinline__ void adam_update_store_g(const AdamLaunch& a, const AdamConsts& c, uint32_t i0,
                                                    const G& grad) {
    unsigned nz = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        Pack<N> p = adam_plane_g<N>(a, c, d, c.lr[0], i0, grad, nz);
        const float lo = a.bbox_min[d], hi = a.bbox_max[d];
#pragma unroll
        for (int l = 0; l < N; ++l) p.v[l] = fminf(hi, fmaxf(lo, p.v[l]));
        stp_stream<N>(a.params + (uint64_t)d * a.cap + i0, p);
    }
#pragma unroll
    for (int d = 3; d < 6; ++d)
        stp_stream<N>(a.params + (uint64_t)d * a.cap + i0, adam_plane_g<N>(a, c, d, c.lr[2], i0, grad, nz));
    stp_stream<N>(a.params + (uint64_t)10 * a.cap + i0, adam_plane_g<N>(a, c, 10, c.lr[1], i0, grad, nz));
    Pack<N> q[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) q[d] = adam_plane_g<N>(a, c, 6 + d, c.lr[3], i0, grad, nz);
#pragma unroll
    for (int l = 0; l < N; ++l) adam_renorm(q[0].v[l], q[1].v[l], q[2].v[l], q[3].v[l]);
#pragma unroll
    for (int d = 0; d < 4; ++d) stp_stream<N>(a.params + (uint64_t)(6 + d) * a.cap + i0, q[d]);
}

template <int N>
__device__ __forceinline__ void adam_update_store(const AdamLaunch& a, const AdamConsts& c, uint32_t i0,
                                                  const uint32_t* gslot) {
    adam_update_store_g<N>(a, c, i0, [&](int k) { return adam_grad<N>(a, k, i0, gslot); });
}

template <int N>
__device__ __forceinline__ void adam_store(const AdamLaunch& a, uint32_t i0, const Pack<N> p[11]) {
#pragma unroll
    for (int d = 0; d < 11; ++d) stp_stream<N>(a.params + (uint64_t)d * a.cap + i0, p[d]);
}

}  // namespace gpk
