// chain.cuh — stage 2 + the gradient store of the backward chain
// (backward.hpp:141-185), shared by K_chain (chain.cu, FMA contraction on) and
// K_chain_exact (prep.cu, the reference's fp64 operation order, --fmad=false).
#pragma once

#include "common.cuh"

namespace gpk {

// Stage-2 merge of one survivor's per-tile sums in tile order (backward.hpp:141-145).
// The partials of up to 4 tiles are requested together before any is added
// (a survivor covers 1-4 tiles at these scales): one L2 round trip instead of
// one per tile; the adds keep tile order (the same bits). Split in two so the
// caller can do independent work between the loads and the adds.
struct PartialsBatch {
    float2 q[4][3];
    unsigned np;
    const float2* part;
};

__device__ __forceinline__ void merge_partials_issue(const ChainLaunch& a, const SurvivorRecord& rec,
                                                     PartialsBatch& pb) {
    const unsigned ntx = rec.hi_x / kTile - rec.lo_x / kTile + 1;
    const unsigned nty = rec.hi_y / kTile - rec.lo_y / kTile + 1;
    pb.np = ntx * nty;
    pb.part = reinterpret_cast<const float2*>(a.partials + 6ull * rec.pair_base);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if ((unsigned)u < pb.np) {
            pb.q[u][0] = pb.part[3 * u];
            pb.q[u][1] = pb.part[3 * u + 1];
            pb.q[u][2] = pb.part[3 * u + 2];
        }
}

__device__ __forceinline__ void merge_partials_finish(const PartialsBatch& pb, double acc[6]) {
#pragma unroll
    for (int j = 0; j < 6; ++j) acc[j] = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if ((unsigned)u < pb.np) {
            acc[0] += (double)pb.q[u][0].x;
            acc[1] += (double)pb.q[u][0].y;
            acc[2] += (double)pb.q[u][1].x;
            acc[3] += (double)pb.q[u][1].y;
            acc[4] += (double)pb.q[u][2].x;
            acc[5] += (double)pb.q[u][2].y;
        }
    for (unsigned k = 4; k < pb.np; ++k) {
        const float2 p0 = pb.part[3 * k], p1 = pb.part[3 * k + 1], p2 = pb.part[3 * k + 2];
        acc[0] += (double)p0.x;
        acc[1] += (double)p0.y;
        acc[2] += (double)p1.x;
        acc[3] += (double)p1.y;
        acc[4] += (double)p2.x;
        acc[5] += (double)p2.y;
    }
}

__device__ __forceinline__ void merge_partials(const ChainLaunch& a, const SurvivorRecord& rec, double acc[6]) {
    PartialsBatch pb;
    merge_partials_issue(a, rec, pb);
    merge_partials_finish(pb, acc);
}

// Gradient of set index i (survivor slot cid): the dense planes, or the slot
// planes in slot-gradient mode (coalesced: a CTA's survivors are consecutive).
__device__ __forceinline__ void store_chain(const ChainLaunch& a, uint32_t i, uint32_t cid, const float g[11],
                                            const float dmu[3], const double acc[6]) {
    const bool finite = isfinite(g[10]) && isfinite(g[0] + g[1] + g[2]) &&
                        isfinite(g[3] + g[4] + g[5]) && isfinite(g[6] + g[7] + g[8] + g[9]);
    if (!finite) record_error(a.err, kErrNumeric, i);  // backward.hpp:175-185
    float* dst = a.slot_grads ? a.slot_grads + cid : a.grads + i;
    if (a.urows) {  // data-parallel union row (a survivor is always in the union)
        const uint32_t m = a.umap[i];
        dst = (m && m - 1 < a.ucap) ? a.urows + (m - 1) : nullptr;
    }
    if (dst)
#pragma unroll
        for (int k = 0; k < 11; ++k) dst[(uint64_t)k * a.cap] = g[k];
    if (a.slot_grads && !a.urows) a.gmap[i] = (uint16_t)(cid % kDecideGroupSize + 1);
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

}  // namespace gpk
