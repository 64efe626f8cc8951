// prep.cu — the fp64 half of the per-slice preprocessing and everything that
// must round like the reference (built with --fmad=false; see focus.cuh):
//   K_decide       the rest of prepare_gaussians (render.hpp:91-138) for
//                  K_filter's candidates (cull.cu) and the TileGrid pair list
//                  (render.hpp:142-160): fp64 closed form with ~1e-9
//                  ambiguity bands, the reference's own operation order inside
//                  a band, survivors compacted in set order into group-major
//                  slots, pairs bucketed by tile per group (stable: ascending
//                  slot inside a bucket) or emitted in (survivor, tile) order
//                  for the radix passes (sort.cu).
//   K_chain_exact  the reference-order fp64 backward chain for the survivors
//                  decided on the fp64 path (the others: K_chain, chain.cu).
//   k_prepared_full  every PreparedGaussian field (gpk_get_prepared_fields).
//   voxelizer      prepare_voxel_prims + VoxelTiles emission (k_vprep) and
//                  the voxel backward chain (k_vchain) (voxelize.hpp:52-240).
#include "chain.cuh"
#include "common.cuh"
#include "focus.cuh"

namespace gpk {

namespace {

__device__ __forceinline__ void load_params(const float* __restrict__ params, uint64_t cap,
                                            uint32_t i, float p[11]) {
#pragma unroll
    for (int k = 0; k < 11; ++k) p[k] = __ldg(params + (uint64_t)k * cap + i);
}

// ---- K_decide ------------------------------------------------------------------
// The rest of prepare_gaussians + the TileGrid pair list (render.hpp:91-160),
// one CTA per kDecideChunks consecutive K_filter chunks (a "group"; few enough
// groups that all CTAs are resident together), groups taken in ticket order:
//   1. each candidate gets the decision-grade fp64 closed form (fast_decide)
//      and, within ~1e-9 of a decision boundary, the reference's own fp64
//      evaluation (focus_prepare): survivors and pixel bounds — therefore tile
//      pairs — are the reference's bit for bit. Survivors are compacted in set
//      order: 48 B record + 48 B params at group-major survivor slots.
//   2. group aggregate (survivors, pairs) through a wait-free ordered prefix
//      over group words (predecessors hold earlier tickets: they are running
//      or done and publish before they wait).
//   3. survivor slots, and (tile, survivor slot) pairs in (survivor, tile)
//      order — the order a stable sort on the tile key needs to reproduce the
//      reference's ascending per-tile lists — with the first radix pass's
//      digit histograms (global, per sort tile, per super-tile).
constexpr int kDecideThreads = 256;
constexpr int kDecideGroup = kDecideGroupSize;
constexpr int kPairMap = 1024;  // pairs of a group mapped to (survivor, tile) in shared memory

template <int kMinB>
__global__ void __launch_bounds__(kDecideThreads, kMinB) k_decide(const PrepLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    extern __shared__ unsigned s_dyn_u[];
    unsigned* s_incl = s_dyn_u;                                              // kDecideGroup
    uint16_t(*s_rect)[3] = reinterpret_cast<uint16_t(*)[3]>(s_dyn_u + kDecideGroup);  // kDecideGroup x 3
    __shared__ unsigned s_hist[kMaxSortPasses][kMaxBuckets];
    __shared__ unsigned s_cnt[2][kDecideThreads / 32];
    __shared__ unsigned s_cpre[kDecideChunks + 1];
    __shared__ unsigned s_grp, s_nsurv, s_nexact;
    __shared__ unsigned s_bits[kDecideGroup / 32];  // survivor bits of the group (a.surv_bits)
    __shared__ unsigned long long s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned dmask = (1u << a.digit_bits) - 1;
    const unsigned nb = dmask + 1;
    const int tiles_x = a.slice.tiles_x;
    for (int k = tid; k < a.passes * kMaxBuckets; k += kDecideThreads) (&s_hist[0][0])[k] = 0;
    for (int k = tid; k < kDecideGroup / 32; k += kDecideThreads) s_bits[k] = 0;
    if (tid == 0) {
        s_grp = blockIdx.x;
        s_nsurv = 0;
        s_nexact = 0;
    }
    __syncthreads();
    if (warp < kDecideChunks / 32) {  // exclusive prefix of the group's chunk counts
        const unsigned c = s_grp * kDecideChunks + tid;
        const unsigned v = c < a.nfilter ? __ldcg(&a.cand_count[c]) : 0u;
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        s_cpre[tid] = incl - v;
        if (lane == 31) s_cnt[0][warp] = incl;
    }
    __syncthreads();
    if (tid < kDecideChunks && warp > 0)
        for (int w = 0; w < warp; ++w) s_cpre[tid] += s_cnt[0][w];
    if (tid == 0) {
        unsigned tot = 0;
        for (int w = 0; w < kDecideChunks / 32; ++w) tot += s_cnt[0][w];
        s_cpre[kDecideChunks] = tot;
    }
    __syncthreads();
    const unsigned g = s_grp;
    // the preceding K_filter / fused Adam + cull cleared the dense gradient
    // planes as the state word said (the dense chain sets it again)
    if (a.grads && blockIdx.x == 0 && tid == 0) *a.grads_dirty = 0u;
    const uint32_t base = g * kDecideGroup;
    const unsigned nc = s_cpre[kDecideChunks];

    // ---- 1. exact decision, survivors compacted in order -------------------------
    for (unsigned j0 = 0, r = 0; j0 < nc; j0 += kDecideThreads, r ^= 1) {
        const unsigned j = j0 + tid;
        SurvivorRecord rec;
        float pf[11];
        uint32_t i = 0;
        bool survive = false;
        if (j < nc) {
            int q = 0;  // chunk of candidate j: last q with s_cpre[q] <= j
#pragma unroll
            for (int step = kDecideChunks / 2; step > 0; step >>= 1)
                if (s_cpre[q + step] <= j) q += step;
            load_cand(a.cand + (uint64_t)base + q * kFilterBlock + (j - s_cpre[q]), pf, i);
            uint32_t flag = 0;
            const int fr = fast_decide(pf, a.slice, rec);
            if (fr == kFastSurvive) {
                survive = true;
            } else if (fr == kAmbiguous) {
                flag = kExactFlag;
                // near a decision boundary: the reference's own fp64 evaluation
                double pd[11];
#pragma unroll
                for (int t = 0; t < 11; ++t) pd[t] = (double)pf[t];
                Focus f;
                const int res = focus_prepare(pd, a.slice, f);
                if (res == kSurvive) {
                    survive = true;
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
                } else if (res > 0) {
                    record_error(a.err, res, i);
                }
            }
            rec.gidx = i | flag;
            rec.pair_base = 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, survive);
        const unsigned mx = __ballot_sync(0xffffffffu, survive && (rec.gidx & kExactFlag));
        if (lane == 0) {
            s_cnt[r][warp] = __popc(m);
            if (mx) atomicAdd(&s_nexact, (unsigned)__popc(mx));
        }
        __syncthreads();
        unsigned rank = s_nsurv + __popc(m & lanemask_lt());
        for (int w = 0; w < warp; ++w) rank += s_cnt[r][w];
        if (survive) {
            a.records[base + rank] = rec;
            store_cand(a.surv_params + base + rank, pf, i);
            a.survivor_list[base + rank] = i;
            atomicOr(&s_bits[(i - base) >> 5], 1u << (i & 31));
            // fp64-decided survivors take the fp64 chain (K_chain_exact, which
            // runs beside K_chain once the backward is done)
            if (rec.gidx & kExactFlag) a.exact_list[atomicAdd(&a.ctrl->chain_exact, 1u)] = base + rank;
            const unsigned tx0 = rec.lo_x / kTile, ty0 = rec.lo_y / kTile;
            const unsigned ntx = rec.hi_x / kTile - tx0 + 1, nty = rec.hi_y / kTile - ty0 + 1;
            s_rect[rank][0] = (uint16_t)tx0;
            s_rect[rank][1] = (uint16_t)ty0;
            s_rect[rank][2] = (uint16_t)ntx;
            s_incl[rank] = ntx * nty;
        }
        __syncthreads();
        if (tid == 0) {
            unsigned t = 0;
            for (int w = 0; w < kDecideThreads / 32; ++w) t += s_cnt[r][w];
            s_nsurv += t;
        }
    }
    __syncthreads();
    const unsigned S = s_nsurv;
    if (a.surv_bits)  // the group's 4096 bits, every word (no clearing between slices)
        for (int k = tid; k < kDecideGroup / 32; k += kDecideThreads) a.surv_bits[(uint64_t)g * (kDecideGroup / 32) + k] = s_bits[k];
    if (tid == 0) {  // statistics (gpk_prepare_stats)
        if (nc) atomicAdd(&a.ctrl->candidates, nc);
        if (s_nexact) atomicAdd(&a.ctrl->exact_decided, s_nexact);
    }

    // ---- 2. inclusive scan of the pair counts, ordered group prefix -------------
    {
        constexpr int kPer = kDecideGroup / kDecideThreads;  // consecutive survivors per thread
        const unsigned j0 = tid * kPer;
        unsigned run = 0;
        for (int q = 0; q < kPer; ++q) run += (j0 + q < S) ? s_incl[j0 + q] : 0u;
        unsigned incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_cnt[0][warp] = incl;
        __syncthreads();
        unsigned ex = incl - run;
        for (int w = 0; w < warp; ++w) ex += s_cnt[0][w];
        for (int q = 0; q < kPer && j0 + q < S; ++q) {
            ex += s_incl[j0 + q];
            s_incl[j0 + q] = ex;
        }
    }
    __syncthreads();
    const unsigned Pb = S ? s_incl[S - 1] : 0u;
    // ---- 2. reserve the group's pair range (no ordering between groups here:
    // the radix pass orders pairs of equal tile by group index, i.e. by slot)
    if (tid == 0) {
        const unsigned P0 = atomicAdd(&a.ctrl->pairs, Pb);
        if (S) atomicAdd(&a.ctrl->survivors, S);
        if ((unsigned long long)P0 + Pb > a.pair_cap) a.ctrl->pair_overflow = 1u;
        a.grp_pairs[g] = make_uint2(P0, Pb);
        a.grp_surv[g] = S;
        s_excl = P0;
    }
    __syncthreads();

    // ---- 3. pair bases and pair emission ------------------------------------------
    const unsigned P0 = (unsigned)s_excl;
    // a group of at most kPairMap pairs (the common case) maps each pair to
    // its (survivor, tile) up front: survivor j writes its rect's tiles in
    // row-major order (no per-pair search or division below)
    unsigned* s_pair = s_dyn_u + kDecideGroup + kDecideGroup * 3 / 2 + kDecideThreads / 32 * kMaxBuckets / 2;
    const bool direct = Pb <= (unsigned)kPairMap;
    for (unsigned j = tid; j < S; j += kDecideThreads) {
        const unsigned k0 = j ? s_incl[j - 1] : 0u;
        a.records[base + j].pair_base = P0 + k0;
        if (direct) {
            const unsigned ntx = s_rect[j][2], nty = (s_incl[j] - k0) / ntx;
            const unsigned t0 = s_rect[j][1] * (unsigned)tiles_x + s_rect[j][0];
            unsigned k = k0;
            for (unsigned dy = 0; dy < nty; ++dy)
                for (unsigned dx = 0; dx < ntx; ++dx) s_pair[k++] = (j << 20) | (t0 + dy * (unsigned)tiles_x + dx);
        }
    }
    if (direct) __syncthreads();
    // tile of the group's k-th pair (pairs in (survivor, tile-in-rect) order)
    auto pair_tile = [&](unsigned k, unsigned& surv) {
        if (direct) {
            const unsigned e = s_pair[k];
            surv = e >> 20;
            return e & 0xfffffu;
        }
        unsigned lo = 0, hi = S - 1;
        while (lo < hi) {
            const unsigned mid = (lo + hi) >> 1;
            if (s_incl[mid] > k) hi = mid; else lo = mid + 1;
        }
        surv = lo;
        const unsigned local = k - (lo ? s_incl[lo - 1] : 0u);
        const unsigned ntx = s_rect[lo][2];
        return (s_rect[lo][1] + local / ntx) * (unsigned)tiles_x + s_rect[lo][0] + local % ntx;
    };
    if (a.bucket_tab) {
        // single-pass slice (every tile is one digit): bucket the group's pairs
        // by tile — counts, bucket starts (published for k_gather), then slots
        // into their buckets in pair order (stable). Pairs go in rounds of
        // 1024, warp w taking 4 x 32 consecutive ones; a round's tiles are
        // found once (binary search over the survivors' pair counts) and, for
        // a one-round group (the common case), kept in registers for the fill.
        constexpr int kSub = 4;
        constexpr unsigned kRound = kDecideThreads * kSub;
        unsigned tl[kSub], jj[kSub];
        auto round_tiles = [&](unsigned r0) {
#pragma unroll
            for (int q = 0; q < kSub; ++q) {
                const unsigned k = r0 + (unsigned)(warp * kSub + q) * 32 + lane;
                tl[q] = k < Pb ? pair_tile(k, jj[q]) : 0xffffffffu;
            }
        };
        for (unsigned r0 = 0; r0 < Pb; r0 += kRound) {
            round_tiles(r0);
#pragma unroll
            for (int q = 0; q < kSub; ++q) {  // warp-aggregated counts
                const unsigned peers = __match_any_sync(0xffffffffu, tl[q]);
                if (tl[q] != 0xffffffffu && (__ffs(peers) - 1) == lane)
                    atomicAdd(&s_hist[0][tl[q]], (unsigned)__popc(peers));
            }
        }
        __syncthreads();
        unsigned* s_start = &s_hist[1][0];
        {
            constexpr int kPer = kMaxBuckets / kDecideThreads;
            const unsigned d0 = tid * kPer;
            unsigned v[kPer], run = 0;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                v[q] = s_hist[0][d0 + q];
                run += v[q];
            }
            unsigned incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) s_cnt[0][warp] = incl;
            __syncthreads();
            unsigned ex = incl - run;
            for (int w = 0; w < warp; ++w) ex += s_cnt[0][w];
            // the group's column of bucket starts (+ end) in the tile-major table
            unsigned* tcol = a.bucket_tab + g;
            const uint64_t gs = a.bucket_gstride;
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                s_start[d0 + q] = ex;
                if (d0 + q < nb) tcol[(d0 + q) * gs] = P0 + ex;
                s_hist[0][d0 + q] = 0;  // becomes the fill counter
                ex += v[q];
            }
            if (tid == 0) tcol[nb * gs] = P0 + Pb;
        }
        __syncthreads();
        // stable fill: each bucket receives its pairs in pair order (= ascending
        // slot, one pair per survivor and tile), so the gather is a plain
        // concatenation. Per round: warp w ranks its pairs with
        // __match_any_sync against its own counter of the tile; a pair's slot
        // in its bucket is the bucket's fill before the round + the counts of
        // the tile in earlier warps + its rank. Only the round's tiles are
        // touched (no per-digit sweeps).
        uint16_t(*s_w16)[kMaxBuckets] = reinterpret_cast<uint16_t(*)[kMaxBuckets]>(s_dyn_u + kDecideGroup + kDecideGroup * 3 / 2);
        for (unsigned r0 = 0; r0 < Pb; r0 += kRound) {
            if (Pb > kRound) round_tiles(r0);  // (one round: the tiles are still in registers)
#pragma unroll
            for (int q = 0; q < kSub; ++q)
                if (tl[q] != 0xffffffffu)
#pragma unroll
                    for (int w = 0; w < kDecideThreads / 32; ++w) s_w16[w][tl[q]] = 0;
            __syncthreads();
            unsigned rk[kSub], pc[kSub];
#pragma unroll
            for (int q = 0; q < kSub; ++q) {
                const bool valid = tl[q] != 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, tl[q]);
                const unsigned prior = valid ? s_w16[warp][tl[q]] : 0u;
                __syncwarp();
                const bool leader = valid && (__ffs(peers) - 1) == lane;
                if (leader) s_w16[warp][tl[q]] = (uint16_t)(prior + __popc(peers));
                __syncwarp();
                rk[q] = prior + __popc(peers & lanemask_lt());
                pc[q] = leader ? (unsigned)__popc(peers) : 0u;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kSub; ++q)
                if (tl[q] != 0xffffffffu) {
                    unsigned b = s_hist[0][tl[q]] + rk[q];
                    for (int w = 0; w < warp; ++w) b += s_w16[w][tl[q]];
                    const unsigned long long pos = (unsigned long long)P0 + s_start[tl[q]] + b;
                    if (pos < a.pair_cap) a.vals[pos] = base + jj[q];
                }
            __syncthreads();  // every base read before the fills advance
#pragma unroll
            for (int q = 0; q < kSub; ++q)
                if (pc[q]) atomicAdd(&s_hist[0][tl[q]], pc[q]);
            __syncthreads();
        }
        // (each tile's list start is derived by its gather from the rows)
        return;
    }
    for (unsigned k = tid; k < Pb; k += kDecideThreads) {
        unsigned lo;
        const unsigned tile = pair_tile(k, lo);
        const unsigned long long pos = (unsigned long long)P0 + k;
        if (pos < a.pair_cap) {
            a.keys[pos] = tile;
            a.vals[pos] = base + lo;
            for (int ps = 0; ps < a.passes; ++ps)
                atomicAdd(&s_hist[ps][(tile >> (a.digit_bits * ps)) & dmask], 1u);
        }
    }
    __syncthreads();
    // first radix pass: this group's digit-count row (plain stores, every digit),
    // its super-row and the global counts of every pass
    unsigned* row = a.tile_hist0 + (uint64_t)g * nb;
    unsigned* super = sort_super_row(a.tile_hist0, a.sort_tiles_cap, nb, g);
    for (unsigned d = tid; d <= dmask; d += kDecideThreads) {
        const unsigned v = s_hist[0][d];
        row[d] = v;
        if (v) atomicAdd(&super[d], v);
    }
    for (int ps = 0; ps < a.passes; ++ps)
        for (unsigned d = tid; d <= dmask; d += kDecideThreads) {
            const unsigned v = s_hist[ps][d];
            if (v) atomicAdd(&a.hist[ps * kMaxBuckets + d], v);
        }
}

// K_chain_exact: the reference's fp64 chain for the deferred survivors.
__global__ void __launch_bounds__(128) k_chain_exact(const ChainLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned E = *a.exact_count;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        const uint32_t cid = a.exact_list[e];  // record slot
        const SurvivorRecord rec = a.records[cid];
        float pf[11];
        uint32_t i;
        load_cand(a.sparams + cid, pf, i);
        double acc[6];
        merge_partials(a, rec, acc);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        Focus f;
        focus_prepare(pd, a.slice, f);
        double gd[11];
        D3 dl_dmu;
        focus_backward(pd, f, acc, a.slice, gd, dl_dmu);
        float g[11], dmu[3] = {(float)dl_dmu.x, (float)dl_dmu.y, (float)dl_dmu.z};
#pragma unroll
        for (int k = 0; k < 11; ++k) g[k] = (float)gd[k];
        store_chain(a, i, cid, g, dmu, acc);
    }
}

// ---- PreparedGaussian in full (render.hpp:68-79) ----------------------------------
// For the survivors listed by slot (set order), every field the reference's
// prepare_gaussians fills, in the reference's own fp64 operation order
// (focus_prepare; this TU is built --fmad=false): alpha, opacity_r,
// alpha_tilde, mu_c, mu_e, sigma_c, sigma_c_inv, sigma_e, mu_2d, cov2d,
// conic, det2 — 47 doubles per survivor (include/gpile_b200.h). Read-out only:
// the pixel kernels use the 48 B SurvivorRecord.
__global__ void __launch_bounds__(128) k_prepared_full(const CandParams* __restrict__ sparams,
                                                       const uint32_t* __restrict__ slots, unsigned S,
                                                       const SliceArgs s, double* __restrict__ out) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= S) return;
    float pf[11];
    uint32_t idx;
    load_cand(sparams + slots[k], pf, idx);
    double pd[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) pd[t] = (double)pf[t];
    Focus f;
    focus_prepare(pd, s, f);
    D33 sigma, rot, sc;
    D3 scale;
    world_covariance(pd, s.mod, sigma, rot, scale);
    if (s.identity_rot) {
        sc = sigma;
    } else {
        D33 Rc;
#pragma unroll
        for (int i = 0; i < 9; ++i) Rc.m[i / 3][i % 3] = s.R[i];
        sc = m33_mul(m33_mul(Rc, sigma), m33_t(Rc));
    }
    double* o = out + 47ull * k;
    o[0] = f.alpha;
    o[1] = f.op;
    o[2] = f.alpha_tilde;
    o[3] = f.mu_c.x, o[4] = f.mu_c.y, o[5] = f.mu_c.z;
    o[6] = f.mu_e.x, o[7] = f.mu_e.y, o[8] = f.mu_e.z;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        o[9 + i] = sc.m[i / 3][i % 3];
        o[18 + i] = f.A.m[i / 3][i % 3];
        o[27 + i] = f.Se.m[i / 3][i % 3];
    }
    o[36] = f.mu_e.x, o[37] = f.mu_e.y;  // mu_2d (render.hpp:53-56)
    o[38] = f.cov_a, o[39] = f.cov_b, o[40] = f.cov_c, o[41] = f.cov_d;
    o[42] = f.con_a, o[43] = f.con_b, o[44] = f.con_c, o[45] = f.con_d;
    o[46] = f.det2;
}

// ---- voxelizer: prepare_voxel_prims + VoxelTiles (voxelize.hpp:52-105) ---------
// Persistent CTAs take 256-primitive chunks in set order. Per primitive: the
// world covariance and its inverse in the reference's fp64 order (support
// bounds must reproduce the reference's integer voxel ranges exactly,
// voxelize.hpp:66-74; invert_covariance raises the same errors), a 64 B record
// for the evaluation kernel, and (8^3-tile, primitive) pairs emitted in
// (primitive, tile) order through the same wait-free ordered prefix as K_exact.
__global__ void __launch_bounds__(256) k_vprep(const VoxPrepLaunch a) {
    // Two chunks in flight per CTA: chunk c's primitives are computed and its
    // aggregate published, then chunk c-1's (claimed the previous round)
    // prefix is looked up and its pairs emitted — by then its predecessors
    // have long published, so the look-up rarely waits.
    __shared__ unsigned s_chunk;
    __shared__ unsigned long long s_incl[2][256];
    __shared__ uint16_t s_t0[2][256][3];
    __shared__ uint16_t s_nt[2][256][2];  // tiles along x and y of the primitive's box
    __shared__ unsigned long long s_warp[8];
    __shared__ unsigned long long s_excl;
    __shared__ unsigned s_hist[kMaxSortPasses][kMaxBuckets];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = tid; k < kMaxSortPasses * kMaxBuckets; k += 256) (&s_hist[0][0])[k] = 0;
    const unsigned dmask = (1u << a.digit_bits) - 1;
    const unsigned nchunks = (a.n + 255) / 256;
    const VoxArgs& v = a.v;
    constexpr float kK = -0.72134752044448170368f;  // -0.5 * log2(e)

    unsigned prev = 0xffffffffu;  // chunk awaiting emission (buffer cur ^ 1)
    int cur = 0;
    while (true) {
        __syncthreads();
        if (tid == 0) s_chunk = atomicAdd(&a.ctrl->exact_chunk_ctr, 1u);
        __syncthreads();
        const unsigned chunk = s_chunk;
        const bool have = chunk < nchunks;
        if (have) {
            const uint32_t i = chunk * 256 + tid;
            unsigned long long val = 0;
            if (i < a.n) {
                float pf[11];
                load_params(a.params, a.cap, i, pf);
                double pd[11];
#pragma unroll
                for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
                D33 sigma, rot, inv;
                D3 scale;
                int e = world_covariance(pd, v.mod, sigma, rot, scale);
                if (!e) e = invert_cov(sigma, scale, v.mod, inv);
                if (e) {
                    record_error(a.err, e, i);
                } else {
                    const double alpha = 1.0 / (1.0 + exp(-pd[10]));
                    int lo[3], hi[3];
                    bool inside = true;
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        const double half = v.support * sqrt(sigma.m[d][d]);
                        const double lo_w = pd[d] - half, hi_w = pd[d] + half;
                        lo[d] = max(0, x86_trunc_int(ceil((lo_w - v.origin[d]) / v.spacing[d])));
                        hi[d] = min(v.dims[d] - 1, x86_trunc_int(floor((hi_w - v.origin[d]) / v.spacing[d])));
                        if (lo[d] > hi[d]) inside = false;
                    }
                    if (inside) {
                        unsigned np = 1;
                        unsigned nt[3];
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            const int t0 = lo[d] / v.tile[d];
                            nt[d] = (unsigned)(hi[d] / v.tile[d] - t0 + 1);
                            np *= nt[d];
                            s_t0[cur][tid][d] = (uint16_t)t0;
                        }
                        s_nt[cur][tid][0] = (uint16_t)nt[0];
                        s_nt[cur][tid][1] = (uint16_t)nt[1];
                        val = (1ull << 32) | np;
                        VoxRecord rec;
                        rec.mu[0] = pf[0];
                        rec.mu[1] = pf[1];
                        rec.mu[2] = pf[2];
                        rec.log2a = (float)log2(alpha);
                        rec.a[0] = (float)inv.m[0][0] * kK;
                        rec.a[1] = (float)inv.m[1][1] * kK;
                        rec.a[2] = (float)inv.m[2][2] * kK;
                        rec.a[3] = (float)(inv.m[0][1] + inv.m[1][0]) * kK;
                        rec.a[4] = (float)(inv.m[0][2] + inv.m[2][0]) * kK;
                        rec.a[5] = (float)(inv.m[1][2] + inv.m[2][1]) * kK;
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            rec.lo[d] = (uint16_t)lo[d];
                            rec.hi[d] = (uint16_t)hi[d];
                        }
                        rec.gidx = i;
                        rec.pair_base = 0;
                        rec.pad = 0;
                        a.records[i] = rec;
                    }
                }
            }
            unsigned long long incl = val;
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
            s_incl[cur][tid] = incl;
            __syncthreads();
            if (tid == 0) warp_prefix_publish(a.chunk_words, chunk, s_incl[cur][255]);
        }
        if (prev != 0xffffffffu) {
            const int pb = cur ^ 1;
            const unsigned long long agg = s_incl[pb][255];
            if (warp == 0) {
                const unsigned long long excl = warp_prefix_aggregates(a.chunk_words, prev, agg, false);
                if (lane == 0) {
                    s_excl = excl;
                    if (prev == nchunks - 1) {
                        const unsigned long long tot = excl + agg;
                        const unsigned P = (unsigned)(tot & 0xffffffffull);
                        a.ctrl->survivors = (unsigned)(tot >> 32);
                        a.ctrl->pairs = P;
                        a.ctrl->pair_overflow = (P > a.pair_cap) ? 1u : 0u;
                    }
                }
            }
            __syncthreads();
            const unsigned S0 = (unsigned)(s_excl >> 32);
            const unsigned P0 = (unsigned)(s_excl & 0xffffffffull);
            const unsigned long long* inc = s_incl[pb];
            {
                const uint32_t i = prev * 256 + tid;
                const unsigned long long pv = tid ? inc[tid - 1] : 0ull;
                if ((inc[tid] >> 32) != (pv >> 32)) {
                    a.survivor_list[S0 + (unsigned)(pv >> 32)] = i;
                    a.records[i].pair_base = P0 + (unsigned)(pv & 0xffffffffull);
                }
            }
            const unsigned Pb = (unsigned)(agg & 0xffffffffull);
            for (unsigned k = tid; k < Pb; k += 256) {
                unsigned lo = 0, hi = 255;
                while (lo < hi) {
                    const unsigned mid = (lo + hi) >> 1;
                    if ((unsigned)(inc[mid] & 0xffffffffull) > k) hi = mid; else lo = mid + 1;
                }
                const unsigned before = lo ? (unsigned)(inc[lo - 1] & 0xffffffffull) : 0u;
                const unsigned local = k - before;
                const unsigned ntx = s_nt[pb][lo][0], nty = s_nt[pb][lo][1];
                const unsigned dx = local % ntx, rest = local / ntx;
                const unsigned dy = rest % nty, dz = rest / nty;
                // z-major tile index (voxelize.hpp:98-101): ((tz * ny) + ty) * nx + tx
                const unsigned tile = ((s_t0[pb][lo][2] + dz) * (unsigned)v.ntiles[1] + (s_t0[pb][lo][1] + dy)) *
                                          (unsigned)v.ntiles[0] + (s_t0[pb][lo][0] + dx);
                const unsigned long long pos = (unsigned long long)P0 + k;
                if (pos < a.pair_cap) {
                    a.keys[pos] = tile;
                    a.vals[pos] = prev * 256 + lo;
                    if (a.passes > 0) {
                        const unsigned st = (unsigned)(pos / ((uint64_t)kSortTile << a.tile_shift));
                        sort_count(a.tile_hist0, a.sort_tiles_cap, dmask + 1, st, tile & dmask, 1u);
                    }
                    for (int ps = 0; ps < a.passes; ++ps)
                        atomicAdd(&s_hist[ps][(tile >> (a.digit_bits * ps)) & dmask], 1u);
                }
            }
        }
        if (!have) break;
        prev = chunk;
        cur ^= 1;
    }
    __syncthreads();
    for (int ps = 0; ps < a.passes; ++ps)
        for (unsigned d = tid; d <= dmask; d += 256) {
            const unsigned c = s_hist[ps][d];
            if (c) atomicAdd(&a.hist[ps * kMaxBuckets + d], c);
        }
}

// voxelize_backward stage 3 (voxelize.hpp:217-232): merge per-tile sums in
// tile order, dL/dSigma = sym(-Sigma^-1 dL/dSigma^-1 Sigma^-1), world chain.
__global__ void __launch_bounds__(128) k_vchain(const VoxChainLaunch a) {
    const unsigned S = a.ctrl->survivors;
    for (unsigned slot = blockIdx.x * blockDim.x + threadIdx.x; slot < S;
         slot += gridDim.x * blockDim.x) {
        const uint32_t i = a.survivor_list[slot];
        const VoxRecord rec = a.records[i];
        unsigned np = 1;
#pragma unroll
        for (int d = 0; d < 3; ++d) np *= (unsigned)(rec.hi[d] / a.v.tile[d] - rec.lo[d] / a.v.tile[d] + 1);
        double acc[10];
#pragma unroll
        for (int j = 0; j < 10; ++j) acc[j] = 0.0;
        const float* part = a.partials + 10ull * rec.pair_base;
        for (unsigned k = 0; k < np; ++k)
#pragma unroll
            for (int j = 0; j < 10; ++j) acc[j] += (double)part[10 * k + j];
        float pf[11];
        load_params(a.params, a.cap, i, pf);
        double pd[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) pd[k] = (double)pf[k];
        D33 sigma, rot, inv;
        D3 scale;
        world_covariance(pd, a.v.mod, sigma, rot, scale);
        invert_cov(sigma, scale, a.v.mod, inv);
        D33 dA;
        dA.m[0][0] = acc[4];
        dA.m[1][1] = acc[5];
        dA.m[2][2] = acc[6];
        dA.m[0][1] = dA.m[1][0] = acc[7];
        dA.m[0][2] = dA.m[2][0] = acc[8];
        dA.m[1][2] = dA.m[2][1] = acc[9];
        D33 ds = m33_scale(m33_mul(m33_mul(inv, dA), inv), -1.0);
        ds = m33_scale(m33_add(ds, m33_t(ds)), 0.5);
        double d_ls[3], d_q[4];
        chain_world(pd, ds, a.v.mod, d_ls, d_q);
        const double alpha = 1.0 / (1.0 + exp(-pd[10]));
        float g[11] = {(float)acc[1], (float)acc[2], (float)acc[3], (float)d_ls[0], (float)d_ls[1],
                       (float)d_ls[2], (float)d_q[0], (float)d_q[1], (float)d_q[2], (float)d_q[3],
                       (float)(acc[0] * (alpha * (1.0 - alpha)))};
        if (!isfinite(g[10] + g[0] + g[3] + g[6])) record_error(a.err, kErrNumeric, i);  // voxelize.hpp:234-238
#pragma unroll
        for (int k = 0; k < 11; ++k) a.grads[(uint64_t)k * a.cap + i] = g[k];
    }
}

}  // namespace

void launch_prepared_full(const CandParams* sparams, const uint32_t* slots, unsigned S, const SliceArgs& s,
                          double* out, cudaStream_t st) {
    if (S) k_prepared_full<<<(S + 127) / 128, 128, 0, st>>>(sparams, slots, S, s, out);
}

void launch_vox_prep(const VoxPrepLaunch& a, cudaStream_t st) {
    if (a.n) k_vprep<<<a.grid, 256, 0, st>>>(a);
}

void launch_vox_chain(const VoxChainLaunch& a, int grid, cudaStream_t st) {
    k_vchain<<<grid, 128, 0, st>>>(a);
}

void launch_bin(const PrepLaunch& a, int num_sms, cudaStream_t st) {
    if (!a.n) return;
    // survivors' pair prefixes and rects, the stable fill's warp tables, the pair map
    const int smem = kDecideGroup * (4 + 6) + 8 * kMaxBuckets * 2 + kPairMap * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_decide<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_decide<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const unsigned groups = (a.nfilter + kDecideChunks - 1) / kDecideChunks;
    // one wave at 2 CTAs/SM: the unconstrained registers (114); more groups
    // than that (large sets): 3 CTAs/SM (80 registers, a 64 B spill) — C5 bin
    // 54.7 -> 46.5 us, C2 19.3 -> 19.9 us measured
    if (groups > 2u * (unsigned)num_sms) launch_pdl(k_decide<3>, dim3(groups), dim3(kDecideThreads), smem, st, a);
    else launch_pdl(k_decide<2>, dim3(groups), dim3(kDecideThreads), smem, st, a);
}

void launch_chain_exact(const ChainLaunch& a, int grid, cudaStream_t st) {
    launch_pdl(k_chain_exact, dim3(std::max(1, grid / 8)), dim3(128), 0, st, a);
}

}  // namespace gpk
