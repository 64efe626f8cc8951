// sort.cu — hand-written stable LSD radix sort of (tile key, slot) pairs, one
// kernel per digit of up to kMaxDigitBits bits (one pass for up to 1024 tiles
// = a 512x512 slice, two passes up to 2^20 tiles).
//
// Stability is the whole point: the output must list each tile's survivors in
// ascending slot (= set) order to reproduce the reference's per-tile lists
// (render.hpp:151-157) bit-exactly.
//
// Sort tiles. The first pass over K_decide's output takes the K_decide GROUPS
// as its tiles, in group order: each group wrote its pairs in (slot, tile)
// order into a range it reserved atomically (anywhere in the pair array), its
// digit-count row and its super-row counts. Ordering groups by index here is
// what makes the result stable in slot order, so K_decide never waits on
// another group. Later passes (and the voxelizer's single ordered emission) use
// tiles of kSortTile consecutive positions, counted by the producing pass.
//
// Wait-free passes: a CTA knows a tile's output offsets up front — global digit
// base (exclusive scan of the global histogram) + the column sum of the digit
// rows of all earlier tiles (whole super-tiles from the super rows, then at
// most kSuperTiles-1 rows) — and never waits on another CTA. Inside a tile,
// rounds of kSortTile pairs keep running per-digit offsets; in a round, warp w
// owns a contiguous segment processed 32 at a time, ranks from
// __match_any_sync, so the order inside a tile is the input order.
#include "common.cuh"

namespace gpk {

namespace {

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const SortLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_whist[8][kMaxBuckets];   // per-warp digit counts -> offsets
    __shared__ unsigned s_base[kMaxBuckets];       // running digit offsets of this tile
    __shared__ unsigned s_gbase[kMaxBuckets];      // exclusive scan of the pass histogram
    __shared__ unsigned s_delta[kMaxBuckets];      // round: output position - staging slot, per digit
    __shared__ unsigned s_wsum[32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
    const bool groups = a.grp_pairs != nullptr;
    const unsigned tile_keys = (unsigned)kSortTile << a.tile_shift;
    const unsigned ntiles = groups ? a.ngroups : (P + tile_keys - 1) / tile_keys;
    const unsigned nb = 1u << a.bits;
    const unsigned mask = nb - 1;
    // narrow digits: a round's pairs are staged digit-major in shared memory so
    // the scatter writes runs (C5's 64-digit passes: -2 us); at 512 digits
    // (the voxelizer) runs average 2 pairs and the staging costs more (+7 us)
    const bool staged = nb <= 256;
    if (blockIdx.x == 0 && tid == 0 && a.grp_begin) a.grp_begin[nb] = P;
    if (blockIdx.x == 0 && tid == 0 && !a.tile_hist_next) {
        // rows the filter clears before the next prepare: the largest tile
        // count any pass of this sort used (group rows or position tiles)
        const unsigned pos_tiles = (P + tile_keys - 1) / tile_keys;
        a.prev_sort_words[0] = max(ntiles, max(pos_tiles, a.ngroups));
        a.prev_sort_words[1] = nb;
        a.prev_sort_words[2] = (unsigned)a.pass + 1;
    }

    // ---- global digit base: exclusive scan of the histogram (nb <= 1024), once
    // per CTA
    if (blockIdx.x < ntiles) {
        constexpr int kPer = kMaxBuckets / kSortThreads;  // 4 digits per thread
        unsigned v[kPer], run = 0;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const unsigned d = tid * kPer + i;
            v[i] = d < nb ? a.hist[d] : 0;
            run += v[i];
        }
        unsigned incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        unsigned ex = incl - run;
        for (int w = 0; w < warp; ++w) ex += s_wsum[w];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const unsigned d = tid * kPer + i;
            s_gbase[d] = ex;
            // last pass: the digit groups' sorted start positions let the
            // pixel kernels find their tile's range without a search
            if (a.grp_begin && blockIdx.x == 0 && d < nb) a.grp_begin[d] = ex;
            ex += v[i];
        }
        __syncthreads();
    }

    for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
        unsigned first, count;
        if (groups) {
            const uint2 gp = __ldcg(&a.grp_pairs[t]);
            first = min(gp.x, P);
            count = min(gp.x + gp.y, P) - first;
        } else {
            first = t * tile_keys;
            count = min(P - first, tile_keys);
        }
        // ---- add the counts of all earlier tiles: the super row holds the
        // prefix over the earlier super-tiles (k_super_scan), then the earlier
        // tiles of this super-tile (<= 15 rows). Thread owns 4 consecutive
        // digits (one 16 B load per row); rows are unrolled so all of a
        // thread's loads are in flight together.
        {
            const unsigned* region = a.tile_hist;
            const unsigned sup = t / kSuperTiles, t0 = sup * kSuperTiles;
            const unsigned nrows = 1 + (t - t0);  // the super prefix, then tile rows
            auto row_of = [&](unsigned r) -> const unsigned* {
                return r == 0 ? region + (a.sort_tiles_cap + sup) * nb : region + (size_t)(t0 + r - 1) * nb;
            };
            if (nb >= 4) {
                const unsigned d0 = tid * 4;
                if (d0 < nb) {
                    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 8
                    for (unsigned r = 0; r < nrows; ++r) {
                        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(row_of(r) + d0));
                        acc.x += v.x;
                        acc.y += v.y;
                        acc.z += v.z;
                        acc.w += v.w;
                    }
                    s_base[d0] = s_gbase[d0] + acc.x;
                    s_base[d0 + 1] = s_gbase[d0 + 1] + acc.y;
                    s_base[d0 + 2] = s_gbase[d0 + 2] + acc.z;
                    s_base[d0 + 3] = s_gbase[d0 + 3] + acc.w;
                }
            } else if ((unsigned)tid < nb) {
                unsigned acc = 0;
                for (unsigned r = 0; r < nrows; ++r) acc += row_of(r)[tid];
                s_base[tid] = s_gbase[tid] + acc;
            }
        }

        if (groups && count <= (unsigned)kSortTile) {
            // ---- short group: staged in shared memory by all threads, then one
            // warp ranks the pairs in input order, 32 at a time, against running
            // per-digit counters (no per-warp tables). Position tiles are full
            // (all but the last) and take the 8-warp path below.
            uint32_t* s_key = &s_whist[0][0];
            uint32_t* s_val = &s_whist[4][0];
            for (unsigned i = tid; i < count; i += kSortThreads) {
                s_key[i] = a.keys_in[first + i];
                s_val[i] = a.vals_in[first + i];
            }
            __syncthreads();  // s_base and the staged pairs complete
            if (warp == 0) {
                for (unsigned r0 = 0; r0 < count; r0 += 32) {
                    const unsigned idx = r0 + lane;
                    const bool valid = idx < count;
                    const uint32_t key = valid ? s_key[idx] : 0xffffffffu;
                    const uint32_t val = valid ? s_val[idx] : 0u;
                    const unsigned d = valid ? ((key >> a.shift) & mask) : 0xffffffffu;
                    const unsigned peers = __match_any_sync(0xffffffffu, d);
                    unsigned base = 0;
                    if (valid) base = s_base[d];
                    __syncwarp();
                    if (valid && (__ffs(peers) - 1) == lane) s_base[d] = base + __popc(peers);
                    __syncwarp();
                    if (valid) {
                        const unsigned pos = base + __popc(peers & lanemask_lt());
                        a.keys_out[pos] = key;
                        a.vals_out[pos] = val;
                        if (a.tile_hist_next) {
                            const unsigned nd = (key >> (a.shift + a.bits)) & (a.next_buckets - 1);
                            sort_count(a.tile_hist_next, a.sort_tiles_cap, a.next_buckets, pos / tile_keys, nd, 1u);
                        }
                    }
                }
            }
        } else {
        // ---- long tile: rounds of kSortTile pairs, in input order ----------------
        for (unsigned r0 = 0; r0 < count; r0 += kSortTile) {
            for (int w = 0; w < 8; ++w)
                for (unsigned d = tid; d < nb; d += kSortThreads) s_whist[w][d] = 0;
            __syncthreads();
            // rank: warp-local stable ranks via match_any
            uint32_t key[kSortItems], val[kSortItems];
            unsigned rank[kSortItems];
            const unsigned seg = r0 + warp * (kSortItems * 32);
            const unsigned lim = min(count - r0, (unsigned)kSortTile) + r0;
#pragma unroll
            for (int r = 0; r < kSortItems; ++r) {  // all loads in flight before the ranking
                const unsigned idx = seg + r * 32 + lane;
                const bool valid = idx < lim;
                key[r] = valid ? __ldcs(a.keys_in + first + idx) : 0xffffffffu;
                val[r] = valid ? __ldcs(a.vals_in + first + idx) : 0u;
            }
#pragma unroll
            for (int r = 0; r < kSortItems; ++r) {
                const unsigned idx = seg + r * 32 + lane;
                const bool valid = idx < lim;
                const unsigned d = valid ? ((key[r] >> a.shift) & mask) : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                unsigned prior = 0;
                if (valid) prior = s_whist[warp][d];
                __syncwarp();
                if (valid && (__ffs(peers) - 1) == lane) s_whist[warp][d] = prior + __popc(peers);
                __syncwarp();
                rank[r] = prior + __popc(peers & lanemask_lt());
            }
            __syncthreads();
            if (!staged) {
                // wide digits (runs of ~2 pairs per digit per round): per digit,
                // exclusive prefix over warps on top of the running base, then
                // scatter directly
                for (unsigned d = tid; d < nb; d += kSortThreads) {
                    unsigned base = s_base[d];
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        const unsigned c = s_whist[w][d];
                        s_whist[w][d] = base;
                        base += c;
                    }
                    s_base[d] = base;  // the next round of this tile continues here
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < kSortItems; ++r)
                    if (seg + r * 32 + lane < lim) {
                        const unsigned p = s_whist[warp][(key[r] >> a.shift) & mask] + rank[r];
                        a.keys_out[p] = key[r];
                        a.vals_out[p] = val[r];
                        if (a.tile_hist_next) {
                            const unsigned nd = (key[r] >> (a.shift + a.bits)) & (a.next_buckets - 1);
                            sort_count(a.tile_hist_next, a.sort_tiles_cap, a.next_buckets, p / tile_keys, nd, 1u);
                        }
                    }
                __syncthreads();
                continue;
            }
            // per digit (4 consecutive per thread): exclusive prefix over warps on
            // top of the running base; the round's digit counts, scanned over the
            // digits, give each pair its slot in a digit-major staging order
            {
                const unsigned d0 = tid * 4;
                unsigned cnt[4], tot = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned d = d0 + q;
                    cnt[q] = 0;
                    if (d < nb) {
                        unsigned base = s_base[d];
                        const unsigned b0 = base;
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            const unsigned c = s_whist[w][d];
                            s_whist[w][d] = base;
                            base += c;
                        }
                        s_base[d] = base;  // the next round of this tile continues here
                        cnt[q] = base - b0;
                    }
                    tot += cnt[q];
                }
                unsigned incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                if (lane == 31) s_wsum[warp] = incl;
                __syncthreads();
                unsigned loc = incl - tot;
                for (int w = 0; w < warp; ++w) loc += s_wsum[w];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned d = d0 + q;
                    // output position = staging slot + delta (mod 2^32)
                    if (d < nb) s_delta[d] = (s_base[d] - cnt[q]) - loc;
                    loc += cnt[q];
                }
            }
            __syncthreads();
            unsigned pos[kSortItems];
#pragma unroll
            for (int r = 0; r < kSortItems; ++r) {
                const unsigned d = (key[r] >> a.shift) & mask;
                pos[r] = (seg + r * 32 + lane < lim) ? s_whist[warp][d] + rank[r] : 0u;
            }
            __syncthreads();  // the warp rows are read; they become the staging area
            uint32_t* s_sk = &s_whist[0][0];
            uint32_t* s_sv = &s_whist[1][0];
#pragma unroll
            for (int r = 0; r < kSortItems; ++r)
                if (seg + r * 32 + lane < lim) {
                    const unsigned L = pos[r] - s_delta[(key[r] >> a.shift) & mask];
                    s_sk[L] = key[r];
                    s_sv[L] = val[r];
                }
            __syncthreads();
            // scatter from the staging order: consecutive threads write runs of
            // one digit to consecutive positions (+ next pass's per-tile counts)
            const unsigned nround = lim - r0;
            for (unsigned L = tid; L < nround; L += kSortThreads) {
                const uint32_t k = s_sk[L];
                const unsigned p = L + s_delta[(k >> a.shift) & mask];
                a.keys_out[p] = k;
                a.vals_out[p] = s_sv[L];
                if (a.tile_hist_next) {
                    const unsigned nd = (k >> (a.shift + a.bits)) & (a.next_buckets - 1);
                    sort_count(a.tile_hist_next, a.sort_tiles_cap, a.next_buckets, p / tile_keys, nd, 1u);
                }
            }
            __syncthreads();
        }
        }
        __syncthreads();  // s_base / s_wsum are rewritten for the next tile
    }
}

// Before a pass: the super rows (counts of 16 sort tiles each) become their
// exclusive prefix over the super-tiles, digit by digit (CTA per digit,
// block scan of the column), so a tile's offsets need one super row and at
// most 15 tile rows whatever the number of tiles.
constexpr int kScanThreads = 512;

__global__ void __launch_bounds__(kScanThreads) k_super_scan(unsigned* __restrict__ region, uint64_t tiles_cap,
                                                             unsigned nb, const Control* ctrl, uint64_t pair_cap,
                                                             unsigned ngroups, unsigned tile_keys) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_wsum[kScanThreads / 32];
    __shared__ unsigned s_carry;
    const unsigned d = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned P = stored_pairs(ctrl, pair_cap);
    const unsigned ntiles = ngroups ? ngroups : (P + tile_keys - 1) / tile_keys;
    const unsigned nsup = (ntiles + kSuperTiles - 1) / kSuperTiles;
    unsigned* col = region + tiles_cap * nb + d;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (unsigned s0 = 0; s0 < nsup; s0 += kScanThreads) {
        const unsigned sidx = s0 + tid;
        const unsigned v = sidx < nsup ? __ldcg(&col[(size_t)sidx * nb]) : 0u;
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        unsigned ex = s_carry + incl - v;
        for (int w = 0; w < warp; ++w) ex += s_wsum[w];
        if (sidx < nsup) col[(size_t)sidx * nb] = ex;
        __syncthreads();
        if (tid == kScanThreads - 1) s_carry = ex + v;
        __syncthreads();
    }
}

// ---- k_gather --------------------------------------------------------------------
// Single-pass slices (every tile is one digit): instead of a radix pass, one
// CTA per tile concatenates the tile's buckets — one per K_decide group, in
// group order, each filled in ascending slot order by K_decide — into the
// tile's final list: ascending slot order, like the reference's lists.
constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads) k_gather(const GatherLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_ex[kGatherThreads + 1], s_b[kGatherThreads], s_wsum[2 * kGatherThreads / 32];
    __shared__ unsigned s_range[2];
    const unsigned d = blockIdx.x;
    // the tile's pair records, in list order, built as the list is copied
    const int tx = (int)(d % (unsigned)a.slice.tiles_x), ty = (int)(d / (unsigned)a.slice.tiles_x);
    const double X0 = ((double)(tx * kTile) - a.slice.ppx) * a.slice.sx;
    const double Y0 = ((double)(ty * kTile) - a.slice.ppy) * a.slice.sy;
    auto emit = [&](unsigned pos, unsigned, uint32_t slot) {
        a.vals_out[pos] = slot;
        store_pair_record(a.pairs + pos, make_pair_record(a.records[slot], tx, ty, X0, Y0));
    };
    gather_tile_list<kGatherThreads, 1>(a.bucket_tab, a.ngroups, a.gstride, d, a.ntiles, a.tile_begin,
                                        stored_pairs(a.ctrl, a.pair_cap), a.pair_cap, a.vals_in, emit, s_ex, s_b,
                                        s_wsum, s_range);
}

// Position j of a sorted key list opens every tile in (key[j-1], key[j]]
// (key[-1] = -1, key[P] = ntiles): over j in [0, P] every start[0 .. ntiles]
// is written once. Returns key[j] (ntiles at j = P).
__device__ __forceinline__ unsigned mark_key_starts(const uint32_t* __restrict__ keys, unsigned P, unsigned ntiles,
                                                    unsigned j, unsigned* __restrict__ start) {
    const unsigned tile = j < P ? keys[j] : ntiles;
    const unsigned prev = j ? keys[j - 1] : 0xffffffffu;
    for (unsigned t = prev + 1; t <= tile; ++t) start[t] = j;
    return tile;
}

// The tile starts of a sorted key list (the voxelizer's 8^3 tiles).
__global__ void __launch_bounds__(256) k_key_starts(const uint32_t* __restrict__ keys, const Control* ctrl,
                                                    uint64_t pair_cap, unsigned ntiles, unsigned* __restrict__ start) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned P = stored_pairs(ctrl, pair_cap);
    for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j <= P; j += gridDim.x * blockDim.x)
        mark_key_starts(keys, P, ntiles, j, start);
}

// Multi-pass slices: the pair record of every sorted position (its tile is its
// key), and the tile starts: position j opens every tile in (key[j-1], key[j]]
// (key[-1] = -1, key[P] = ntiles), so the pixel kernels read their range with
// two loads instead of searching the sorted keys.
__global__ void __launch_bounds__(256) k_pair_records(const uint32_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ vals,
                                                      const SurvivorRecord* __restrict__ records,
                                                      PairRecord* __restrict__ pairs, unsigned* __restrict__ tile_start,
                                                      const Control* ctrl, uint64_t pair_cap, const SliceArgs sl) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned P = stored_pairs(ctrl, pair_cap);
    const unsigned ntiles = (unsigned)(sl.tiles_x * sl.tiles_y);
    for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j <= P; j += gridDim.x * blockDim.x) {
        const unsigned tile = mark_key_starts(keys, P, ntiles, j, tile_start);
        if (j == P) break;
        const int tx = (int)(tile % (unsigned)sl.tiles_x), ty = (int)(tile / (unsigned)sl.tiles_x);
        const double X0 = ((double)(tx * kTile) - sl.ppx) * sl.sx;
        const double Y0 = ((double)(ty * kTile) - sl.ppy) * sl.sy;
        store_pair_record(pairs + j, make_pair_record(records[vals[j]], tx, ty, X0, Y0));
    }
}

}  // namespace

void launch_gather(const GatherLaunch& a, cudaStream_t st) {
    if (a.ntiles) launch_pdl(k_gather, dim3(a.ntiles), dim3(kGatherThreads), 0, st, a);
}

void launch_pair_records(const uint32_t* keys, const uint32_t* vals, const SurvivorRecord* records, PairRecord* pairs,
                         unsigned* tile_start, const Control* ctrl, uint64_t pair_cap, const SliceArgs& slice,
                         int num_sms, cudaStream_t st) {
    launch_pdl(k_pair_records, dim3(num_sms * 8), dim3(256), 0, st, keys, vals, records, pairs, tile_start, ctrl,
               pair_cap, slice);
}

void launch_key_starts(const uint32_t* keys, const Control* ctrl, uint64_t pair_cap, unsigned ntiles,
                       unsigned* start, int num_sms, cudaStream_t st) {
    launch_pdl(k_key_starts, dim3(num_sms * 8), dim3(256), 0, st, keys, ctrl, pair_cap, ntiles, start);
}

void launch_super_scan(unsigned* region, uint64_t tiles_cap, unsigned nb, const Control* ctrl, uint64_t pair_cap,
                       unsigned ngroups, unsigned tile_keys, cudaStream_t st) {
    launch_pdl(k_super_scan, dim3(nb), dim3(kScanThreads), 0, st, region, tiles_cap, nb, ctrl, pair_cap, ngroups,
               tile_keys);
}

void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st) {
    launch_pdl(k_sort_pass, dim3(grid), dim3(kSortThreads), 0, st, a);
}

}  // namespace gpk
