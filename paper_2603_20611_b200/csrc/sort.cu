// sort.cu — hand-written stable LSD radix sort of (tile key, candidate slot)
// pairs, one kernel per 8-bit digit.
//
// Stability is the whole point: pairs arrive in ascending candidate slot
// (= set order), so a stable sort by tile reproduces the reference's per-tile
// lists in ascending prepared index (render.hpp:151-157) bit-exactly.
//
// Wait-free passes: the producer of a pass's input (K_exact for pass 0, pass p
// for pass p+1) also counts, per 2048-key sort tile, how many keys carry each
// digit value. A sort CTA therefore knows its output offsets up front —
// global digit base (exclusive scan of the global histogram) + the column sum
// of the per-tile histograms of all earlier tiles (coalesced L2 reads) — and
// never waits on another CTA. Inside a tile, warp w owns a contiguous 256-key
// segment processed in 8 rounds of 32; ranks within a round come from
// __match_any_sync, so the tile-local order is the input order.
#include "common.cuh"

namespace gpk {

namespace {

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const SortLaunch a) {
    __shared__ unsigned s_whist[8][256];
    __shared__ unsigned s_part[8][256];
    __shared__ unsigned s_dbase[256];
    __shared__ unsigned s_wsum[8];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
    const unsigned ntiles = (P + kSortTile - 1) / kSortTile;

    // global digit base: exclusive scan of this pass's histogram
    {
        const unsigned v = a.hist[tid];
        unsigned incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        unsigned add = 0;
        for (int w = 0; w < warp; ++w) add += s_wsum[w];
        s_dbase[tid] = incl - v + add;
    }
    if (blockIdx.x == 0 && tid == 0 && !a.tile_hist_next) *a.prev_sort_tiles = ntiles;

    for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // ---- offsets of earlier tiles: warp w sums rows j = w, w+8, ... < t
        {
            unsigned acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            const uint4* rows = reinterpret_cast<const uint4*>(a.tile_hist);
            for (unsigned j = warp; j < t; j += 8) {
                const uint4 x = rows[(size_t)j * 64 + lane * 2];
                const uint4 y = rows[(size_t)j * 64 + lane * 2 + 1];
                acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += x.w;
                acc[4] += y.x; acc[5] += y.y; acc[6] += y.z; acc[7] += y.w;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) s_part[warp][lane * 8 + i] = acc[i];
        }
#pragma unroll
        for (int w = 0; w < 8; ++w) s_whist[w][tid] = 0;
        __syncthreads();

        // ---- rank: warp-local stable ranks via match_any -----------------
        uint32_t key[kSortItems], val[kSortItems];
        unsigned rank[kSortItems];
        const unsigned seg = t * kSortTile + warp * (kSortItems * 32);
#pragma unroll
        for (int r = 0; r < kSortItems; ++r) {
            const unsigned idx = seg + r * 32 + lane;
            const bool valid = idx < P;
            key[r] = valid ? a.keys_in[idx] : 0xffffffffu;
            val[r] = valid ? a.vals_in[idx] : 0u;
            const unsigned d = valid ? ((key[r] >> a.shift) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            unsigned prior = 0;
            if (valid) prior = s_whist[warp][d];
            __syncwarp();
            if (valid && (__ffs(peers) - 1) == lane) s_whist[warp][d] = prior + __popc(peers);
            __syncwarp();
            rank[r] = prior + __popc(peers & lanemask_lt());
        }
        __syncthreads();

        // ---- per digit: base = global digit base + earlier tiles; warp prefixes
        {
            unsigned base = s_dbase[tid];
#pragma unroll
            for (int w = 0; w < 8; ++w) base += s_part[w][tid];
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const unsigned c = s_whist[w][tid];
                s_whist[w][tid] = base;
                base += c;
            }
        }
        __syncthreads();

        // ---- scatter (+ next pass's per-tile digit counts) ------------------
#pragma unroll
        for (int r = 0; r < kSortItems; ++r) {
            const unsigned idx = seg + r * 32 + lane;
            if (idx < P) {
                const unsigned d = (key[r] >> a.shift) & 255u;
                const unsigned pos = s_whist[warp][d] + rank[r];
                a.keys_out[pos] = key[r];
                a.vals_out[pos] = val[r];
                if (a.tile_hist_next)
                    atomicAdd(&a.tile_hist_next[(pos / kSortTile) * 256 + ((key[r] >> (a.shift + 8)) & 255u)], 1u);
            }
        }
        __syncthreads();
    }
}

}  // namespace

void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st) {
    k_sort_pass<<<grid, kSortThreads, 0, st>>>(a);
}

}  // namespace gpk
