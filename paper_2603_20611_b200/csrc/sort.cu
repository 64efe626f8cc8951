// sort.cu — hand-written stable LSD radix sort of (tile key, candidate id)
// pairs, one onesweep pass per 8-bit digit.
//
// Stability is the whole point: pairs arrive in ascending candidate id (= set
// order), so a stable sort by tile reproduces the reference's per-tile lists
// in ascending prepared index (render.hpp:151-157) bit-exactly.
//
// Per pass, one persistent grid claims 2048-key tiles in order. Inside a tile,
// warp w owns a contiguous 256-key segment processed in 8 rounds of 32; ranks
// within a round come from __match_any_sync, so the block-local order is the
// input order. Tile-to-tile offsets per digit come from a decoupled look-back
// on 64-bit status words tagged with a device-side epoch (no per-pass memset,
// graph-replay safe). Global digit offsets come from the histograms K_prep
// accumulated while emitting the pairs.
#include "common.cuh"

namespace gpk {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 30;
constexpr unsigned long long kFlagPrefix = 2ull << 30;
constexpr unsigned long long kCountMask = (1ull << 30) - 1;

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const SortLaunch a) {
    __shared__ unsigned s_whist[8][256];
    __shared__ unsigned s_digit_base[256];
    __shared__ unsigned s_tile_excl[256];
    __shared__ unsigned s_wsum[8];
    __shared__ unsigned s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned P = stored_pairs(a.ctrl_ro, a.pair_cap);
    const unsigned ntiles = (P + kSortTile - 1) / kSortTile;
    const unsigned epoch = (*a.epoch) * 4u + (unsigned)a.pass;
    const unsigned long long etag = (unsigned long long)epoch << 32;

    // exclusive scan of this pass's global digit histogram
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
        s_digit_base[tid] = incl - v + add;
    }

    while (true) {
        __syncthreads();
        if (tid == 0) s_tile = atomicAdd(&a.ctrl->sort_tile_ctr[a.pass], 1u);
#pragma unroll
        for (int w = 0; w < 8; ++w) s_whist[w][tid] = 0;
        __syncthreads();
        const unsigned t = s_tile;
        if (t >= ntiles) break;

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

        // ---- per digit: exclusive prefix over warps, tile count ------------
        unsigned count = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const unsigned c = s_whist[w][tid];
            s_whist[w][tid] = count;
            count += c;
        }

        // ---- decoupled look-back for digit `tid` ---------------------------
        unsigned long long* st = a.status + (unsigned long long)t * 256 + tid;
        unsigned excl = 0;
        if (t == 0) {
            st_release_u64(st, etag | kFlagPrefix | count);
        } else {
            st_release_u64(st, etag | kFlagAgg | count);
            long j = (long)t - 1;
            while (j >= 0) {
                const unsigned long long w =
                    ld_acquire_u64(a.status + (unsigned long long)j * 256 + tid);
                if ((w & 0xffffffff00000000ull) != etag || (w & (3ull << 30)) == 0) continue;
                excl += (unsigned)(w & kCountMask);
                if (w & kFlagPrefix) break;
                --j;
            }
            st_release_u64(st, etag | kFlagPrefix | (excl + count));
        }
        s_tile_excl[tid] = excl;
        __syncthreads();

        // ---- scatter -------------------------------------------------------
#pragma unroll
        for (int r = 0; r < kSortItems; ++r) {
            const unsigned idx = seg + r * 32 + lane;
            if (idx < P) {
                const unsigned d = (key[r] >> a.shift) & 255u;
                const unsigned pos = s_digit_base[d] + s_tile_excl[d] + s_whist[warp][d] + rank[r];
                a.keys_out[pos] = key[r];
                a.vals_out[pos] = val[r];
            }
        }
    }
}

}  // namespace

void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st) {
    k_sort_pass<<<grid, kSortThreads, 0, st>>>(a);
}

}  // namespace gpk
