// sort.cu — hand-written stable LSD radix sort of (tile key, candidate slot)
// pairs, one kernel per digit of up to kMaxDigitBits bits (one pass for up to
// 1024 tiles = a 512x512 slice, two passes up to 2^20 tiles).
//
// Stability is the whole point: pairs arrive in ascending candidate slot
// (= set order), so a stable sort by tile reproduces the reference's per-tile
// lists in ascending prepared index (render.hpp:151-157) bit-exactly.
//
// Wait-free passes: the producer of a pass's input (K_exact for pass 0, pass p
// for pass p+1) also counts, per kSortTile-key sort tile, how many keys carry
// each digit value. A sort CTA therefore knows its output offsets up front —
// global digit base (exclusive scan of the global histogram) + the column sum
// of the per-tile histograms of all earlier tiles (coalesced L2 reads) — and
// never waits on another CTA. Inside a tile, warp w owns a contiguous segment
// processed in rounds of 32; ranks within a round come from __match_any_sync,
// so the tile-local order is the input order.
#include "common.cuh"

namespace gpk {

namespace {

__global__ void __launch_bounds__(kSortThreads) k_sort_pass(const SortLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_whist[8][kMaxBuckets];   // per-warp digit counts -> offsets
    __shared__ unsigned s_base[kMaxBuckets];       // digit base for this tile
    __shared__ unsigned s_wsum[32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
    const unsigned ntiles = (P + kSortTile - 1) / kSortTile;
    const unsigned nb = 1u << a.bits;
    const unsigned mask = nb - 1;
    if (blockIdx.x == 0 && tid == 0 && a.grp_begin) a.grp_begin[nb] = P;
    if (blockIdx.x == 0 && tid == 0 && !a.tile_hist_next) {
        a.prev_sort_words[0] = ntiles;
        a.prev_sort_words[1] = nb;
        a.prev_sort_words[2] = (unsigned)a.pass + 1;
    }
    const unsigned* super_rows = a.tile_hist + a.sort_tiles_cap * nb;

    for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // ---- global digit base: exclusive scan of the histogram (nb <= 1024)
        {
            constexpr int kPer = kMaxBuckets / kSortThreads;  // 4 digits per thread
            unsigned v[kPer], run = 0;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const unsigned d = tid * kPer + i;
                v[i] = d < nb ? a.hist[d] : 0u;
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
                s_base[d] = ex;
                // last pass: the digit groups' sorted start positions let the
                // pixel kernels find their tile's range without a search
                if (a.grp_begin && t == 0 && d < nb) a.grp_begin[d] = ex;
                ex += v[i];
            }
            for (int w = 0; w < 8; ++w)
                for (unsigned d = tid; d < nb; d += kSortThreads) s_whist[w][d] = 0;
            __syncthreads();
        }
        // ---- add the counts of all earlier tiles: whole super-tiles from the
        // super rows, then the earlier tiles of this super-tile (<= 15 rows).
        // Thread owns 4 consecutive digits (one 16 B load per row); rows are
        // unrolled so all of a thread's loads are in flight together.
        {
            const unsigned sup = t / kSuperTiles;
            const unsigned t0 = sup * kSuperTiles;
            const unsigned nrows = sup + (t - t0);  // super rows first, then tile rows
            if (nb >= 4) {
                const unsigned d0 = tid * 4;
                if (d0 < nb) {
                    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 8
                    for (unsigned r = 0; r < nrows; ++r) {
                        const unsigned* row = r < sup ? super_rows + (size_t)r * nb
                                                      : a.tile_hist + (size_t)(t0 + r - sup) * nb;
                        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(row + d0));
                        acc.x += v.x;
                        acc.y += v.y;
                        acc.z += v.z;
                        acc.w += v.w;
                    }
                    s_base[d0] += acc.x;
                    s_base[d0 + 1] += acc.y;
                    s_base[d0 + 2] += acc.z;
                    s_base[d0 + 3] += acc.w;
                }
            } else if ((unsigned)tid < nb) {
                unsigned acc = 0;
                for (unsigned r = 0; r < nrows; ++r)
                    acc += r < sup ? super_rows[(size_t)r * nb + tid] : a.tile_hist[(size_t)(t0 + r - sup) * nb + tid];
                s_base[tid] += acc;
            }
            __syncthreads();
        }

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

        // ---- per digit: exclusive prefix over warps on top of the tile base
        for (unsigned d = tid; d < nb; d += kSortThreads) {
            unsigned base = s_base[d];
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const unsigned c = s_whist[w][d];
                s_whist[w][d] = base;
                base += c;
            }
        }
        __syncthreads();

        // ---- scatter (+ next pass's per-tile digit counts) ------------------
#pragma unroll
        for (int r = 0; r < kSortItems; ++r) {
            const unsigned idx = seg + r * 32 + lane;
            if (idx < P) {
                const unsigned d = (key[r] >> a.shift) & mask;
                const unsigned pos = s_whist[warp][d] + rank[r];
                a.keys_out[pos] = key[r];
                a.vals_out[pos] = val[r];
                if (a.tile_hist_next) {
                    const unsigned nd = (key[r] >> (a.shift + a.bits)) & (a.next_buckets - 1);
                    const unsigned st = pos / kSortTile;
                    atomicAdd(&a.tile_hist_next[(size_t)st * a.next_buckets + nd], 1u);
                    atomicAdd(&a.tile_hist_next[(a.sort_tiles_cap + st / kSuperTiles) * a.next_buckets + nd], 1u);
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace

void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st) {
    launch_pdl(k_sort_pass, dim3(grid), dim3(kSortThreads), 0, st, a);
}

}  // namespace gpk
