// raster.cu — per-tile pixel accumulation kernels (forward and backward).
//
// Forward replaces rasterize_prepared (render.hpp:166-192):
//   one CTA per 16x16 tile, one thread per pixel, warps own 8x4 pixel blocks.
//   Survivor records of the tile's list are staged through shared memory in
//   batches of 256 (one gather per thread; the records are L2-resident), each
//   converted to tile-local fp32 offsets from its fp64 centre (SURVEY.md
//   §7.3.3: absolute fp32 pixel coordinates lose 3.6e-4 at 2048^2). Each warp
//   ballots which of 32 records touch its 8x4 block and walks only those, in
//   list order — so every pixel sums its Gaussians in ascending set order like
//   the reference, deterministically. exp runs on MUFU.EX2 with the -1/2*log2(e)
//   factor folded into the conic.
//
// Backward replaces stage 1 of backward_prepared (backward.hpp:108-139):
//   per tile, batches of 64 (tile, Gaussian) pairs are split into row items
//   (one row of the pair's tile-clipped footprint each, <= 16 pixels), spread
//   over 256 threads for balance; row sums land in shared memory and are
//   reduced per pair in row order, then written to the pair's PRE-SORT
//   position, so K_chain can merge a Gaussian's tiles in tile order
//   (backward.hpp:141-145) without atomics: bitwise reproducible.
#include "common.cuh"

namespace gpk {

namespace {

constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// First index in keys[0, n) whose value is >= target (keys sorted), one warp.
__device__ __forceinline__ unsigned warp_lower_bound(const uint32_t* __restrict__ keys, unsigned n,
                                                     unsigned target) {
    const int lane = threadIdx.x & 31;
    unsigned lo = 0, hi = n;  // answer in [lo, hi]
    while (hi - lo > 32) {
        const unsigned span = hi - lo;
        const unsigned pos = lo + (unsigned)(((unsigned long long)span * (lane + 1)) / 32) - 1;
        const bool less = keys[pos] < target;
        const unsigned m = __ballot_sync(0xffffffffu, less);
        const int c = __popc(m);  // probes are monotone: lanes [0, c) are < target
        const unsigned new_lo = c ? (lo + (unsigned)(((unsigned long long)span * c) / 32)) : lo;
        const unsigned new_hi =
            (c < 32) ? (lo + (unsigned)(((unsigned long long)span * (c + 1)) / 32) - 1) : hi;
        lo = new_lo;
        hi = new_hi;
    }
    const unsigned pos = lo + lane;
    const bool less = pos < hi && keys[pos] < target;
    return lo + __popc(__ballot_sync(0xffffffffu, less));
}

__device__ __forceinline__ unsigned clip_rect(const SurvivorRecord& r, int x0, int y0) {
    const int cx0 = max((int)r.lo_x - x0, 0), cx1 = min((int)r.hi_x - x0, kTile - 1);
    const int cy0 = max((int)r.lo_y - y0, 0), cy1 = min((int)r.hi_y - y0, kTile - 1);
    return (unsigned)cx0 | ((unsigned)cx1 << 8) | ((unsigned)cy0 << 16) | ((unsigned)cy1 << 24);
}

__global__ void __launch_bounds__(256) k_raster_fwd(const RasterLaunch a) {
    __shared__ float4 s_r0[256];  // ox, oy, a*k, 2b*k
    __shared__ float4 s_r1[256];  // d*k, alpha_tilde, rect bits, -
    __shared__ unsigned s_range[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % a.slice.tiles_x, ty = tile / a.slice.tiles_x;
    const int x0 = tx * kTile, y0 = ty * kTile;
    const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
    if (warp < 2) {
        const unsigned r = warp_lower_bound(a.keys, P, (unsigned)tile + warp);
        if (lane == 0) s_range[warp] = r;
    }
    // pixel of this thread: warp w -> 8x4 block
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;
    const int lx = wx0 + (lane & 7), ly = wy0 + (lane >> 3);
    const double X0 = ((double)x0 - a.slice.ppx) * a.slice.sx;
    const double Y0 = ((double)y0 - a.slice.ppy) * a.slice.sy;
    const float fx = (float)(lx * a.slice.sx), fy = (float)(ly * a.slice.sy);
    __syncthreads();
    const unsigned start = s_range[0], end = s_range[1];

    float acc = 0.f;
    for (unsigned b = start; b < end; b += 256) {
        const unsigned nb = min(256u, end - b);
        __syncthreads();
        if (tid < nb) {
            const SurvivorRecord r = a.records[a.vals[b + tid]];
            const float ox = (float)(r.mu2d_x - X0), oy = (float)(r.mu2d_y - Y0);
            s_r0[tid] = make_float4(ox, oy, r.conic_a * kNegHalfLog2e,
                                    2.f * r.conic_b * kNegHalfLog2e);
            s_r1[tid] = make_float4(r.conic_d * kNegHalfLog2e, r.alpha_tilde,
                                    __uint_as_float(clip_rect(r, x0, y0)), 0.f);
        }
        __syncthreads();
        for (unsigned g = 0; g < nb; g += 32) {
            bool hit = false;
            if (g + lane < nb) {
                const unsigned rc = __float_as_uint(s_r1[g + lane].z);
                const int cx0 = rc & 255, cx1 = (rc >> 8) & 255, cy0 = (rc >> 16) & 255, cy1 = rc >> 24;
                hit = cx0 <= wx0 + 7 && cx1 >= wx0 && cy0 <= wy0 + 3 && cy1 >= wy0;
            }
            unsigned m = __ballot_sync(0xffffffffu, hit);
            while (m) {
                const int k = __ffs(m) - 1;
                m &= m - 1;
                const float4 r0 = s_r0[g + k];
                const float4 r1 = s_r1[g + k];
                const unsigned rc = __float_as_uint(r1.z);
                const int cx0 = rc & 255, cx1 = (rc >> 8) & 255, cy0 = (rc >> 16) & 255, cy1 = rc >> 24;
                const bool inside = lx >= cx0 && lx <= cx1 && ly >= cy0 && ly <= cy1;
                const float dx = fx - r0.x, dy = fy - r0.y;
                const float e = fmaf(r0.z * dx, dx, fmaf(r0.w * dx, dy, r1.x * dy * dy));
                const float v = r1.y * ex2_approx(e);
                acc += inside ? v : 0.f;
            }
        }
    }
    const int i = x0 + lx, j = y0 + ly;
    if (i < a.slice.W && j < a.slice.H) a.image[(size_t)j * a.slice.W + i] = acc;
}

constexpr int kBwdBatch = 64;

__global__ void __launch_bounds__(256) k_raster_bwd(const RasterLaunch a) {
    __shared__ float s_dl[kTile * kTile];
    __shared__ float4 s_p0[kBwdBatch];       // ox, oy, conic a, conic b
    __shared__ float4 s_p1[kBwdBatch];       // conic d, alpha_tilde, rect bits, -
    __shared__ unsigned s_pos[kBwdBatch];    // output pair position
    __shared__ unsigned s_roff[kBwdBatch + 1];
    __shared__ uint16_t s_item[kBwdBatch * kTile];
    __shared__ float s_part[6][kBwdBatch * kTile];
    __shared__ unsigned s_range[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % a.slice.tiles_x, ty = tile / a.slice.tiles_x;
    const int x0 = tx * kTile, y0 = ty * kTile;
    const unsigned P = stored_pairs(a.ctrl, a.pair_cap);
    if (warp < 2) {
        const unsigned r = warp_lower_bound(a.keys, P, (unsigned)tile + warp);
        if (lane == 0) s_range[warp] = r;
    }
    {
        const int i = x0 + (tid & 15), j = y0 + (tid >> 4);
        s_dl[tid] = (i < a.slice.W && j < a.slice.H) ? a.dl_di[(size_t)j * a.slice.W + i] : 0.f;
    }
    const double X0 = ((double)x0 - a.slice.ppx) * a.slice.sx;
    const double Y0 = ((double)y0 - a.slice.ppy) * a.slice.sy;
    const float sxf = (float)a.slice.sx, syf = (float)a.slice.sy;
    __syncthreads();
    const unsigned start = s_range[0], end = s_range[1];

    for (unsigned b = start; b < end; b += kBwdBatch) {
        const unsigned nb = min((unsigned)kBwdBatch, end - b);
        __syncthreads();
        unsigned nrows = 0;
        if (tid < nb) {
            const SurvivorRecord r = a.records[a.vals[b + tid]];
            const unsigned rc = clip_rect(r, x0, y0);
            s_p0[tid] = make_float4((float)(r.mu2d_x - X0), (float)(r.mu2d_y - Y0), r.conic_a,
                                    r.conic_b);
            s_p1[tid] = make_float4(r.conic_d, r.alpha_tilde, __uint_as_float(rc), 0.f);
            const int ntx = r.hi_x / kTile - r.lo_x / kTile + 1;
            const int li = (ty - r.lo_y / kTile) * ntx + (tx - r.lo_x / kTile);
            s_pos[tid] = r.pair_base + (unsigned)li;
            nrows = ((rc >> 24) - ((rc >> 16) & 255)) + 1;
        }
        // exclusive scan of nrows over the batch (threads 0..63 = warps 0,1)
        if (warp < 2) {
            unsigned incl = nrows;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            s_roff[tid + 1] = incl;  // per-warp inclusive, fixed below
        }
        __syncthreads();
        if (tid >= 32 && tid < 64) s_roff[tid + 1] += s_roff[32];
        if (tid == 0) s_roff[0] = 0;
        __syncthreads();
        if (tid < nb) {
            const unsigned o = s_roff[tid];
            for (unsigned r = 0; r < nrows; ++r) s_item[o + r] = (uint16_t)((tid << 4) | r);
        }
        __syncthreads();
        const unsigned nitems = s_roff[nb];
        for (unsigned it = tid; it < nitems; it += 256) {
            const unsigned k = s_item[it] >> 4, r = s_item[it] & 15u;
            const float4 p0 = s_p0[k], p1 = s_p1[k];
            const unsigned rc = __float_as_uint(p1.z);
            const int cx0 = rc & 255, cx1 = (rc >> 8) & 255, cy0 = (rc >> 16) & 255;
            const int y = cy0 + (int)r;
            const float dy = (float)y * syf - p0.y;
            float a_t = 0.f, gmx = 0.f, gmy = 0.f, cxx = 0.f, cxy = 0.f, cyy = 0.f;
            for (int x = cx0; x <= cx1; ++x) {
                const float gi = s_dl[y * kTile + x];
                if (gi == 0.f) continue;  // backward.hpp:125
                const float dx = (float)x * sxf - p0.x;
                const float cdx = p0.z * dx + p0.w * dy;
                const float cdy = p0.w * dx + p1.x * dy;
                const float g = ex2_approx(kNegHalfLog2e * (dx * cdx + dy * cdy));
                a_t += gi * g;
                const float w = p1.y * g * gi;
                gmx += cdx * w;
                gmy += cdy * w;
                const float hw = -0.5f * w;
                cxx += hw * dx * dx;
                cxy += hw * dx * dy;
                cyy += hw * dy * dy;
            }
            s_part[0][it] = a_t;
            s_part[1][it] = gmx;
            s_part[2][it] = gmy;
            s_part[3][it] = cxx;
            s_part[4][it] = cxy;
            s_part[5][it] = cyy;
        }
        __syncthreads();
        if (tid < nb) {
            float o[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (unsigned it = s_roff[tid]; it < s_roff[tid + 1]; ++it) {
#pragma unroll
                for (int q = 0; q < 6; ++q) o[q] += s_part[q][it];
            }
            const unsigned pos = s_pos[tid];
            if (pos < a.pair_cap) {
                float2* dst = reinterpret_cast<float2*>(a.partials + 6ull * pos);
                dst[0] = make_float2(o[0], o[1]);
                dst[1] = make_float2(o[2], o[3]);
                dst[2] = make_float2(o[4], o[5]);
            }
        }
    }
}

}  // namespace

void launch_raster_fwd(const RasterLaunch& a, cudaStream_t st) {
    const int tiles = a.slice.tiles_x * a.slice.tiles_y;
    if (tiles > 0) k_raster_fwd<<<tiles, 256, 0, st>>>(a);
}

void launch_raster_bwd(const RasterLaunch& a, cudaStream_t st) {
    const int tiles = a.slice.tiles_x * a.slice.tiles_y;
    if (tiles > 0) k_raster_bwd<<<tiles, 256, 0, st>>>(a);
}

}  // namespace gpk
