// raster.cu — per-tile pixel accumulation kernels (forward and backward).
//
// Forward replaces rasterize_prepared (render.hpp:166-192):
//   one CTA of 128 threads per 16x16 tile; warp w owns the tile rows
//   [4w, 4w + 4), each lane two horizontally adjacent pixels of one row.
//   The tile's pairs are one contiguous run of 32 B PairRecords (tile-local
//   fp32 centre from the fp64 mean — SURVEY.md §7.3.3: absolute fp32 pixel
//   coordinates lose 3.6e-4 at 2048^2 — scaled conic, alpha_tilde, the bit
//   mask of covered tile rows/columns, the pair's partials position), written
//   by the gather; the forward stages them into shared memory in batches of
//   256 with double-buffered cp.async.bulk (TMA) copies on an mbarrier. In the
//   training step the forward builds its own tile's list and records (the
//   gather fused in), stages them directly and stores them for the backward.
//   Each warp ballots which of 32 records touch its rows and walks only
//   those, in list order —
//   every pixel sums its Gaussians in ascending set order like the reference,
//   deterministically; a lane shares a record's row terms between its two
//   pixels. exp runs on MUFU.EX2 with the -1/2*log2(e) factor folded into the
//   conic.
//
// Backward replaces stage 1 of backward_prepared (backward.hpp:108-139):
//   the tile's PairRecords are staged into shared memory by cp.async.bulk
//   (TMA, double-buffered batches of 256), bucketed by work
//   (rows-per-lane x width, largest first) and processed one QUAD (4 lanes)
//   per pair: lane q takes rows q, q+4, ... of the tile-clipped footprint and
//   walks each row left to right. The per-pixel work is factored through the
//   linearity of the six sums: with u = dL/dI * exp(-q/2),
//     dA = sum u,  dmu = at * C * (sum u dx, sum u dy),
//     dconic = -at/2 * (sum u dx^2, sum u dx dy, sum u dy^2),
//   and within a row dy is constant, so a pixel costs 3 FMA for the exponent,
//   one MUFU.EX2 and 5 FMA/FADD for the sums. The quad's sums are combined by
//   a fixed xor-shuffle tree and written to the pair's PRE-SORT position, so
//   K_chain merges a Gaussian's tiles in tile order (backward.hpp:141-145):
//   bitwise reproducible run to run, no float atomics.
#include "common.cuh"

namespace gpk {

namespace {

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// [begin, end) of the tile's pairs in the sorted list: the tile starts (the
// single-pass gather's, or k_pair_records' after radix passes).
__device__ __forceinline__ void tile_range(const RasterLaunch& a, int tile, unsigned* s_range) {
    if (a.grp_shift < 0) {  // no sort pass: a single tile
        if (threadIdx.x == 0) {
            s_range[0] = 0;
            s_range[1] = stored_pairs(a.ctrl, a.pair_cap);
        }
        return;
    }
    if (threadIdx.x < 2) s_range[threadIdx.x] = __ldcg(&a.grp_begin[tile + threadIdx.x]);
}

// Double-buffered TMA staging of a tile's PairRecords: batch q of [start, end)
// goes to buffer q & 1; one elected thread arms the buffer's mbarrier with
// the batch's bytes and issues one bulk copy. Callers wait with pair_wait and
// re-arm a buffer only after a CTA barrier (every warp done reading it).
constexpr int kPairBatch = 256;

struct PairStage {
    PairRecord (*buf)[kPairBatch];
    uint64_t* bar;
    unsigned start, end;
};

__device__ __forceinline__ void pair_issue(const PairStage& ps, const PairRecord* pairs, unsigned q) {
    const unsigned b = ps.start + q * kPairBatch;
    if (b >= ps.end) return;
    const unsigned nb = min((unsigned)kPairBatch, ps.end - b);
    mbar_expect_tx(&ps.bar[q & 1], nb * (unsigned)sizeof(PairRecord));
    bulk_g2s(ps.buf[q & 1], pairs + b, nb * (unsigned)sizeof(PairRecord), &ps.bar[q & 1]);
}

__device__ __forceinline__ void pair_wait(const PairStage& ps, unsigned q) { mbar_wait(&ps.bar[q & 1], (q >> 1) & 1); }

// Forward: 128 threads per tile, warp w owns the tile's rows [4w, 4w + 4),
// lane l the horizontally adjacent pixels (2 (l mod 8) + {0, 1}, 4w + l / 8).
// A record is walked by the warps whose rows it covers; per record a lane
// shares the row terms (dy, kb2 dy, kd dy^2) between its two pixels. Every
// pixel sums the records that cover it in list order (ascending set index,
// like the reference) with exactly the per-pixel arithmetic of one pixel per
// thread: the image is the same bits.
constexpr int kFwdThreads = 128;

__device__ __forceinline__ void fwd_batch(const PairRecord* recs, unsigned nb, unsigned warp_y, unsigned ybit,
                                          unsigned xb0, unsigned xb1, f32x2 fx01, float fy, f32x2& acc) {
    const int lane = threadIdx.x & 31;
    const float4* s4 = reinterpret_cast<const float4*>(recs);
    for (unsigned g = 0; g < nb; g += 32) {
        const bool hit = g + lane < nb && (recs[g + lane].rect & warp_y);
        unsigned m = __ballot_sync(0xffffffffu, hit);
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const float4 r0 = s4[2 * (g + k)];  // {ox, oy, ka, kb2}
            const float4 r1 = s4[2 * (g + k) + 1];  // {kd, at, mask, pos}
            const unsigned mask = __float_as_uint(r1.z);
            const float dy = fy - r0.y;
            const float B = r0.w * dy, Cc = r1.x * dy * dy;
            // the lane's two pixels as packed fp32 pairs (FFMA2/FADD2: each
            // lane rounds like the scalar ops, the same bits)
            const f32x2 dx = ffma2(f2(1.f, 1.f), fx01, f2(-r0.x, -r0.x));
            const float2 e = f2_unpack(ffma2(dx, ffma2(f2(r0.z, r0.z), dx, f2(B, B)), f2(Cc, Cc)));
            const bool iny = (mask & ybit) != 0;
            const float2 w = make_float2(iny && (mask & xb0) ? r1.y : 0.f, iny && (mask & xb1) ? r1.y : 0.f);
            acc = ffma2(f2(w), f2(ex2_approx(e.x), ex2_approx(e.y)), acc);
        }
    }
}

__global__ void __launch_bounds__(kFwdThreads) k_raster_fwd(const RasterLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ __align__(128) PairRecord s_pr[2][kPairBatch];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ unsigned s_range[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // 2-D grid (tiles_x, tiles_y): no per-thread division for the tile coordinates
    const int tx = blockIdx.x, ty = blockIdx.y, tile = ty * a.slice.tiles_x + tx;
    const bool produce = a.bucket_tab != nullptr;
    const int x0 = tx * kTile, y0 = ty * kTile;
    const double X0 = ((double)x0 - a.slice.ppx) * a.slice.sx;
    const double Y0 = ((double)y0 - a.slice.ppy) * a.slice.sy;
    if (produce) {
        // the training step's forward gathers its own tile's list (k_gather's
        // work, 256 groups per chunk) and builds each position's PairRecord as
        // it is copied: into the first staging batch when it falls there, and
        // to global memory for the backward (and this kernel's later batches)
        __shared__ unsigned s_ex[kFwdThreads * 2 + 1], s_b[kFwdThreads * 2], s_wsum[2 * kFwdThreads / 32];
        auto emit = [&](unsigned pos, unsigned idx, uint32_t slot) {
            a.vals_out[pos] = slot;
            const PairRecord pr = make_pair_record(a.records[slot], tx, ty, X0, Y0);
            if (idx < kPairBatch) store_pair_record(&s_pr[0][idx], pr);
            store_pair_record(a.pairs + pos, pr);
        };
        gather_tile_list<kFwdThreads, 2>(a.bucket_tab, a.ngroups, a.gstride, (unsigned)tile,
                                         (unsigned)(a.slice.tiles_x * a.slice.tiles_y),
                                         const_cast<unsigned*>(a.grp_begin), stored_pairs(a.ctrl, a.pair_cap),
                                         a.pair_cap, a.vals_in, emit, s_ex, s_b, s_wsum, s_range);
    } else {
        tile_range(a, tile, s_range);
    }
    if (!produce && tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    const int lx = 2 * (lane & 7), ly = warp * 4 + (lane >> 3);
    const unsigned ybit = 1u << (16 + ly), xb0 = 1u << lx, xb1 = 2u << lx;
    const unsigned warp_y = 0xfu << (16 + warp * 4);
    const float fx0 = (float)(lx * a.slice.sx), fx1 = (float)((lx + 1) * a.slice.sx);
    const float fy = (float)(ly * a.slice.sy);
    __syncthreads();
    const PairStage ps{s_pr, s_bar, s_range[0], s_range[1]};
    const unsigned nbatch = (ps.end - ps.start + kPairBatch - 1) / kPairBatch;

    const f32x2 fx01 = f2(fx0, fx1);
    f32x2 acc = f2(0.f, 0.f);
    if (produce) {
        // batch 0 was staged by the gather; later batches (tiles of more than
        // kPairBatch pairs) come back from the records this CTA just stored
        for (unsigned q = 0; q < nbatch; ++q) {
            const unsigned b = ps.start + q * kPairBatch, nb = min((unsigned)kPairBatch, ps.end - b);
            if (q > 0) {
                for (unsigned t = tid; t < 2 * nb; t += kFwdThreads)
                    reinterpret_cast<float4*>(s_pr[0])[t] = __ldcg(reinterpret_cast<const float4*>(a.pairs + b) + t);
                __syncthreads();
            }
            fwd_batch(s_pr[0], nb, warp_y, ybit, xb0, xb1, fx01, fy, acc);
            __syncthreads();
        }
    } else {
        if (tid == 0) {
            pair_issue(ps, a.pairs, 0);
            pair_issue(ps, a.pairs, 1);
        }
        for (unsigned q = 0; q < nbatch; ++q) {
            const unsigned nb = min((unsigned)kPairBatch, ps.end - (ps.start + q * kPairBatch));
            pair_wait(ps, q);
            fwd_batch(s_pr[q & 1], nb, warp_y, ybit, xb0, xb1, fx01, fy, acc);
            if (q + 2 < nbatch) {
                __syncthreads();  // buffer q & 1 read by every warp
                if (tid == 0) pair_issue(ps, a.pairs, q + 2);
            }
        }
    }
    const int i = x0 + lx, j = y0 + ly;
    const float acc0 = f2_unpack(acc).x, acc1 = f2_unpack(acc).y;
    if (j < a.slice.H) {
        float* row = a.image + (size_t)j * a.slice.W;
        if (i < a.slice.W) row[i] = acc0;
        if (i + 1 < a.slice.W) row[i + 1] = acc1;
    }
}

// Training step: dL/dI of the tile from k_ssim_fwd's three partial planes
// (metrics.hpp:218-223: the window is self-adjoint, dSSIM/dI = W g1 + 2 I W g2
// + T W g3) plus the L1 sign term (loss.hpp:29-33) — the work of k_ssim_bwd,
// done here so it costs no kernel of its own. Reflected borders (metrics.hpp:
// 77-83); the tile's dL/dI is also stored (GPK_BUF_DL_DI stays meaningful).
constexpr int kSsimR = 5, kSsimH = kTile + 2 * kSsimR;

__device__ __forceinline__ int reflect_idx(int p, int n) {
    while (p < 0 || p >= n) {
        if (p < 0) p = -p - 1;
        if (p >= n) p = 2 * n - 1 - p;
    }
    return p;
}

__device__ __forceinline__ void ssim_dl_tile(const RasterLaunch& a, int x0, int y0, float* s_dl) {
    __shared__ float s_g[3][kSsimH][kSsimH + 1];
    __shared__ float s_h[3][kSsimH][kTile + 1];
    const int W = a.slice.W, H = a.slice.H;
    const size_t P = (size_t)W * H;
    float px = 0.f, py = 0.f;  // this thread's pixel, requested first
    {
        const int pi = x0 + (threadIdx.x & 15), pj = y0 + (threadIdx.x >> 4);
        if (pi < W && pj < H) {
            px = a.image[(size_t)pj * W + pi];
            py = a.target[(size_t)pj * W + pi];
        }
    }
    {
        // all loads of the haloed g planes in flight at once, then to shared;
        // an interior tile's halo needs no reflection (the common case at large
        // slices): one uniform branch per CTA, row r of the halo at g + r * W
        constexpr int kPer = (kSsimH * kSsimH + 255) / 256;
        constexpr int kPlane = kSsimH * (kSsimH + 1);
        float v[3][kPer];
        int soff[kPer];  // r * (kSsimH + 1) + c = idx + r
        const bool inner = x0 >= kSsimR && y0 >= kSsimR && x0 + kTile + kSsimR <= W && y0 + kTile + kSsimR <= H;
        if (inner) {
            const float* g = a.ssim_g + (size_t)(y0 - kSsimR) * W + (x0 - kSsimR);
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * 256;
                const int r = idx / kSsimH;
                soff[k] = idx + r;
                if (idx < kSsimH * kSsimH) {
                    const unsigned o = (unsigned)(r * W + (idx - r * kSsimH));
                    v[0][k] = g[o];
                    v[1][k] = g[P + o];
                    v[2][k] = g[2 * P + o];
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * 256;
                const int r = idx / kSsimH;
                soff[k] = idx + r;
                if (idx < kSsimH * kSsimH) {
                    const size_t o = (size_t)reflect_idx(y0 + r - kSsimR, H) * W +
                                     reflect_idx(x0 + (idx - r * kSsimH) - kSsimR, W);
                    v[0][k] = a.ssim_g[o];
                    v[1][k] = a.ssim_g[P + o];
                    v[2][k] = a.ssim_g[2 * P + o];
                }
            }
        }
        float* sg = &s_g[0][0][0];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (threadIdx.x + k * 256 < kSsimH * kSsimH) {
                sg[soff[k]] = v[0][k];
                sg[kPlane + soff[k]] = v[1][k];
                sg[2 * kPlane + soff[k]] = v[2][k];
            }
    }
    __syncthreads();
    // rows: a thread filters 8 consecutive outputs of one plane row from 18
    // inputs held in registers (each output still sums its 11 taps in order)
    // (packed g1/g2 pairs measured slower: 47 registers, 5 CTAs/SM, or no gain
    // when capped at 40)
    if (threadIdx.x < kSsimH * 3 * 2) {
        const int r = threadIdx.x / 6, q = (threadIdx.x % 6) >> 1, c0 = (threadIdx.x & 1) * 8;
        float v[8 + 2 * kSsimR];
#pragma unroll
        for (int t = 0; t < 8 + 2 * kSsimR; ++t) v[t] = s_g[q][r][c0 + t];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            float h = 0.f;
#pragma unroll
            for (int t = 0; t < 2 * kSsimR + 1; ++t) h += a.w[t] * v[o + t];
            s_h[q][r][c0 + o] = h;
        }
    }
    __syncthreads();
    // columns: a thread filters 4 consecutive outputs of one plane column from
    // 14 inputs in registers, into s_g (free now) as A[q][row][col]
    float(*s_A)[kTile][kTile + 1] = reinterpret_cast<float(*)[kTile][kTile + 1]>(&s_g[0][0][0]);
    if (threadIdx.x < 3 * kTile * 4) {
        const int q = threadIdx.x / (kTile * 4), c = threadIdx.x % kTile, r0 = ((threadIdx.x / kTile) & 3) * 4;
        float v[4 + 2 * kSsimR];
#pragma unroll
        for (int t = 0; t < 4 + 2 * kSsimR; ++t) v[t] = s_h[q][r0 + t][c];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < 2 * kSsimR + 1; ++t) acc += a.w[t] * v[o + t];
            s_A[q][r0 + o][c] = acc;
        }
    }
    __syncthreads();
    const int r = threadIdx.x >> 4, c = threadIdx.x & 15;
    const int i = x0 + c, j = y0 + r;
    float dl = 0.f;
    if (i < W && j < H) {
        const float x = px, y = py;
        const float A0 = s_A[0][r][c], A1 = s_A[1][r][c], A2 = s_A[2][r][c];
        const size_t o = (size_t)j * W + i;
        const float gs = A0 + 2.f * x * A1 + y * A2;
        const float d = x - y;
        dl = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * a.inv_n + a.ssim_k * (-gs);
        const_cast<float*>(a.dl_di)[o] = dl;
    }
    s_dl[threadIdx.x] = dl;
}

constexpr int kWorkBuckets = 16;

__global__ void __launch_bounds__(256) k_raster_bwd(const RasterLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ __align__(128) PairRecord s_pr[2][kPairBatch];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ float s_dl[kTile * kTile];
    __shared__ unsigned s_bucket[kWorkBuckets];
    __shared__ uint8_t s_order[kPairBatch];
    __shared__ unsigned s_range[2];

    const int tid = threadIdx.x;
    const int tx = blockIdx.x, ty = blockIdx.y, tile = ty * a.slice.tiles_x + tx;  // 2-D grid
    if (a.fin.partial && tile == 0) {  // the training step's loss (k_ssim_fwd's partials)
        __shared__ double s_red[2 * 32];
        loss_reduce(a.fin, s_red);
    }
    const int x0 = tx * kTile, y0 = ty * kTile;
    tile_range(a, tile, s_range);
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const PairStage ps{s_pr, s_bar, s_range[0], s_range[1]};
    const unsigned nbatch = (ps.end - ps.start + kPairBatch - 1) / kPairBatch;
    if (tid == 0) {  // the first records land while dL/dI is formed
        pair_issue(ps, a.pairs, 0);
        pair_issue(ps, a.pairs, 1);
    }
    if (a.ssim_g) {
        ssim_dl_tile(a, x0, y0, s_dl);
    } else {
        const int i = x0 + (tid & 15), j = y0 + (tid >> 4);
        s_dl[tid] = (i < a.slice.W && j < a.slice.H) ? __ldg(&a.dl_di[(size_t)j * a.slice.W + i]) : 0.f;
    }
    const float sxf = (float)a.slice.sx, syf = (float)a.slice.sy;
    constexpr float kInvK = 1.f / kNegHalfLog2e;

    for (unsigned q = 0; q < nbatch; ++q) {
        const unsigned nb = min((unsigned)kPairBatch, ps.end - (ps.start + q * kPairBatch));
        const PairRecord* recs = s_pr[q & 1];
        if (tid < kWorkBuckets) s_bucket[tid] = 0;
        pair_wait(ps, q);
        __syncthreads();  // buckets cleared; s_dl complete (first batch)
        // ---- the batch's pairs bucketed by per-lane work (largest first) -------
        unsigned slot = 0xffffffffu;
        if ((unsigned)tid < nb) {
            const unsigned m = recs[tid].rect;
            const unsigned xm = m & 0xffffu, ym = m >> 16;
            const unsigned w = (31 - __clz(xm)) - (__ffs(xm) - 1) + 1, h = (31 - __clz(ym)) - (__ffs(ym) - 1) + 1;
            const unsigned work = ((h + 3) >> 2) * w;  // rows per lane x row length, <= 64
            const unsigned bk = (kWorkBuckets - 1) - min(work >> 2, (unsigned)kWorkBuckets - 1);
            slot = (bk << 16) | atomicAdd(&s_bucket[bk], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            const unsigned v = tid < kWorkBuckets ? s_bucket[tid] : 0u;
            unsigned incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += u;
            }
            if (tid < kWorkBuckets) s_bucket[tid] = incl - v;
        }
        __syncthreads();
        if (slot != 0xffffffffu) s_order[s_bucket[slot >> 16] + (slot & 0xffffu)] = (uint8_t)tid;
        __syncthreads();

        // ---- one quad per pair ------------------------------------------------
        const int quad = tid >> 2, ql = tid & 3;
        const float4* s4 = reinterpret_cast<const float4*>(recs);
        for (unsigned o0 = 0; o0 < nb; o0 += kPairBatch / 4) {
            const unsigned o = o0 + quad;
            const bool active = o < nb;  // quads are whole: all 4 lanes agree
            float U = 0.f, UX = 0.f, UY = 0.f, UXX = 0.f, UXY = 0.f, UYY = 0.f;
            float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;  // {ox, oy, ka, kb2}, {kd, at, mask, pos}
            if (active) {
                const unsigned k = s_order[o];
                p0 = s4[2 * k];
                p1 = s4[2 * k + 1];
                const unsigned m = __float_as_uint(p1.z), xm = m & 0xffffu, ym = m >> 16;
                const int cx0 = __ffs(xm) - 1, cx1 = 31 - __clz(xm), cy0 = __ffs(ym) - 1, cy1 = 31 - __clz(ym);
                const float ka = p0.z, kb2 = p0.w, kd = p1.x;
                for (int y = cy0 + ql; y <= cy1; y += 4) {
                    const float dy = fmaf((float)y, syf, -p0.y);
                    const float B = kb2 * dy, Cc = kd * dy * dy;
                    const float* row = s_dl + y * kTile;
                    float ru = 0.f, rux = 0.f, ruxx = 0.f;
#pragma unroll 4
                    for (int x = cx0; x <= cx1; ++x) {
                        const float dx = fmaf((float)x, sxf, -p0.x);
                        const float u = row[x] * ex2_approx(fmaf(dx, fmaf(ka, dx, B), Cc));
                        ru += u;
                        const float ux = u * dx;
                        rux += ux;
                        ruxx = fmaf(ux, dx, ruxx);
                    }
                    U += ru;
                    UX += rux;
                    UXX += ruxx;
                    UY = fmaf(dy, ru, UY);
                    UXY = fmaf(dy, rux, UXY);
                    UYY = fmaf(dy * dy, ru, UYY);
                }
            }
#pragma unroll
            for (int sh = 1; sh <= 2; sh <<= 1) {
                U += __shfl_xor_sync(0xffffffffu, U, sh);
                UX += __shfl_xor_sync(0xffffffffu, UX, sh);
                UY += __shfl_xor_sync(0xffffffffu, UY, sh);
                UXX += __shfl_xor_sync(0xffffffffu, UXX, sh);
                UXY += __shfl_xor_sync(0xffffffffu, UXY, sh);
                UYY += __shfl_xor_sync(0xffffffffu, UYY, sh);
            }
            const unsigned pos = __float_as_uint(p1.w);
            if (active && ql == 0 && pos < a.pair_cap) {
                // PixelAccum (backward.hpp:129-136): dA, dmu = w C d, dconic = -w/2 d d^T
                // (C = the stored scaled conic / (-1/2 log2 e))
                const float at = p1.y, atk = at * kInvK, h = -0.5f * at;
                float2* dst = reinterpret_cast<float2*>(a.partials + 6ull * pos);
                dst[0] = make_float2(U, atk * fmaf(p0.z, UX, 0.5f * p0.w * UY));
                dst[1] = make_float2(atk * fmaf(0.5f * p0.w, UX, p1.x * UY), h * UXX);
                dst[2] = make_float2(h * UXY, h * UYY);
            }
        }
        __syncthreads();  // buffer q & 1 and s_order consumed
        if (tid == 0 && q + 2 < nbatch) pair_issue(ps, a.pairs, q + 2);
    }
}

}  // namespace

void launch_raster_fwd(const RasterLaunch& a, cudaStream_t st) {
    if (a.slice.tiles_x > 0 && a.slice.tiles_y > 0)
        launch_pdl(k_raster_fwd, dim3(a.slice.tiles_x, a.slice.tiles_y), dim3(kFwdThreads), 0, st, a);
}

void launch_raster_bwd(const RasterLaunch& a, cudaStream_t st) {
    if (a.slice.tiles_x > 0 && a.slice.tiles_y > 0)
        launch_pdl(k_raster_bwd, dim3(a.slice.tiles_x, a.slice.tiles_y), dim3(256), 0, st, a);
}

}  // namespace gpk
