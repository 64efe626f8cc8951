// common.cuh — device-side data layout shared by every sm_100a kernel.
//
// HBM layout of one session:
//   params  : 11 f32 SoA planes (mu xyz, log-scale xyz, quat wxyz, raw alpha),
//             plane p at params + p*cap  — the 44 B checkpoint record split
//             into coalesced planes (checkpoint.hpp:14-16).
//   grads   : same 11-plane layout, dense (exact zeros for culled primitives,
//             grad_chain.hpp:12-22).
//   records : one 48 B SurvivorRecord per candidate id. Candidate ids are
//             block-major (K_prep block b owns ids [b*1024, b*1024+count_b)) and
//             strictly increasing in set index, so a STABLE sort of (tile, id)
//             pairs reproduces the reference's per-tile ascending lists
//             (render.hpp:146-159).
//   keys/vals: (tile, candidate id) pairs, emitted in (id, tile) order, then
//             stably radix-sorted by tile.
//   partials: 6 f32 per pair at its pre-sort position -> the per-survivor merge
//             in tile order equals the reference merge order (backward.hpp:142-145).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include <utility>

namespace gpk {

constexpr int kTile = 16;                  // RasterConfig::tile_size (render.hpp:28)
constexpr int kPrepThreads = 256;
constexpr int kPrepItems = 4;
constexpr int kPrepBlock = kPrepThreads * kPrepItems;   // Gaussians per K_prep block
constexpr int kSortThreads = 256;
constexpr int kSortItems = 4;
constexpr int kSortTile = kSortThreads * kSortItems;    // keys per sort tile (one CTA)
constexpr int kMaxDigitBits = 10;                       // radix digit width <= 10 bits
constexpr int kMaxBuckets = 1 << kMaxDigitBits;
constexpr int kMaxSortPasses = 2;                       // up to 2^20 image tiles
constexpr int kSuperTiles = 16;                         // sort tiles per super-tile histogram row
constexpr int kNumParams = 11;
constexpr int kMaxBatch = 8;                            // slices per batched step (gpk_train_step_batch)

// Digit-count rows of one radix pass (a region of sort_status, nb counts per
// row): a row per sort tile [0, tiles_cap), then a super row per 16 tiles.
// Before the pass reads them, k_super_scan turns the super rows into their
// exclusive prefix over the super-tiles, so a tile's output offsets add one
// super row and at most 15 tile rows.
__host__ __device__ __forceinline__ uint64_t sort_supers_cap(uint64_t tiles_cap) {
    return (tiles_cap + kSuperTiles - 1) / kSuperTiles;
}
__device__ __forceinline__ unsigned* sort_super_row(unsigned* region, uint64_t tiles_cap, unsigned nb, unsigned t) {
    return region + (tiles_cap + t / kSuperTiles) * nb;
}
// v more keys of digit d in sort tile t (its tile and super rows)
__device__ __forceinline__ void sort_count(unsigned* region, uint64_t tiles_cap, unsigned nb, unsigned t, unsigned d,
                                           unsigned v) {
    atomicAdd(&region[(uint64_t)t * nb + d], v);
    atomicAdd(&sort_super_row(region, tiles_cap, nb, t)[d], v);
}

// Error codes recorded on the device (mirrors gpk_status).
enum DevErr : int {
    kErrNone = 0,
    kErrInvalid = 1,      // std::invalid_argument (zero quaternion, non-positive scale)
    kErrDegenerate = 2,   // DegenerateCovariance (render.hpp:111-112, core.hpp:190-195)
    kErrNumeric = 3,      // NumericFailure (backward.hpp:182-184)
};

// One survivor of the cull on the current slice (PreparedGaussian,
// render.hpp:68-79, reduced to what the pixel kernels read).
struct alignas(16) SurvivorRecord {
    double mu2d_x, mu2d_y;                        // mean of the 2-D marginal (world units)
    float conic_a, conic_b, conic_d, alpha_tilde;  // Sigma_2d^-1 and alpha*op/sqrt(det)
    uint16_t lo_x, hi_x, lo_y, hi_y;              // inclusive pixel bounds (render.hpp:123-126)
    uint32_t gidx;                                // index in the GaussianSet
    uint32_t pair_base;                           // pre-sort position of its first (tile) pair
};
static_assert(sizeof(SurvivorRecord) == 48, "record must stay 48 B");

// One (tile, survivor) pair as the pixel kernels consume it: tile-major, in
// list order (the reference's per-tile lists, render.hpp:142-160), 32 B. The
// centre is relative to the tile's first pixel centre, formed in fp64 from the
// survivor's fp64 mean (absolute fp32 pixel coordinates lose
// 3.6e-4 at 2048^2). A tile's pairs are one contiguous run: the forward and
// backward stage them into shared memory with cp.async.bulk (TMA) copies.
struct alignas(16) PairRecord {
    float ox, oy;        // mu_2d - pixel_centre(tile x0, y0), world units
    float ka, kb2, kd;   // conic a, 2b, d times -1/2 log2(e): exponent = dx(ka dx + kb2 dy) + kd dy^2
    float at;            // alpha_tilde
    uint32_t rect;       // tile-clipped footprint as bit masks: bits [0,16) covered columns, [16,32) rows
    uint32_t pos;        // pre-sort pair position (the backward's partials, K_chain's merge order)
};
static_assert(sizeof(PairRecord) == 32, "pair record must stay 32 B");

constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)

// The pair record of survivor r on tile (tx, ty) (x0 = 16 tx, y0 = 16 ty pixels).
__device__ __forceinline__ PairRecord make_pair_record(const SurvivorRecord& r, int tx, int ty, double X0, double Y0) {
    const int x0 = tx * kTile, y0 = ty * kTile;
    PairRecord p;
    p.ox = (float)(r.mu2d_x - X0);
    p.oy = (float)(r.mu2d_y - Y0);
    p.ka = r.conic_a * kNegHalfLog2e;
    p.kb2 = 2.f * r.conic_b * kNegHalfLog2e;
    p.kd = r.conic_d * kNegHalfLog2e;
    p.at = r.alpha_tilde;
    const int cx0 = max((int)r.lo_x - x0, 0), cx1 = min((int)r.hi_x - x0, kTile - 1);
    const int cy0 = max((int)r.lo_y - y0, 0), cy1 = min((int)r.hi_y - y0, kTile - 1);
    const unsigned xm = ((2u << cx1) - (1u << cx0)) & 0xffffu;
    const unsigned ym = ((2u << cy1) - (1u << cy0)) & 0xffffu;
    p.rect = xm | (ym << 16);
    const unsigned ntx = r.hi_x / kTile - r.lo_x / kTile + 1;
    p.pos = r.pair_base + (unsigned)((ty - r.lo_y / kTile) * ntx + (tx - r.lo_x / kTile));
    return p;
}
__device__ __forceinline__ void store_pair_record(PairRecord* dst, const PairRecord& p) {
    float4* d = reinterpret_cast<float4*>(dst);
    d[0] = make_float4(p.ox, p.oy, p.ka, p.kb2);
    d[1] = make_float4(p.kd, p.at, __uint_as_float(p.rect), __uint_as_float(p.pos));
}

// One candidate's parameters, gathered once by K_filter from the SoA planes
// (which it streams anyway) so later stages read 48 contiguous bytes instead of
// 11 scattered 32 B sectors.
struct alignas(16) CandParams {
    float p[11];
    uint32_t idx;                                 // index in the GaussianSet
};
static_assert(sizeof(CandParams) == 48, "candidate params must stay 48 B");

__device__ __forceinline__ void load_cand(const CandParams* __restrict__ c, float p[11], uint32_t& idx) {
    const float4* v = reinterpret_cast<const float4*>(c);
    const float4 a = __ldg(v), b = __ldg(v + 1), d = __ldg(v + 2);
    p[0] = a.x; p[1] = a.y; p[2] = a.z; p[3] = a.w;
    p[4] = b.x; p[5] = b.y; p[6] = b.z; p[7] = b.w;
    p[8] = d.x; p[9] = d.y; p[10] = d.z;
    idx = __float_as_uint(d.w);
}
__device__ __forceinline__ void store_cand(CandParams* c, const float p[11], uint32_t idx) {
    float4* v = reinterpret_cast<float4*>(c);
    v[0] = make_float4(p[0], p[1], p[2], p[3]);
    v[1] = make_float4(p[4], p[5], p[6], p[7]);
    v[2] = make_float4(p[8], p[9], p[10], __uint_as_float(idx));
}

// Gradient-buffer state word (persistent): the dense gradient planes are zero
// except at dirty_idx[0 .. count) (the previous backward's survivors), or
// kGradsDense when anything else wrote them (set_gradients, allreduce, voxel
// backward, reallocation): the next prepare then clears them densely.
constexpr unsigned kGradsDense = 0xffffffffu;

// Slice geometry + PSF + raster config, passed by value to every kernel.
struct SliceArgs {
    double R[9];          // R_c row-major
    double t[3];
    double sx, sy, ppx, ppy;
    double inv_sx, inv_sy;  // 1/pixel_spacing (fast path only; the reference path divides)
    double sigma_z;
    double tau;
    double footprint;     // footprint_sigmas
    double mod;           // scale_modifier
    int W, H;
    int tiles_x, tiles_y;
    int identity_rot;     // R_c == I exactly: world_to_camera reduces to mu + t bit-exactly
};

// Small control block, memset to zero at the start of every prepare. Its size
// is a multiple of 64 B so the arrays packed after it stay 8 B aligned.
struct alignas(64) Control {
    unsigned int prep_block_ctr;               // dynamic block id of K_filter
    unsigned int sort_tile_ctr[kMaxSortPasses];
    unsigned int survivors;                    // S, written by the last K_exact chunk
    unsigned int pairs;                        // T (uncapped)
    unsigned int pair_overflow;                // T > capacity
    unsigned int adam_done_ctr;
    unsigned int candidates;                   // C: K_filter candidates (summed by K_decide)
    unsigned int exact_chunk_ctr;              // chunk claims of K_exact
    unsigned int chain_exact;                  // survivors deferred to the fp64 chain
    unsigned int exact_decided;                // survivors decided on the reference-order fp64 path
    unsigned int dirty_ctr;                    // K_chain: next slot of the dirty-gradient list
    unsigned int decide_done;                  // K_decide groups finished (last one scans the tiles)
    unsigned int pad[2];
};

constexpr int kExactChunk = 256;               // candidates per K_exact chunk (= threads)

// Device-side error record (sticky until the host reads and clears it).
struct ErrorState {
    unsigned long long first_index[4];         // per DevErr code: min primitive index
};

__device__ __forceinline__ void record_error(ErrorState* e, int code, unsigned long long idx) {
    atomicMin(&e->first_index[code], idx);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Ordered prefix, executed by one full warp of block `b`: publish the block's
// aggregate as one ready-tagged word, then read predecessors backwards in
// windows of 512 (16 independent loads in flight per lane). A window that holds
// a published inclusive prefix ends the walk at the latest one; otherwise its
// aggregates are summed and the walk continues. The block then publishes its
// own inclusive prefix. A window costs ~1-2 L2 round trips after its slowest
// word is ready, so in-order claimed work (every predecessor resident or done)
// stops within the first window — O(1) words per block instead of O(b).
// words[b] = kReady | [kIncl] | value (value < 2^62); words zeroed before the kernel.
// publish = false: the caller published words[b] = kReady | agg earlier
// (warp_prefix_publish), e.g. before working on its next block.
__device__ __forceinline__ void warp_prefix_publish(unsigned long long* words, unsigned b, unsigned long long agg) {
    st_release_u64(&words[b], (1ull << 63) | agg);
}
__device__ __forceinline__ unsigned long long warp_prefix_aggregates(unsigned long long* words,
                                                                     unsigned b,
                                                                     unsigned long long agg,
                                                                     bool publish = true) {
    const int lane = threadIdx.x & 31;
    constexpr unsigned long long kReady = 1ull << 63, kIncl = 1ull << 62, kVal = kIncl - 1;
    if (publish && lane == 0) warp_prefix_publish(words, b, agg);
    unsigned long long excl = 0;
    for (unsigned hi = b; hi > 0;) {
        const unsigned lo = hi > 32 * 16 ? hi - 32 * 16 : 0u;
        // lane's words: j = hi - 1 - (i * 32 + lane), newest first
        unsigned long long w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int j = (int)hi - 1 - (i * 32 + lane);
            w[i] = (j >= (int)lo) ? ld_acquire_u64(&words[j]) : kReady;
        }
        int newest = -1;  // latest inclusive word this lane saw
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int j = (int)hi - 1 - (i * 32 + lane);
            while (!(w[i] & kReady)) w[i] = ld_acquire_u64(&words[j]);
            if ((w[i] & kIncl) && j >= (int)lo && j > newest) newest = j;
        }
        const int stop = __reduce_max_sync(0xffffffffu, newest);
        unsigned long long part = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int j = (int)hi - 1 - (i * 32 + lane);
            if (j >= (int)lo && j >= stop) part += w[i] & kVal;  // word `stop` adds its inclusive prefix
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (stop >= 0) break;
        hi = lo;
    }
    if (lane == 0) st_release_u64(&words[b], kReady | kIncl | (excl + agg));
    return excl;
}

// Decoupled look-back, executed by one full warp of block `b`: publishes the
// block aggregate, sums predecessors 32 at a time until an inclusive prefix is
// found, publishes its own inclusive prefix and returns the exclusive one.
// flags[b]: 0 = nothing, 1 = aggregate in agg_arr[b], 2 = prefix in incl_arr[b].
__device__ __forceinline__ unsigned long long warp_lookback(unsigned* flags,
                                                            unsigned long long* agg_arr,
                                                            unsigned long long* incl_arr,
                                                            unsigned b, unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    if (b == 0) {
        if (lane == 0) {
            incl_arr[0] = agg;
            st_release_u32(&flags[0], 2u);
        }
        return 0;
    }
    if (lane == 0) {
        agg_arr[b] = agg;
        st_release_u32(&flags[b], 1u);
    }
    long j = (long)b - 1;
    while (true) {
        const long idx = j - lane;
        unsigned f = 2u;
        unsigned long long val = 0;
        if (idx >= 0) {
            do {
                f = ld_acquire_u32(&flags[idx]);
            } while (f == 0u);
            val = (f == 2u) ? ld_relaxed_u64(&incl_arr[idx]) : ld_relaxed_u64(&agg_arr[idx]);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, f == 2u);
        const int first = pm ? __ffs(pm) - 1 : 31;
        unsigned long long part = (lane <= first) ? val : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (pm) break;
        j -= 32;
    }
    if (lane == 0) {
        incl_arr[b] = excl + agg;
        st_release_u32(&flags[b], 2u);
    }
    return excl;
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier helpers ---------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy, completion signalled on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// shared -> global bulk store (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---- packed fp32 pairs (sm_100 FFMA2 / FMUL2) --------------------------------
// Two independent fp32 lanes per instruction, each rounded exactly like the
// scalar op (fma.rn / mul.rn): the same bits as two scalar ops in half the
// issue slots. A scalar operand is broadcast with f2(x, x) (folded into the
// instruction's .F32 operand form). Measured (tests/probes/ffma2_probe.cu):
// the FMA pipe peak is unchanged, an FMA + MUFU + integer mix runs 1.4x faster.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f32x2 f2(float2 v) { return f2(v.x, v.y); }
__device__ __forceinline__ float2 f2_unpack(f32x2 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// ---- programmatic dependent launch (PDL) -------------------------------------
// Every kernel of the step chain lets its successor start launching as soon as
// all of its own CTAs are resident, and waits for its predecessor's completion
// (and memory) before touching its outputs. Back-to-back kernels then overlap
// launch latency and tails instead of draining the GPU between them. Both are
// no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_entry() {
#ifdef GPK_PDL_EARLY_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... Params, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Last-CTA tickets: a device-scope acq_rel fetch-add. Issued by one thread
// after a CTA barrier it releases the CTA's writes (the barrier orders them
// before it; PTX causality is cumulative) and, for the last CTA, acquires
// everyone else's — no separate fence.sc (MEMBAR.SC) round trip.
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* ctr) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    return old;
}

// Pairs actually stored for the current slice (T capped by the buffer size).
__device__ __forceinline__ unsigned stored_pairs(const Control* c, uint64_t cap) {
    const unsigned long long p = c->pairs;
    return (unsigned)(p < (unsigned long long)cap ? p : (unsigned long long)cap);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// One tile's list from the K_decide buckets (render.hpp:142-160 order): the
// buckets of tile d — one per K_decide group, each already in ascending slot
// order (K_decide fills them stably) — concatenated in group order. The list
// starts where the pairs of tiles < d end: a group's row holds its bucket
// starts, so row_g[d] - row_g[0] is the group's count of pairs in tiles < d
// and the tile's start is their sum over the groups (read with the bucket
// bounds; no global prefix over the tiles is needed). The whole CTA
// (kThreads, kItems groups per thread per chunk) copies cooperatively: an
// exclusive scan of the chunk's bucket sizes, then every thread takes list
// positions and finds its bucket by binary search — work linear in the list
// length and independent of how the pairs are spread over groups (a
// clustered set can put hundreds of one group's survivors into one tile).
// The table is tile-major (entry (d, g) at d * gstride + g): a tile's bounds
// over the groups are three contiguous runs (rows d, d + 1 and 0). Every list
// position is handed to emit(position, index in the list, slot) as it is copied (the callers
// write the list and build the position's PairRecord in the same pass).
// Publishes tile_begin[d] (and the end, tile_begin[ntiles], from the last
// tile) and leaves [begin, end) in s_range. Ends with a barrier.
template <int kThreads, int kItems, typename Emit>
__device__ __forceinline__ void gather_tile_list(const unsigned* __restrict__ bucket_tab, unsigned ngroups,
                                                 unsigned gstride, unsigned d, unsigned ntiles,
                                                 unsigned* tile_begin, unsigned P, uint64_t cap,
                                                 const uint32_t* vals_in, Emit emit,
                                                 unsigned* s_ex /* kThreads * kItems + 1 */,
                                                 unsigned* s_b /* kThreads * kItems */,
                                                 unsigned* s_wsum /* 2 * kThreads / 32 */,
                                                 unsigned* s_range /* 2 */) {
    constexpr unsigned kChunk = kThreads * kItems;
    constexpr int kWarps = kThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned out = 0;
    if (ngroups > kChunk) {  // the start first, over every group (the chunks below need it)
        unsigned part = 0;
        for (unsigned g = tid; g < ngroups; g += kThreads)
            part += min(__ldcg(&bucket_tab[(uint64_t)d * gstride + g]), P) - min(__ldcg(&bucket_tab[g]), P);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) s_wsum[kWarps + warp] = part;
        __syncthreads();
        for (int w = 0; w < kWarps; ++w) out += s_wsum[kWarps + w];
    }
    bool first = true;
    unsigned begin = out;  // (single chunk: set below)
    for (unsigned g0 = 0; g0 < ngroups; g0 += kChunk) {
        unsigned b[kItems], cnt[kItems], run = 0, below = 0;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {  // group g's bucket for tile d: [row[d], row[d + 1])
            const unsigned g = g0 + tid * kItems + q;
            unsigned e = 0, z = 0;
            b[q] = 0;
            if (g < ngroups) {
                b[q] = min(__ldcg(&bucket_tab[(uint64_t)d * gstride + g]), P);
                e = min(__ldcg(&bucket_tab[(uint64_t)(d + 1) * gstride + g]), P);
                z = min(__ldcg(&bucket_tab[g]), P);
            }
            cnt[q] = e > b[q] ? e - b[q] : 0u;
            run += cnt[q];
            below += b[q] - z;
        }
        unsigned incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (ngroups <= kChunk) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
        }
        if (lane == 31) s_wsum[warp] = incl;
        if (lane == 0 && ngroups <= kChunk) s_wsum[kWarps + warp] = below;
        __syncthreads();
        if (first && ngroups <= kChunk) {
            out = 0;
            for (int w = 0; w < kWarps; ++w) out += s_wsum[kWarps + w];
            begin = out;
        }
        first = false;
        unsigned ex = incl - run;
        for (int w = 0; w < warp; ++w) ex += s_wsum[w];
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            s_ex[tid * kItems + q] = ex;
            s_b[tid * kItems + q] = b[q];
            ex += cnt[q];
        }
        if (tid == kThreads - 1) s_ex[kChunk] = ex;
        __syncthreads();
        const unsigned total = s_ex[kChunk];
        for (unsigned t = tid; t < total; t += kThreads) {
            unsigned q = 0;  // last bucket starting at or before t (empty buckets share starts)
#pragma unroll
            for (unsigned step = kChunk / 2; step > 0; step >>= 1)
                if (s_ex[q + step] <= t) q += step;
            // (bounds: only a pair overflow, whose step is replayed, can exceed them)
            if ((uint64_t)out + t < cap) emit(out + t, out - begin + t, __ldcg(&vals_in[s_b[q] + (t - s_ex[q])]));
        }
        out += total;
        __syncthreads();  // s_ex / s_b / s_wsum are rewritten by the next chunk
    }
    if (ngroups == 0) begin = out = 0;
    // (a pair overflow, whose step is replayed, is the only way past the cap)
    begin = (unsigned)min((uint64_t)begin, cap);
    out = (unsigned)min((uint64_t)out, cap);
    if (tid == 0) {
        tile_begin[d] = begin;
        if (d + 1 == ntiles) tile_begin[ntiles] = out;
        s_range[0] = begin;
        s_range[1] = out;
    }
    __syncthreads();
}

struct AdamConsts {
    float b1, b2, ib1, ib2;   // beta1, beta2, 1 - beta1, 1 - beta2
    float ibc1, isbc2, eps;   // 1 / bc1, 1 / sqrt(bc2), eps
    float lr[4];              // position, opacity, scale, rotation
    // Deferred zero-gradient steps (LazyAdam): an upper bound of |delta p| of
    // this step for any moment state with |m| <= kratio sqrt(v) (per lr group),
    // and the sum of it over this step and the kLazyWindow - 2 before it.
    float drift[4], cum[4];
    float kratio;             // the moment-state bound the drift assumes (1.02 K)
    long long step;           // the step these constants are for (AdamState::step after it)
};

// ---- deferred zero-gradient Adam steps ("lazy" training steps) ---------------
// A Gaussian outside a slice's survivors has an exactly zero gradient, and its
// Adam update (optimize.hpp:195-221) is then a fixed function of its own
// parameters and moments and of the step's constants. A lazy training step
// updates only the survivors and one window of N / kLazyWindow Gaussians (by
// step number); every other Gaussian keeps the step pending. t_done[i] is the
// AdamState::step its stored parameters and moments are current at; pending
// steps t_done+1 .. t are replayed in order with the same fp32 operations as
// the eager update (the constants of the last kLazyRing steps are kept), so
// the values are the eager ones bit for bit — K_filter replays them for every
// Gaussian it cannot cull from the stored (stale) parameters widened by the
// largest possible drift of kLazyWindow - 1 steps (Adam's update is bounded:
// |m| <= K sqrt(v), K = (1 - b1) / sqrt((1 - b2)(1 - b1^2 / b2)), checked on
// every stored state; a violation sets `bad` and K_filter then replays all).
constexpr int kLazyRing = 32;    // AdamConsts of step s at ring[s % kLazyRing]
constexpr int kLazyWindow = 16;  // a Gaussian is brought up to date at least every 16 steps
struct LazyAdam {
    uint32_t* t_done;
    AdamConsts* ring;
    long long* step;          // AdamState::step (device)
    float* m;
    float* v;
    unsigned* bad;
    float bbox_min[3], bbox_max[3];
};

// Kernel-launch wrappers (defined in the .cu files, called by session.cu).
struct PrepLaunch {
    const float* params;      // 11 planes x cap
    uint64_t cap;             // plane stride
    uint32_t n;
    float* grads;             // cleared (dense or sparse, see kGradsDense) when non-null
    unsigned* grads_dirty;          // persistent gradient-buffer state word
    const uint32_t* dirty_idx;      // previous survivors' set indices
    CandParams* cand;         // K_filter -> K_decide: candidate params, block-major slots
    unsigned* cand_count;     // candidates per chunk (plain stores)
    CandParams* surv_params;  // survivor params by survivor slot
    uint2* grp_pairs;         // per K_decide group: (first pair position, pair count)
    unsigned* bucket_tab;     // single-pass slices: bucket starts, tile-major (else nullptr)
    unsigned bucket_gstride;  // groups per tile row of bucket_tab
    unsigned* tile_begin;     // (unused by K_decide: the gather derives each tile's start)
    unsigned* grp_surv;       // per K_decide group: survivors (slots g*4096 + [0, S_g))
    unsigned* surv_bits;      // optional: bit i = Gaussian i survived (K_decide writes its group's words)
    unsigned nfilter;         // 64-Gaussian chunks
    SurvivorRecord* records;  // indexed by candidate slot
    uint32_t* survivor_list;  // survivor slot -> set index (K_decide)
    uint32_t* exact_list;     // slots of the fp64-decided survivors (count: Control::chain_exact)
    unsigned* head;           // K_filter: zero these head_words first (the control head), or nullptr
    unsigned head_words;
    uint32_t* keys;           // pre-sort tile keys
    uint32_t* vals;           // pre-sort candidate slots
    uint64_t pair_cap;
    unsigned* hist;           // kMaxSortPasses x kMaxBuckets global digit counts
    unsigned* tile_hist0;     // pass-0 region: per sort tile rows, then per super-tile rows
    unsigned* tile_hist_all;  // kMaxSortPasses regions of hist_region words (zeroed by K_filter)
    uint64_t sort_tiles_cap;
    uint64_t hist_region;     // words per pass region
    unsigned* prev_sort_words;  // persistent: {sort tiles, buckets, passes} of the previous sort
    int passes;
    int digit_bits;           // radix digit width of every pass
    unsigned long long* exact_words;  // per chunk: ready<<63 | S<<32 | P (zeroed per prepare)
    Control* ctrl;
    ErrorState* err;
    SliceArgs slice;
    // lazy training steps: K_filter replays the pending steps of every Gaussian
    // it does not cull (lazy_on = 0: the parameters are current)
    int lazy_on;
    LazyAdam lazy;
};

constexpr int kFilterItems = 4;                            // consecutive Gaussians per K_filter lane
constexpr int kFilterBlock = 32 * kFilterItems;            // Gaussians per K_filter warp chunk (128)
constexpr int kDecideChunks = 32;                          // K_filter chunks per K_decide group
constexpr int kDecideGroupSize = kDecideChunks * kFilterBlock;  // Gaussians per group (4096)
constexpr int kParamAlign = 512;                           // plane stride (capacity) granularity

// Gather (single radix digit covers every tile): K_decide bucketed each
// group's pairs by tile and wrote the bucket starts; one CTA per tile
// concatenates its buckets in group order (= slot order).
struct GatherLaunch {
    const unsigned* bucket_tab;    // tile-major: (tile d, group g) bucket start at d * gstride + g; row nb = ends
    unsigned ngroups;
    unsigned ntiles;
    unsigned gstride;              // groups per tile row
    unsigned* tile_begin;          // out: tile list starts (+ end), derived by the gather
    const uint32_t* vals_in;       // bucketed slots
    uint32_t* vals_out;            // per-tile lists, ascending slot
    const Control* ctrl;
    uint64_t pair_cap;
    // the tile-major pair records of the lists (PairRecord)
    const SurvivorRecord* records;
    PairRecord* pairs;
    SliceArgs slice;
};
void launch_gather(const GatherLaunch& a, cudaStream_t st);
// Multi-pass slices: the pair records of the sorted lists, one per position,
// and the tiles' start positions (tile_start[0 .. tiles], the last = P).
void launch_pair_records(const uint32_t* keys, const uint32_t* vals, const SurvivorRecord* records, PairRecord* pairs,
                         unsigned* tile_start, const Control* ctrl, uint64_t pair_cap, const SliceArgs& slice,
                         int num_sms, cudaStream_t st);

struct SortLaunch {
    const uint32_t* keys_in;
    const uint32_t* vals_in;
    uint32_t* keys_out;
    uint32_t* vals_out;
    const unsigned* hist;          // 2^bits global counts of this pass's digit
    const unsigned* tile_hist;     // this pass's region: tile rows then super-tile rows (2^bits each)
    unsigned* tile_hist_next;      // next pass's region (nullptr on the last pass)
    uint64_t sort_tiles_cap;       // offset (in rows) of the super-tile rows
    unsigned* prev_sort_words;     // written by the last pass: {sort tiles, buckets, passes}
    unsigned* grp_begin;           // last pass only: first sorted position of every digit (+ end)
    const uint2* grp_pairs;        // pass over K_decide output: sort tiles are its groups (in group
    unsigned ngroups;              //   order = slot order); nullptr: tiles of kSortTile << tile_shift positions
    int shift;
    int tile_shift;                // position tiles are kSortTile << tile_shift keys (<= ~1024 tiles)
    int bits;                      // digit width of this pass
    unsigned next_buckets;         // 2^bits of the next pass
    int pass;
    const Control* ctrl;
    uint64_t pair_cap;
};

// Words between the global digit histograms and the chunk words of the
// control head: first sorted position of every last-pass digit group (+ end).
constexpr int kGroupBeginWords = kMaxBuckets + 4;

// The photometric loss from the loss kernel's per-CTA partial sums (ssim sum,
// l1 sum; loss.hpp:29-35): L = l1/N + lambda*dssim*(1 - ssim/N). Reduced by a
// whole CTA in a fixed order (thread t sums CTAs t, t + blockDim, ..., then a
// fixed warp/block tree): deterministic run to run. Written by thread 0 to
// *loss and, when given, straight into the caller's pinned host memory (a
// posted write, visible to the host once the kernel has completed).
struct LossFinish {
    const double* partial;  // nullptr: nothing to finish
    unsigned nblk;
    int with_ssim;
    double inv_n, lambda, dssim_scale;
    double* loss;
    double* loss_host;
};

__device__ __forceinline__ void block_sum2(double& a, double& b, double* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
        s_red[2 * warp] = a;
        s_red[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = 0.0;
        b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += s_red[2 * w];
            b += s_red[2 * w + 1];
        }
    }
}

__device__ __forceinline__ void loss_reduce(const LossFinish& f, double* s_red /* 2 * 32 */) {
    double ss = 0.0, l1 = 0.0;
    for (unsigned k = threadIdx.x; k < f.nblk; k += blockDim.x) {
        ss += __ldcg(&f.partial[2 * k]);
        l1 += __ldcg(&f.partial[2 * k + 1]);
    }
    block_sum2(ss, l1, s_red);
    if (threadIdx.x != 0) return;
    // explicit roundings: the same bits whichever kernel this is inlined into
    double L = __dmul_rn(l1, f.inv_n);
    if (f.with_ssim)
        L = __dadd_rn(L, __dmul_rn(__dmul_rn(f.lambda, f.dssim_scale), __dsub_rn(1.0, __dmul_rn(ss, f.inv_n))));
    *f.loss = L;
    if (f.loss_host) *f.loss_host = L;
}

struct RasterLaunch {
    const SurvivorRecord* records;
    const uint32_t* keys;          // sorted tile keys
    const uint32_t* vals;          // sorted candidate ids
    const unsigned* grp_begin;     // first position of each tile (+ end): the single-pass gather's
                                   // starts, or k_pair_records' tile starts after radix passes
    int grp_shift;                 // 0, or -1: no sort pass ran (one tile: [0, P))
    const Control* ctrl;
    uint64_t pair_cap;
    float* image;                  // forward output
    const float* dl_di;            // backward input
    float* partials;               // backward output: 6 f32 per pair (pre-sort position)
    SliceArgs slice;
    // fused SSIM backward (training step): dL/dI = sign(I-T)/N - k (W g1 + 2 I W g2 + T W g3)
    const float* ssim_g;           // 3 planes from k_ssim_fwd, or nullptr (dL/dI given)
    const float* target;
    float ssim_k, inv_n;           // lambda * dssim_scale, 1/(W*H)
    float w[11];                   // window taps
    // fused gather (training step, single-pass slices): the forward CTA first
    // builds its tile's list from K_decide's buckets (k_gather's work) into
    // vals_out (== vals), or nullptr when the lists are built already
    const unsigned* bucket_tab;
    unsigned ngroups, gstride;
    const uint32_t* vals_in;
    uint32_t* vals_out;
    // tile-major pair records: written by the gather (or by the forward when it
    // gathers), read by the pixel kernels through cp.async.bulk
    PairRecord* pairs;
    // training step: the backward's CTA 0 also finishes the loss from
    // k_ssim_fwd's partials (the kernel boundary orders them; no ticket)
    LossFinish fin;
};

struct ChainLaunch {
    const CandParams* sparams;     // survivor params by candidate slot (K_exact)
    uint64_t cap;
    uint32_t* dirty_idx;           // out: survivors' set indices (next prepare's sparse clear)
    unsigned* grads_dirty;         // out: survivor count
    const SurvivorRecord* records;
    const uint32_t* survivor_list;
    const float* partials;
    const Control* ctrl;
    float* grads;                  // dense gradient planes (set-indexed) ...
    float* slot_grads;             // ... or, when non-null, slot-indexed planes (see AdamLaunch)
    uint16_t* gmap;                // slot mode: 1 + the survivor's offset in its group, by set index
    // data-parallel union rows (dp.cu): when urows is non-null the gradient of
    // set index i goes to row umap[i] - 1 of 11 planes (stride cap), rows < ucap
    const uint32_t* umap;
    float* urows;
    uint64_t ucap;
    float* stat_norm;              // optional (screen-space dL/dmu_2d norm)
    uint8_t* stat_observed;        // optional
    float* stat_world;             // optional, 3 per primitive
    double* acc_norm;              // optional DensifyAccum (fit): += |dL/dmu_2d| ...
    int* acc_obs;                  //   ... += 1 ...
    double* acc_world;             //   ... += world dL/dmu
    const uint32_t* exact_list;    // record slots of the fp64 chain (K_decide)
    unsigned* exact_count;         // Control::chain_exact
    const unsigned* grp_surv;      // survivors per K_decide group (CTA per group)
    unsigned* dirty_ctr;           // Control::dirty_ctr
    ErrorState* err;
    SliceArgs slice;
};

// Per-step Adam constants (adam.cuh adam_consts), written by k_adam_consts.
struct AdamLaunch {
    float* params;
    float* grads;         // read (and cleared where non-zero by the fused Adam + cull)
    float* m;
    float* v;
    uint64_t cap;
    uint32_t n;           // primitives [lo, n) are updated (lo > 0: this rank's shard)
    uint32_t lo;
    float bbox_min[3], bbox_max[3];
    double lr[4];         // position, opacity, scale, rotation (or lr0 when scheduled)
    int scheduled;        // lr = lr0 * 0.1^((step-1)/total)
    int total;
    double beta1, beta2, eps;
    long long* step;      // AdamState::step, device
    AdamConsts* consts;   // this step's constants (k_adam_consts; the update kernel stores c.step)
    const Control* ctrl;  // skip when the slice overflowed its pair capacity
    // Slot-gradient mode (the single-GPU training step): when slot_grads is
    // non-null the gradients are not read from `grads` but from the chain's
    // survivor-slot planes (slot g*4096 + j holds group g's j-th survivor);
    // gmap[i] = 1 + j for a survivor i of group g, 0 for every other primitive
    // (zero gradient). Adam clears the map entries it reads. Nothing has to
    // clear dense gradient planes between steps, and Adam reads 2 B per
    // primitive + 44 B per survivor instead of 44 B per primitive.
    const float* slot_grads;
    uint16_t* gmap;
    const uint32_t* surv_gidx;    // slot -> set index (the gradient scatter)
    const unsigned* grp_surv;
    // Batched training step (gpk_train_step_batch, B slices, one Adam): the
    // further slices' slot gradients and maps for k_sum_slots, which sums a
    // primitive's gradient over the slices in slice order (slice 0 =
    // slot_grads / gmap above) into the dense planes and clears every map it
    // reads; src_ctrl: an overflowed slice anywhere skips the update.
    // data-parallel step (dp.cu): when umap is non-null the gradient of
    // Gaussian i is row umap[i] - 1 of slot_grads (0: zero gradient), and
    // uctrl[1] != 0 (union rows beyond the capacity) skips the update
    const uint32_t* umap;
    const unsigned* uctrl;
    int nsrc;                     // further slices (0: a single slice)
    const float* src_slot[kMaxBatch - 1];
    uint16_t* src_gmap[kMaxBatch - 1];
    const Control* src_ctrl[kMaxBatch - 1];
    // the constants ring of the lazy steps (k_adam_consts writes every step's
    // entry) and, for the lazy update kernels, the rest of their state
    LazyAdam lazy;
};

struct LossLaunch {
    const float* image;
    const float* target;
    float* dl_di;
    float* g;            // 3 planes of W*H: g1, g2, g3
    double* partial;     // 2 per CTA: ssim sum, l1 sum
    double* loss;        // output
    double* loss_host;   // optional second output: mapped pinned host memory (gpk_set_loss_sink)
    unsigned* done_ctr;
    int W, H;
    double lambda, dssim_scale;
    float w[11];         // normalized Gaussian taps
    int finish_in_fwd;   // training step (k_ssim_bwd is skipped: the raster backward turns the
                         // SSIM partials into dL/dI): 1 = k_ssim_fwd finalizes the loss
                         // (last-CTA ticket), 0 = the raster backward's CTA 0 does
};
void launch_loss_fwd_only(const LossLaunch& a, cudaStream_t st);

// ---- voxelizer (voxelize.hpp) -------------------------------------------------
// One primitive's voxelizer state (VoxelPrim, voxelize.hpp:42-48), 64 B.
struct alignas(16) VoxRecord {
    float mu[3];          // world mean
    float log2a;          // log2(alpha)
    float a[6];           // Sigma^-1 * (-0.5*log2 e): a00 a11 a22 2a01 2a02 2a12
    uint16_t lo[3], hi[3];  // inclusive voxel index bounds of the support AABB
    uint32_t gidx;
    uint32_t pair_base;
    uint32_t pad;
};
static_assert(sizeof(VoxRecord) == 64, "voxel record must stay 64 B");

struct VoxArgs {
    int dims[3];
    int tile[3];
    int ntiles[3];
    double spacing[3];
    double origin[3];
    double support;
    double mod;
};

struct VoxPrepLaunch {
    const float* params;
    uint64_t cap;
    uint32_t n;
    VoxRecord* records;        // indexed by set index (all N slots)
    uint32_t* survivor_list;   // survivor slot -> set index
    uint32_t* keys;
    uint32_t* vals;
    uint64_t pair_cap;
    unsigned* hist;
    unsigned* tile_hist0;
    uint64_t sort_tiles_cap;
    int passes;
    int digit_bits;
    int tile_shift;            // sort tiles of kSortTile << tile_shift positions (SortLaunch)
    unsigned long long* chunk_words;  // per 256-prim chunk: ready<<63 | S<<32 | P
    Control* ctrl;
    ErrorState* err;
    VoxArgs v;
    int grid;
};

struct VoxEvalLaunch {
    const VoxRecord* records;
    const uint32_t* keys;      // sorted voxel-tile keys
    const uint32_t* vals;      // sorted set indices
    const unsigned* tile_start;  // first sorted position of every tile (+ end, k_key_starts)
    const Control* ctrl;
    uint64_t pair_cap;
    float* volume;             // voxelize output
    const float* dl_dv;        // backward input
    float* partials;           // backward output: 10 f32 per pair (pre-sort position)
    VoxArgs v;
    int dl_global;             // backward: tile too large to stage dL/dV in shared memory
};

struct VoxChainLaunch {
    const float* params;
    uint64_t cap;
    const VoxRecord* records;
    const uint32_t* survivor_list;
    const float* partials;
    const Control* ctrl;
    float* grads;
    ErrorState* err;
    VoxArgs v;
};

// densify_and_prune (optimize.hpp:255-344), densify.cu
struct DensifyLaunch {
    const float* params;           // 11 planes, stride cap
    const float* m;
    const float* v;
    uint64_t cap, n;
    const double* acc_norm;        // DensifyAccum (optimize.hpp:228-249): sum of |dL/dmu_2d|
    const int* acc_obs;            //   observation count
    const double* acc_world;       //   sum of world dL/dmu, 3 per primitive
    double tau, grad_threshold, split_threshold, shrink, mod;
    double bmin[3], bmax[3];
    uint8_t* cls;                  // per primitive: prune / keep / clone / split
    unsigned* block_sums;          // 3 per block: kept, born, split (then their block offsets)
    unsigned* totals;              // 3: kept, born, split
    const double* normals;         // 6 per split parent, in parent order (host Rng)
    float* out_params;             // 11 planes, stride cap_out (cleared)
    float* out_m;
    float* out_v;
    uint64_t cap_out;
};

// layout.cu: 11-f32 records <-> 11 planes of stride cap
void launch_records_to_planes(const float* rec, uint64_t n, float* planes, uint64_t cap, cudaStream_t st);
void launch_planes_to_records(const float* planes, uint64_t cap, uint64_t n, float* rec, cudaStream_t st);
unsigned densify_blocks(uint64_t n);
int set_last_error(int code, const std::string& msg);  // session.cu (thread-local message)
void launch_densify_classify(const DensifyLaunch& a, cudaStream_t st);
void launch_densify_emit(const DensifyLaunch& a, cudaStream_t st);

void launch_vox_prep(const VoxPrepLaunch& a, cudaStream_t st);
void launch_prepared_full(const CandParams* sparams, const uint32_t* slots, unsigned S, const SliceArgs& s,
                          double* out, cudaStream_t st);
void launch_vox_eval(const VoxEvalLaunch& a, cudaStream_t st);
// sort.cu: the tile starts of a sorted key list (start[0 .. ntiles], the last = P)
void launch_key_starts(const uint32_t* keys, const Control* ctrl, uint64_t pair_cap, unsigned ntiles,
                       unsigned* start, int num_sms, cudaStream_t st);
void launch_vox_bwd(const VoxEvalLaunch& a, cudaStream_t st);
void launch_vox_chain(const VoxChainLaunch& a, int grid, cudaStream_t st);

void launch_prep(const PrepLaunch& a, int num_sms, cudaStream_t st);
// dp.cu: the data-parallel union numbering and its dense view
void launch_union_scan(const unsigned* words, unsigned nchunks, unsigned* prefix, unsigned* uctrl, uint64_t ucap,
                       cudaStream_t st);
void launch_union_map(const unsigned* words, const unsigned* prefix, uint32_t n, uint32_t* umap, float* rows,
                      uint64_t cap, uint64_t ucap, cudaStream_t st);
void launch_union_to_dense(const uint32_t* umap, const float* rows, uint64_t cap, uint32_t n, uint64_t ucap,
                           float* grads, cudaStream_t st);
// own / union_words: a data-parallel step (only pose `own` stores candidates;
// the union of every pose's candidates as 4 words per 128-Gaussian chunk)
void launch_prep_multi(const PrepLaunch* pl, int nb, int num_sms, cudaStream_t st, int own = -1,
                       unsigned* union_words = nullptr);
void launch_adam_cull(const AdamLaunch& a, const PrepLaunch& next, cudaStream_t st);
void launch_bin(const PrepLaunch& a, int num_sms, cudaStream_t st);
void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st);
void launch_super_scan(unsigned* region, uint64_t tiles_cap, unsigned nb, const Control* ctrl, uint64_t pair_cap,
                       unsigned ngroups, unsigned tile_keys, cudaStream_t st);
void launch_raster_fwd(const RasterLaunch& a, cudaStream_t st);
void launch_raster_bwd(const RasterLaunch& a, cudaStream_t st);
void launch_chain(const ChainLaunch& a, int grid, int num_sms, cudaStream_t st);
void launch_chain_exact(const ChainLaunch& a, int grid, cudaStream_t st);
void launch_adam(const AdamLaunch& a, cudaStream_t st);
void launch_adam_consts(const AdamLaunch& a, cudaStream_t st);
void launch_sum_slots(const AdamLaunch& a, cudaStream_t st);
void launch_adam_rest(const AdamLaunch& a, const unsigned* surv_bits, int ctas, cudaStream_t st);
void launch_adam_final(const AdamLaunch& a, unsigned ngroups, cudaStream_t st);
// lazy training steps (adam.cu): the survivors' update (pending steps replayed
// first), the step's window of Gaussians, every Gaussian (flush), and the
// start of lazy mode (t_done = step, moment states checked)
void launch_lazy_survivors(const AdamLaunch& a, unsigned ngroups, cudaStream_t st);
void launch_lazy_window(const AdamLaunch& a, cudaStream_t st);
void launch_lazy_flush(const AdamLaunch& a, cudaStream_t st);
void launch_lazy_begin(const AdamLaunch& a, cudaStream_t st);
enum ScatterMode : int { kScatterSet = 1, kScatterAdd = 2, kScatterClearMap = 4 };
void launch_scatter_slot_grads(const AdamLaunch& a, unsigned ngroups, int mode, cudaStream_t st);
void launch_loss(const LossLaunch& a, cudaStream_t st);
unsigned loss_partial_blocks(int W, int H, double lambda);

}  // namespace gpk
