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

namespace gpk {

constexpr int kTile = 16;                  // RasterConfig::tile_size (render.hpp:28)
constexpr int kPrepThreads = 256;
constexpr int kPrepItems = 4;
constexpr int kPrepBlock = kPrepThreads * kPrepItems;   // Gaussians per K_prep block
constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;    // keys per onesweep tile
constexpr int kMaxSortPasses = 3;                       // up to 2^24 tiles
constexpr int kNumParams = 11;

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

// Slice geometry + PSF + raster config, passed by value to every kernel.
struct SliceArgs {
    double R[9];          // R_c row-major
    double t[3];
    double sx, sy, ppx, ppy;
    double sigma_z;
    double tau;
    double footprint;     // footprint_sigmas
    double mod;           // scale_modifier
    int W, H;
    int tiles_x, tiles_y;
    int identity_rot;     // R_c == I exactly: world_to_camera reduces to mu + t bit-exactly
};

// Small control block, memset to zero at the start of every prepare.
struct Control {
    unsigned int prep_block_ctr;               // dynamic block id of K_prep
    unsigned int sort_tile_ctr[kMaxSortPasses];
    unsigned int survivors;                    // S, written by the last K_prep block
    unsigned int pairs;                        // T (uncapped)
    unsigned int pair_overflow;                // T > capacity
    unsigned int adam_done_ctr;
    unsigned int pad[8];
};

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

// Kernel-launch wrappers (defined in the .cu files, called by session.cu).
struct PrepLaunch {
    const float* params;      // 11 planes x cap
    uint64_t cap;             // plane stride
    uint32_t n;
    float* grads;             // zero-filled for non-survivors when non-null
    SurvivorRecord* records;  // indexed by candidate id
    uint32_t* survivor_list;  // slot -> candidate id
    uint32_t* keys;           // pre-sort tile keys
    uint32_t* vals;           // pre-sort candidate ids
    uint64_t pair_cap;
    unsigned* hist;           // kMaxSortPasses x 256 digit counts
    int passes;
    unsigned* epoch;          // persistent sort epoch, bumped once per prepare
    unsigned* prep_flags;     // per block, zeroed each prepare
    unsigned long long* prep_agg;
    unsigned long long* prep_incl;
    Control* ctrl;
    ErrorState* err;
    SliceArgs slice;
};

struct SortLaunch {
    const uint32_t* keys_in;
    const uint32_t* vals_in;
    uint32_t* keys_out;
    uint32_t* vals_out;
    const unsigned* hist;          // 256 counts of this pass
    unsigned long long* status;    // per (tile, digit): epoch<<32 | flag<<30 | count
    const unsigned* epoch;         // persistent sort epoch (device)
    int shift;
    int pass;
    const Control* ctrl_ro;
    Control* ctrl;
    uint64_t pair_cap;
};

struct RasterLaunch {
    const SurvivorRecord* records;
    const uint32_t* keys;          // sorted tile keys
    const uint32_t* vals;          // sorted candidate ids
    const Control* ctrl;
    uint64_t pair_cap;
    float* image;                  // forward output
    const float* dl_di;            // backward input
    float* partials;               // backward output: 6 f32 per pair (pre-sort position)
    SliceArgs slice;
};

struct ChainLaunch {
    const float* params;
    uint64_t cap;
    const SurvivorRecord* records;
    const uint32_t* survivor_list;
    const float* partials;
    const Control* ctrl;
    float* grads;
    float* stat_norm;              // optional (screen-space dL/dmu_2d norm)
    uint8_t* stat_observed;        // optional
    float* stat_world;             // optional, 3 per primitive
    ErrorState* err;
    SliceArgs slice;
};

struct AdamLaunch {
    float* params;
    const float* grads;
    float* m;
    float* v;
    uint64_t cap;
    uint32_t n;
    float bbox_min[3], bbox_max[3];
    double lr[4];         // position, opacity, scale, rotation (or lr0 when scheduled)
    int scheduled;        // lr = lr0 * 0.1^((step-1)/total)
    int total;
    double beta1, beta2, eps;
    long long* step;      // AdamState::step, device
    unsigned* done_ctr;
    const Control* ctrl;  // skip when the slice overflowed its pair capacity
};

struct LossLaunch {
    const float* image;
    const float* target;
    float* dl_di;
    float* g;            // 3 planes of W*H: g1, g2, g3
    double* partial;     // 2 per CTA: ssim sum, l1 sum
    double* loss;        // output
    unsigned* done_ctr;
    int W, H;
    double lambda, dssim_scale;
    float w[11];         // normalized Gaussian taps
};

void launch_prep(const PrepLaunch& a, cudaStream_t st);
void launch_sort_pass(const SortLaunch& a, int grid, cudaStream_t st);
void launch_raster_fwd(const RasterLaunch& a, cudaStream_t st);
void launch_raster_bwd(const RasterLaunch& a, cudaStream_t st);
void launch_chain(const ChainLaunch& a, int grid, cudaStream_t st);
void launch_adam(const AdamLaunch& a, cudaStream_t st);
void launch_loss(const LossLaunch& a, cudaStream_t st);
unsigned loss_partial_blocks(int W, int H, double lambda);

}  // namespace gpk
