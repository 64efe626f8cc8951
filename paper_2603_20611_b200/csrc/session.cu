// session.cu — C-ABI implementation (include/gpile_b200.h): device-resident
// session state, host-side validation with the reference's error semantics,
// and the launch sequence of each reference entry point.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gpile_b200.h"
#include "common.cuh"

using namespace gpk;

namespace {

thread_local std::string t_err;
thread_local int64_t t_err_index = -1;

int fail(int code, const std::string& msg, int64_t index = -1) {
    t_err = msg;
    t_err_index = index;
    return code;
}

}  // namespace

namespace gpk {
// the fit driver (fit.cu) reports through the same thread-local message
int set_last_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace gpk

namespace {

int ok() {
    t_err.clear();
    t_err_index = -1;
    return GPK_OK;
}

#define CK(expr)                                                                        \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            if (_e == cudaErrorMemoryAllocation)                                        \
                return fail(GPK_ERR_OUT_OF_MEMORY, std::string("cuda: ") + cudaGetErrorString(_e)); \
            return fail(GPK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
        }                                                                               \
    } while (0)

#define TRY(expr)                 \
    do {                          \
        int _s = (expr);          \
        if (_s != GPK_OK) return _s; \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool borrowed = false;  // another session's memory (slice contexts share the parameters)
    void release() {
        if (p && !borrowed) cudaFree(p);
        p = nullptr;
        bytes = 0;
        borrowed = false;
    }
    void borrow(const DevBuf& o) {
        release();
        p = o.p;
        bytes = o.bytes;
        borrowed = true;
    }
    // (Re)allocate to at least `need` bytes; contents are NOT preserved.
    cudaError_t ensure(size_t need) {
        if (need <= bytes && p && !borrowed) return cudaSuccess;
        release();
        if (need == 0) need = 16;
        cudaError_t e = cudaMalloc(&p, need);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

struct PrepState {
    bool valid = false;
    SliceArgs slice{};
    int tiles = 0;
    int passes = 0;
    int digit_bits = 0;
    int final_buf = 0;         // which key/val buffer holds the sorted pairs
    bool rasterized = false;
    bool grads_zeroed = false;  // K_prep zero-filled non-survivor gradients
    bool ssim_pending = false;  // training step: the raster backward forms dL/dI from the SSIM partials
    bool lists_pending = false; // single-pass slice whose tile lists the forward builds (fused gather)
    float ssim_k = 0.f, inv_n = 0.f;
    float w[11] = {};
    LossFinish fin{};           // ssim_pending: the loss the raster backward finishes (partial set)
    gpk_slice_pose pose{};
    gpk_psf psf{};
    gpk_raster_config cfg{};
};

}  // namespace

struct gpk_session {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // U1 with a given dL/dI: the forward runs on `side`, concurrently with the
    // backward on `stream` (fork/join by events; captured graphs keep the fork)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr;  // Adam constants on the side stream
    cudaEvent_t ev_xfork = nullptr, ev_xjoin = nullptr;  // K_chain_exact beside K_chain
    // slice targets are uploaded on their own stream and overlap the step's
    // prepare + forward; the loss waits on ev_tgt_ready (see gpk_upload)
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_tgt_fork = nullptr;
    // two target slots (gpk_set_target_slot): a step reads the current slot's
    // buffer, so a caller alternating slots uploads the next slice's target
    // while the previous step still reads the other one; each slot has its own
    // upload-done (ev_tgt_ready) and last-reader (ev_tgt_free) events
    int tgt_slot = 0;
    cudaEvent_t ev_tgt_ready_k[2] = {nullptr, nullptr};
    // recorded after the last kernel that reads the target (the loss, or the
    // raster backward that finishes the SSIM gradient): the next upload's copy
    // starts there, overlapping the rest of the step (chain, Adam) and the next
    // step's prepare and forward
    cudaEvent_t ev_tgt_free_k[2] = {nullptr, nullptr};
    // under capture the release is a side branch (a record node on its own
    // stream, joined at the end of the graph) so the PDL edge from the raster
    // backward to the chain stays programmatic
    cudaStream_t rel_stream = nullptr;
    cudaEvent_t ev_rel_fork = nullptr, ev_rel_join = nullptr;
    bool rel_join_pending = false;
    bool tgt_pending_k[2] = {false, false};
    // data parallelism (gpk_comm_init): this session's NCCL communicator
    void* comm = nullptr;
    int comm_rank = 0, comm_world = 1;
    bool consts_pending = false;  // k_adam_consts was launched ahead (wait on ev_cjoin)
    uint64_t n = 0, cap = 0;
    gpk_bounds bbox{};
    uint64_t pair_cap = 0;
    uint64_t sort_tiles_cap = 0;
    uint64_t hist_region = 0;  // words per radix pass in sort_status

    DevBuf params, grads, adam_m, adam_v, records, survivors;
    DevBuf keys[2], vals[2], partials, sort_status;  // sort_status: per-sort-tile digit counts
    DevBuf pair_recs;  // tile-major PairRecords of the sorted lists (32 B per pair)
    DevBuf tile_start; // multi-pass slices: first sorted position of every tile (+ end)
    DevBuf vox_tile_start;  // the voxelizer's 8^3 tiles: first sorted position (+ end)
    bool loss_in_fwd = false;  // A/B knob: the fused loss finished by k_ssim_fwd's last CTA
    DevBuf head;       // Control | hist | prep flags (memset per prepare)
    DevBuf cand_list;  // K_chain's deferral list (survivor slots for the fp64 chain)
    DevBuf cand;       // CandParams of K_filter's candidates (block-major slots)
    DevBuf cand_count; // candidates per 1024-Gaussian chunk
    DevBuf surv_params;  // CandParams of survivors by survivor slot (K_decide)
    DevBuf dirty_idx;  // set indices of the last backward's survivors
    DevBuf slot_grads; // training-step gradients by survivor slot (11 planes, stride cap)
    bool grads_in_slots = false;  // the latest gradient lives in slot_grads (see AdamLaunch)
    // data-parallel union rows (dp.cu, gpk_train_step_dp)
    DevBuf union_words, union_prefix, umap, urows, uctrl;
    uint64_t ucap = 0;             // rows exchanged per plane (the all-reduce count), <= cap
    bool grads_in_union = false;   // the latest gradient is a data-parallel step's union rows
    DevBuf gmap;       // slot mode: u16 per primitive, 1 + survivor offset in its group (else 0)
    bool gmap_dirty = false;      // a slot backward wrote gmap and no Adam consumed (cleared) it
    DevBuf grp_table;  // per K_decide group: uint2 (first pair, pairs), then u32 survivors
    DevBuf bucket_tab; // single-pass slices: bucket starts, tile-major (tiles + 1 rows of bucket_gs groups)
    unsigned bucket_gs = 0;
    uint2* grp_pairs() { return grp_table.as<uint2>(); }
    unsigned* grp_surv() { return reinterpret_cast<unsigned*>(grp_table.as<char>() + (cap / kDecideGroupSize + 2) * 8); }
    int num_sms = 148;
    // candidates of a slice culled ahead of time by the fused Adam + cull of the
    // previous training step (K_filter can be skipped when they match)
    struct Prefilter {
        bool valid = false;
        gpk_slice_pose pose{};
        gpk_psf psf{};
        gpk_raster_config cfg{};
        uint64_t n = 0;
    } prefilter;
    bool assume_prefiltered = false;  // set while capturing a pipelined train step
    bool fuse_gather = false;         // training step: the next prepare leaves the gather to the forward
    bool fuse_gather_ok = true;       // (GPK_FUSE_GATHER=0: the gather stays its own kernel; A/B measurements)
    // Adam split around the render (single-GPU training step): the
    // non-survivors' update on adam_stream beside the render (k_adam_rest,
    // adam_rest_ctas CTAs, -1 = one per 512 Gaussians), the survivors' after
    // the chain. Off: measured slower on B200 (C2: 0.170-0.300 ms vs 0.139 ms
    // per step — the streaming Adam's CTAs hold the SMs the latency-bound
    // slice kernels need). GPK_ADAM_SPLIT=1 enables it,
    // GPK_ADAM_REST_CTAS sizes it.
    bool adam_split = false;
    int adam_rest_ctas = -1;
    // lazy training steps (LazyAdam, common.cuh): the survivors and one window
    // of Gaussians updated per step, every other Gaussian's zero-gradient step
    // deferred and replayed in order where it is next needed
    bool lazy_on = false;        // mode (GPK_LAZY_ADAM=1 / gpk_set_lazy_adam; measured slower)
    bool lazy_live = false;      // t_done is valid (every deferred step is replayable)
    bool lazy_pending = false;   // a lazy step ran since the last flush
    bool cap_lazy = false;       // capture: the graph being captured runs lazily
    bool cap_lazy_used = false;  // ... and recorded lazy kernels
    bool cap_lazy_writes = false;
    DevBuf t_done;               // u32 per Gaussian
    double* loss_sink = nullptr; // device alias of the caller's pinned host loss slot (gpk_set_loss_sink)
    cudaStream_t adam_stream = nullptr;
    cudaEvent_t ev_rest_fork = nullptr, ev_rest_join = nullptr;
    DevBuf surv_bits;                 // K_decide: bit i = Gaussian i survived the last prepare
    struct CaptureMeta {
        bool needs_prefilter = false, sets_prefilter = false, writes_params = false;
        gpk_slice_pose next_pose{};
    } capture_meta;
    AdamConsts* lazy_ring() { return reinterpret_cast<AdamConsts*>(persist.as<char>() + 256); }
    unsigned* lazy_bad() { return reinterpret_cast<unsigned*>(persist.as<char>() + 256 + kLazyRing * sizeof(AdamConsts)); }
    DevBuf persist;    // ErrorState | epoch | adam step | adam done ctr | loss done ctr | loss
    DevBuf image, dl_di, target_k[2], loss_g, loss_partial;
    DevBuf& tgt() { return target_k[tgt_slot]; }
    cudaEvent_t& ev_tgt_ready() { return ev_tgt_ready_k[tgt_slot]; }
    cudaEvent_t& ev_tgt_free() { return ev_tgt_free_k[tgt_slot]; }
    bool& tgt_pending() { return tgt_pending_k[tgt_slot]; }
    DevBuf stat_norm, stat_obs, stat_world;
    // DensifyAccum (optimize.hpp:228-249), accumulated by every backward's
    // chain while enabled (gpk_densify_accum_enable)
    DevBuf acc_norm, acc_obs, acc_world;
    bool accum_on = false;
    int img_w = 0, img_h = 0;

    PrepState prep;

    // Slice contexts (batched steps, gpk_slice_context): context k >= 1 is a
    // session of its own — stream, per-slice buffers, control head, error
    // word — whose parameter, dense-gradient and Adam planes are this
    // session's (borrowed). owner is set on a context.
    gpk_session* owner = nullptr;
    std::vector<gpk_session*> ctxs;
    cudaEvent_t ev_bjoin = nullptr;  // a context's work of the batched step is done
    cudaEvent_t ev_ord = nullptr;    // a context's copies: ordered after / before its session's stream
    int ctx_used = 0;  // contexts a batched body used (graph capture snapshots their state)

    // voxelizer state (last voxelize / voxelize_backward)
    struct VoxState {
        bool valid = false;
        VoxArgs v{};
        uint64_t tiles = 0, voxels = 0;
        int passes = 0, digit_bits = 0, final_buf = 0;
    } vox;
    DevBuf vox_records, volume, dl_dv_vol, vox_partials;

    // captured step graphs (executable graph + the prepared state it leaves)
    struct Pending {
        int stage;
        cudaEvent_t a, b;
    };
    struct CtxSnap {
        gpk_session* ctx;
        PrepState prep;
        bool grads_in_slots, gmap_dirty;
    };
    struct Graph {
        cudaGraphExec_t exec;
        PrepState prep;
        std::vector<CtxSnap> ctx_state;       // batched graphs: the contexts' state they leave
        uint64_t alloc_epoch;
        bool needs_prefilter = false;  // pipelined train step: starts at K_decide
        bool sets_prefilter = false;   // ... and leaves next_pose culled
        bool writes_params = false;
        bool lazy = false;             // runs lazily (needs t_done valid at launch)
        bool lazy_writes = false;      // ... and leaves deferred steps
        bool grads_in_slots = false;   // where the graph leaves the gradient
        bool grads_in_union = false;
        bool gmap_dirty = false;
        gpk_slice_pose next_pose{};
        std::vector<Pending> timed;  // event-record nodes captured with stage timing on
    };
    bool capturing = false;
    uint64_t alloc_epoch = 0;  // bumped whenever a buffer a captured graph may use is reallocated
    std::vector<Graph> graphs;

    // live stage timing
    bool timing = false;
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double stage_ms[GPK_NUM_STAGES] = {};
    uint64_t stage_cnt[GPK_NUM_STAGES] = {};

    // persist layout
    ErrorState* err() { return persist.as<ErrorState>(); }
    unsigned* epoch() { return reinterpret_cast<unsigned*>(persist.as<char>() + 64); }
    long long* adam_step() { return reinterpret_cast<long long*>(persist.as<char>() + 72); }
    AdamConsts* adam_consts() { return reinterpret_cast<AdamConsts*>(persist.as<char>() + 128); }
    unsigned* loss_done() { return reinterpret_cast<unsigned*>(persist.as<char>() + 84); }
    double* loss() { return reinterpret_cast<double*>(persist.as<char>() + 88); }
    Control* ctrl() { return head.as<Control>(); }
    unsigned* hist() { return reinterpret_cast<unsigned*>(head.as<char>() + sizeof(Control)); }
    unsigned* prev_sort_words() { return reinterpret_cast<unsigned*>(persist.as<char>() + 96); }  // 3 words
    unsigned* grads_dirty() { return reinterpret_cast<unsigned*>(persist.as<char>() + 112); }
    unsigned* grp_begin() {
        return reinterpret_cast<unsigned*>(head.as<char>() + sizeof(Control) +
                                           kMaxSortPasses * kMaxBuckets * sizeof(unsigned));
    }
    unsigned* filter_flags() {  // u64 chunk words (8 B aligned)
        return reinterpret_cast<unsigned*>(head.as<char>() + sizeof(Control) +
                                           (kMaxSortPasses * kMaxBuckets + kGroupBeginWords) * sizeof(unsigned));
    }
};

namespace {

constexpr size_t kPersistBytes = 256 + kLazyRing * sizeof(AdamConsts) + 16;  // .., lazy ring, bad flag

cudaEvent_t take_event(gpk_session* s) {
    if (!s->event_pool.empty()) {
        cudaEvent_t e = s->event_pool.back();
        s->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Fold completed event pairs into the per-stage totals (stream synchronized).
void drain_timing(gpk_session* s) {
    for (auto& p : s->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            s->stage_ms[p.stage] += ms;
            s->stage_cnt[p.stage] += 1;
        }
        s->event_pool.push_back(p.a);
        s->event_pool.push_back(p.b);
    }
    s->pending.clear();
}

// Event pair around one stage launch when timing is enabled.
struct StageScope {
    gpk_session* s;
    int stage;
    cudaEvent_t a = nullptr;
    cudaStream_t strm;
    StageScope(gpk_session* s_, int st, cudaStream_t on = nullptr) : s(s_), stage(st), strm(on ? on : s_->stream) {
        if (!s->timing) return;
        if (s->pending.size() >= 8192 && !s->capturing) {
            cudaStreamSynchronize(strm);
            drain_timing(s);
        }
        a = take_event(s);
        // under capture: an external event node (device timestamp on replay)
        cudaEventRecordWithFlags(a, strm, s->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
    }
    void end() {
        if (!a) return;
        cudaEvent_t b = take_event(s);
        cudaEventRecordWithFlags(b, strm, s->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
        s->pending.push_back({stage, a, b});
        a = nullptr;
    }
    ~StageScope() { end(); }
};

int set_device(gpk_session* s) {
    CK(cudaSetDevice(s->device));
    return GPK_OK;
}

uint64_t filter_blocks(uint64_t n) { return std::max<uint64_t>((n + kFilterBlock - 1) / kFilterBlock, 1); }
uint64_t exact_chunks(uint64_t n) { return std::max<uint64_t>((n + kExactChunk - 1) / kExactChunk, 1); }
// head = Control | global digit histograms | digit-group begins | chunk words
// (u64), memset per prepare
size_t head_size(uint64_t n) {
    // chunk words: K_decide uses one per 4096 Gaussians, the voxelizer one per 256
    return sizeof(Control) + (kMaxSortPasses * kMaxBuckets + kGroupBeginWords) * sizeof(unsigned) +
           exact_chunks(n) * 8;
}

int clear_errors(gpk_session* s) {
    ErrorState e;
    for (int k = 0; k < 4; ++k) e.first_index[k] = ~0ull;
    CK(cudaMemcpyAsync(s->err(), &e, sizeof(e), cudaMemcpyHostToDevice, s->stream));
    return GPK_OK;
}

// Read the device error record (stream must be synchronized) and map the first
// failing primitive to the reference's exception types.
int surface_errors(gpk_session* s, const char* where) {
    ErrorState e;
    CK(cudaMemcpy(&e, s->err(), sizeof(e), cudaMemcpyDeviceToHost));
    int best = 0;
    unsigned long long idx = ~0ull;
    for (int k = 1; k < 4; ++k)
        if (e.first_index[k] < idx) {
            idx = e.first_index[k];
            best = k;
        }
    if (best == 0) return GPK_OK;
    TRY(clear_errors(s));
    CK(cudaStreamSynchronize(s->stream));
    char buf[256];
    switch (best) {
        case kErrInvalid:
            snprintf(buf, sizeof buf, "%s: invalid primitive %llu (zero-norm quaternion or non-positive scale)",
                     where, idx);
            return fail(GPK_ERR_INVALID_ARGUMENT, buf, (int64_t)idx);
        case kErrDegenerate:
            snprintf(buf, sizeof buf, "%s: non-positive det(Sigma_2d) or covariance not SPD for primitive %llu",
                     where, idx);
            return fail(GPK_ERR_DEGENERATE_COVARIANCE, buf, (int64_t)idx);
        default:
            snprintf(buf, sizeof buf, "%s: non-finite gradient for primitive %llu", where, idx);
            return fail(GPK_ERR_NUMERIC_FAILURE, buf, (int64_t)idx);
    }
}

int sync_and_check(gpk_session* s, const char* where) {
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    return surface_errors(s, where);
}

// The gradient planes were written by something other than K_chain: the next
// prepare clears them densely (see kGradsDense).
int mark_grads_dense(gpk_session* s) {
    s->prefilter.valid = false;  // a skipped K_filter would not clear them
    CK(cudaMemsetAsync(s->grads_dirty(), 0xff, 4, s->stream));
    return GPK_OK;
}

uint64_t decide_group_count(uint64_t n);

// Groups per tile row of the tile-major bucket table (sized with the set capacity).
unsigned bucket_gstride(const gpk_session* s) { return s->bucket_gs; }

// Per-sort-tile digit counts of every radix pass (kept zero between prepares:
// K_filter clears the rows the previous prepare used). A pass has one row per
// sort tile: kSortTile consecutive pair positions, or — the first pass over
// K_decide's output — one per K_decide group; the super-tile rows follow at
// row sort_tiles_cap. Sized for both, so neither the pair capacity nor the set
// size can push the group rows into the super rows.
int size_sort_status(gpk_session* s) {
    const uint64_t st_tiles = std::max<uint64_t>((s->pair_cap + kSortTile - 1) / kSortTile,
                                                 decide_group_count(std::max<uint64_t>(s->cap, 1)));
    if (st_tiles <= s->sort_tiles_cap && s->sort_status.p) return GPK_OK;
    const uint64_t region = (st_tiles + sort_supers_cap(st_tiles)) * kMaxBuckets;
    CK(s->sort_status.ensure((size_t)kMaxSortPasses * region * 4));
    CK(cudaMemsetAsync(s->sort_status.p, 0, s->sort_status.bytes, s->stream));
    CK(cudaMemsetAsync(s->prev_sort_words(), 0, 12, s->stream));
    s->sort_tiles_cap = st_tiles;
    s->hist_region = region;
    ++s->alloc_epoch;
    return GPK_OK;
}

int ensure_pairs(gpk_session* s, uint64_t need) {
    if (need <= s->pair_cap && s->keys[0].p) return GPK_OK;
    const uint64_t cap = std::max<uint64_t>(need, 1ull << 16);
    for (int b = 0; b < 2; ++b) {
        CK(s->keys[b].ensure(cap * 4));
        CK(s->vals[b].ensure(cap * 4));
    }
    CK(s->partials.ensure(cap * 24));
    CK(s->pair_recs.ensure(cap * sizeof(PairRecord)));
    ++s->alloc_epoch;
    s->pair_cap = cap;
    return size_sort_status(s);
}

// Tile starts of a multi-pass slice (written by k_pair_records).
int ensure_tile_start(gpk_session* s, uint64_t tiles) {
    const void* before = s->tile_start.p;
    CK(s->tile_start.ensure((size_t)(tiles + 1) * 4));
    if (before != s->tile_start.p) ++s->alloc_epoch;
    return GPK_OK;
}

int ensure_image(gpk_session* s, int w, int h) {
    const size_t px = (size_t)w * h;
    if (s->copy && (px * 4 > s->target_k[0].bytes || (s->target_k[1].p && px * 4 > s->target_k[1].bytes)))
        CK(cudaStreamSynchronize(s->copy));  // no copy into a freed buffer
    const void* before[3] = {s->image.p, s->dl_di.p, s->tgt().p};
    CK(s->image.ensure(px * 4));
    CK(s->dl_di.ensure(px * 4));
    CK(s->tgt().ensure(px * 4));
    const void* other = s->target_k[s->tgt_slot ^ 1].p;
    if (other) CK(s->target_k[s->tgt_slot ^ 1].ensure(px * 4));
    if (before[0] != s->image.p || before[1] != s->dl_di.p || before[2] != s->tgt().p ||
        other != s->target_k[s->tgt_slot ^ 1].p)
        ++s->alloc_epoch;
    s->img_w = w;
    s->img_h = h;
    return GPK_OK;
}

int validate_psf(const gpk_psf* psf) {
    // PsfSpec::validate (core.hpp:112-116)
    if (!(psf->sigma_x > 0.0) || !(psf->sigma_y > 0.0) || !(psf->sigma_z > 0.0) ||
        !std::isfinite(psf->sigma_x) || !std::isfinite(psf->sigma_y) || !std::isfinite(psf->sigma_z))
        return fail(GPK_ERR_INVALID_ARGUMENT, "PsfSpec: sigmas must be positive and finite");
    return GPK_OK;
}

int make_slice(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
               const gpk_raster_config* cfg, SliceArgs& a) {
    if (!pose || !psf || !cfg) return fail(GPK_ERR_INVALID_ARGUMENT, "null pose/psf/config");
    TRY(validate_psf(psf));
    if (pose->width < 1 || pose->height < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, "SlicePose: width/height must be >= 1");
    if (pose->width > 65535 || pose->height > 65535)
        return fail(GPK_ERR_INVALID_ARGUMENT, "SlicePose: width/height above 65535 unsupported");
    if (cfg->tile_size != kTile)
        return fail(GPK_ERR_INVALID_ARGUMENT, "RasterConfig: this backend supports tile_size == 16");
    if (s->n > 0 && !(cfg->scale_modifier > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT,
                    "covariance_from_scale_rotation: scale and mod must be > 0", 0);
    memset(&a, 0, sizeof a);
    bool ident = true;
    for (int i = 0; i < 9; ++i) {
        a.R[i] = pose->rotation[i];
        const double e = (i % 4 == 0) ? 1.0 : 0.0;
        if (pose->rotation[i] != e) ident = false;
    }
    for (int i = 0; i < 3; ++i) a.t[i] = pose->translation[i];
    a.sx = pose->pixel_spacing[0];
    a.sy = pose->pixel_spacing[1];
    a.inv_sx = 1.0 / a.sx;
    a.inv_sy = 1.0 / a.sy;
    a.ppx = pose->principal_point[0];
    a.ppy = pose->principal_point[1];
    a.sigma_z = psf->sigma_z;
    a.tau = cfg->tau;
    a.footprint = cfg->footprint_sigmas;
    a.mod = cfg->scale_modifier;
    a.W = pose->width;
    a.H = pose->height;
    a.tiles_x = (pose->width + kTile - 1) / kTile;
    a.tiles_y = (pose->height + kTile - 1) / kTile;
    a.identity_rot = ident ? 1 : 0;
    return GPK_OK;
}

// Radix plan for the tile key: passes of equal width <= kMaxDigitBits.
void sort_plan(int tiles, int& passes, int& digit_bits) {
    int bits = 0;
    while (bits < 32 && (1ull << bits) < (unsigned long long)tiles) ++bits;
    bits = std::max(bits, 1);  // at least one pass: it orders the K_decide groups
    passes = (bits + kMaxDigitBits - 1) / kMaxDigitBits;
    digit_bits = passes ? (bits + passes - 1) / passes : 0;
}

int launch_sorts(gpk_session* s, int passes, int digit_bits, const uint2* grp_pairs = nullptr,
                 unsigned ngroups = 0, int tile_shift = 0);
uint64_t decide_group_count(uint64_t n);
GatherLaunch gather_args(gpk_session* s);
LazyAdam lazy_args(gpk_session* s);
int lazy_flush_dev(gpk_session* s);
int lazy_sync(gpk_session* s);
int lazy_kill(gpk_session* s);
int lazy_ensure_live(gpk_session* s);
bool lazy_now(gpk_session* s);
int target_release(gpk_session* s);

// K_filter can cull lazily (from stale parameters) only with its quick test:
// an R = I pose and the cull on (launch_prep's filter_on)
bool lazy_filter_ok(const SliceArgs& a) {
    return a.identity_rot && a.tau > 0.0 && a.mod > 1e-10 && a.mod < 1e10 && a.sigma_z > 1e-10 && a.sigma_z < 1e10;
}

PrepLaunch prep_launch(gpk_session* s, const SliceArgs& a, int passes, int digit_bits, bool zero_grads) {
    PrepLaunch pl;
    pl.params = s->params.as<float>();
    pl.cap = s->cap;
    pl.n = (uint32_t)s->n;
    pl.grads = zero_grads ? s->grads.as<float>() : nullptr;
    pl.surv_params = s->surv_params.as<CandParams>();
    pl.cand = s->cand.as<CandParams>();
    pl.cand_count = s->cand_count.as<unsigned>();
    pl.grp_pairs = s->grp_pairs();
    pl.grp_surv = s->grp_surv();
    pl.surv_bits = s->surv_bits.as<unsigned>();
    pl.bucket_tab = passes == 1 ? s->bucket_tab.as<unsigned>() : nullptr;
    pl.bucket_gstride = bucket_gstride(s);
    pl.tile_begin = s->grp_begin();
    pl.grads_dirty = s->grads_dirty();
    pl.dirty_idx = s->dirty_idx.as<uint32_t>();
    pl.nfilter = (unsigned)filter_blocks(s->n);
    pl.records = s->records.as<SurvivorRecord>();
    pl.survivor_list = s->survivors.as<uint32_t>();
    pl.exact_list = s->cand_list.as<uint32_t>();
    pl.head = nullptr;
    pl.head_words = 0;
    pl.keys = s->keys[0].as<uint32_t>();
    pl.vals = s->vals[0].as<uint32_t>();
    pl.pair_cap = s->pair_cap;
    pl.hist = s->hist();
    pl.tile_hist0 = s->sort_status.as<unsigned>();
    pl.tile_hist_all = s->sort_status.as<unsigned>();
    pl.sort_tiles_cap = s->sort_tiles_cap;
    pl.hist_region = s->hist_region;
    pl.prev_sort_words = s->prev_sort_words();
    pl.passes = passes;
    pl.digit_bits = digit_bits;
    pl.exact_words = reinterpret_cast<unsigned long long*>(s->filter_flags());
    pl.ctrl = s->ctrl();
    pl.err = s->err();
    pl.slice = a;
    pl.lazy_on = 0;
    pl.lazy = lazy_args(s);
    return pl;
}

bool prefilter_matches(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                       const gpk_raster_config* cfg) {
    const auto& f = s->prefilter;
    return f.valid && f.n == s->n && std::memcmp(&f.pose, pose, sizeof *pose) == 0 &&
           std::memcmp(&f.psf, psf, sizeof *psf) == 0 && std::memcmp(&f.cfg, cfg, sizeof *cfg) == 0;
}

void set_prefilter(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf, const gpk_raster_config* cfg) {
    s->prefilter.valid = true;
    s->prefilter.pose = *pose;
    s->prefilter.psf = *psf;
    s->prefilter.cfg = *cfg;
    s->prefilter.n = s->n;
}

// A slot backward whose gradient no Adam consumed: clear its map entries (the
// survivors of the current prepared slice).
int clear_gmap(gpk_session* s) {
    if (!s->gmap_dirty) return GPK_OK;
    s->gmap_dirty = false;
    if (!s->prep.valid || s->n == 0) return GPK_OK;
    AdamLaunch c{};
    c.gmap = s->gmap.as<uint16_t>();
    c.surv_gidx = s->survivors.as<uint32_t>();
    c.grp_surv = s->grp_surv();
    launch_scatter_slot_grads(c, (unsigned)decide_group_count(s->n), kScatterClearMap, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

// filtered: K_filter's work for this slice was done already (k_filter_multi of
// a batched step: candidates, control head and sort rows are in place).
int run_prepare(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                const gpk_raster_config* cfg, bool zero_grads, bool filtered = false) {
    SliceArgs a;
    TRY(make_slice(s, pose, psf, cfg, a));
    TRY(ensure_image(s, a.W, a.H));
    if (!s->keys[0].p) TRY(ensure_pairs(s, std::max<uint64_t>(1ull << 20, 8 * s->n)));
    if (s->owner) TRY(lazy_kill(s->owner));  // a context's cull reads its session's parameters
    PrepState& ps = s->prep;
    ps.slice = a;
    ps.tiles = a.tiles_x * a.tiles_y;
    if (ps.tiles > (1 << (kMaxDigitBits * kMaxSortPasses)))
        return fail(GPK_ERR_INVALID_ARGUMENT, "SlicePose: more than 2^20 tiles unsupported");
    sort_plan(ps.tiles, ps.passes, ps.digit_bits);
    if (ps.passes > 1) TRY(ensure_tile_start(s, ps.tiles));
    ps.pose = *pose;
    ps.psf = *psf;
    ps.cfg = *cfg;
    ps.valid = true;
    ps.rasterized = false;
    TRY(clear_gmap(s));  // before the survivor slots change
    ps.grads_zeroed = zero_grads;
    ps.ssim_pending = false;
    s->grads_in_slots = false;  // the survivor slots are about to change
    const uint64_t nbf = filter_blocks(s->n);
    const size_t head_bytes = head_size(s->n);
    StageScope scope_prep(s, GPK_STAGE_PREPARE);
    if (s->n == 0) {
        CK(cudaMemsetAsync(s->head.p, 0, head_bytes, s->stream));
        ps.final_buf = 0;
        return GPK_OK;
    }
    PrepLaunch pl = prep_launch(s, a, ps.passes, ps.digit_bits, zero_grads);
    // K_filter is skipped when the previous training step's fused Adam + cull
    // already produced this slice's candidates (and left the gradients zero)
    const bool pre = zero_grads && (s->assume_prefiltered || prefilter_matches(s, pose, psf, cfg));
    s->prefilter.valid = false;
    if (filtered) {
        // k_filter_multi culled this slice and zeroed its control head
    } else if (!pre) {
        // K_filter zeroes the control head itself (K_decide is the first to use it)
        pl.head = s->head.as<unsigned>();
        pl.head_words = (unsigned)(head_bytes / 4);
        // lazy: K_filter culls from the stored parameters and replays what it
        // keeps; a pose its drift test cannot take gets every deferred step first
        pl.lazy_on = lazy_now(s) ? 1 : 0;
        if (pl.lazy_on && !lazy_filter_ok(a)) {
            TRY(lazy_flush_dev(s));
            if (!s->capturing) s->lazy_pending = false;
            pl.lazy_on = 0;
        }
        if (pl.lazy_on && s->capturing) s->cap_lazy_used = true;
        launch_prep(pl, s->num_sms, s->stream);
        CK(cudaGetLastError());
        pl.head = nullptr;
    } else {
        CK(cudaMemsetAsync(s->head.p, 0, head_bytes, s->stream));
    }
    scope_prep.end();
    {
        StageScope scope_bin(s, GPK_STAGE_BIN);
        launch_bin(pl, s->num_sms, s->stream);
        CK(cudaGetLastError());
    }
    ps.lists_pending = false;
    if (ps.passes == 1 && s->fuse_gather) {
        ps.lists_pending = true;  // the training step's forward gathers its tile lists
    } else if (ps.passes == 1) {
        // every tile is one digit: gather the K_decide buckets instead of a radix pass
        StageScope scope_sort(s, GPK_STAGE_SORT);
        launch_gather(gather_args(s), s->stream);
        CK(cudaGetLastError());
    } else {
        StageScope scope_sort(s, GPK_STAGE_SORT);
        TRY(launch_sorts(s, ps.passes, ps.digit_bits, s->grp_pairs(), (unsigned)decide_group_count(s->n)));
        const int fb = ps.passes & 1;
        launch_pair_records(s->keys[fb].as<uint32_t>(), s->vals[fb].as<uint32_t>(), s->records.as<SurvivorRecord>(),
                            s->pair_recs.as<PairRecord>(), s->tile_start.as<unsigned>(), s->ctrl(), s->pair_cap, a,
                            s->num_sms, s->stream);
        CK(cudaGetLastError());
    }
    ps.final_buf = ps.passes & 1;
    return GPK_OK;
}

uint64_t decide_group_count(uint64_t n) { return (filter_blocks(n) + kDecideChunks - 1) / kDecideChunks; }

// Stable LSD radix passes over the (key, value) pairs in keys[0]/vals[0].
// Position tiles of the voxelizer's radix passes: kSortTile << shift keys, at
// most 4k tiles per pass over its capacity-sized pair list. Every tile reads up
// to 16 digit-count rows (its super-row prefix and the earlier tiles of its
// super-tile), so at C4 (7.9M pairs) 1k-key tiles spend as many L2 bytes on the
// rows as on the keys; 2k-4k-key tiles measured fastest (1k-tile cap: +120 us).
// The slice passes keep 1024-key tiles.
int sort_tile_shift(uint64_t pair_cap) {
    int shift = 0;
    while (((pair_cap + ((uint64_t)kSortTile << shift) - 1) >> (10 + shift)) > 4096 && shift < 12) ++shift;
    return shift;
}

int launch_sorts(gpk_session* s, int passes, int digit_bits, const uint2* grp_pairs, unsigned ngroups,
                 int tile_shift) {
    const int grid = (int)std::max<uint64_t>(
        1, std::min<uint64_t>(std::max<uint64_t>(s->sort_tiles_cap, ngroups), (uint64_t)s->num_sms * 4));
    const size_t region = s->hist_region;
    for (int p = 0; p < passes; ++p) {
        SortLaunch sl;
        sl.keys_in = s->keys[p & 1].as<uint32_t>();
        sl.vals_in = s->vals[p & 1].as<uint32_t>();
        sl.keys_out = s->keys[(p + 1) & 1].as<uint32_t>();
        sl.vals_out = s->vals[(p + 1) & 1].as<uint32_t>();
        sl.hist = s->hist() + kMaxBuckets * p;
        sl.tile_hist = s->sort_status.as<unsigned>() + (size_t)p * region;
        sl.tile_hist_next = (p + 1 < passes) ? s->sort_status.as<unsigned>() + (size_t)(p + 1) * region
                                                : nullptr;
        sl.prev_sort_words = s->prev_sort_words();
        sl.grp_begin = (p + 1 == passes) ? s->grp_begin() : nullptr;
        sl.sort_tiles_cap = s->sort_tiles_cap;
        sl.shift = digit_bits * p;
        sl.tile_shift = tile_shift;
        sl.bits = digit_bits;
        sl.next_buckets = 1u << digit_bits;
        sl.pass = p;
        sl.ctrl = s->ctrl();
        sl.pair_cap = s->pair_cap;
        sl.grp_pairs = p == 0 ? grp_pairs : nullptr;
        sl.ngroups = ngroups;
        launch_super_scan(s->sort_status.as<unsigned>() + (size_t)p * region, s->sort_tiles_cap, 1u << digit_bits,
                          s->ctrl(), s->pair_cap, p == 0 && grp_pairs ? ngroups : 0u,
                          (unsigned)kSortTile << tile_shift, s->stream);
        CK(cudaGetLastError());
        launch_sort_pass(sl, grid, s->stream);
        CK(cudaGetLastError());
    }
    return GPK_OK;
}

RasterLaunch raster_args(gpk_session* s) {
    RasterLaunch r;
    r.records = s->records.as<SurvivorRecord>();
    r.keys = s->keys[s->prep.final_buf].as<uint32_t>();
    r.vals = s->vals[s->prep.final_buf].as<uint32_t>();
    r.grp_begin = s->prep.passes > 1 ? s->tile_start.as<unsigned>() : s->grp_begin();
    r.grp_shift = s->prep.passes ? 0 : -1;
    r.ctrl = s->ctrl();
    r.pair_cap = s->pair_cap;
    r.image = s->image.as<float>();
    r.dl_di = s->dl_di.as<float>();
    r.partials = s->partials.as<float>();
    r.slice = s->prep.slice;
    r.ssim_g = s->prep.ssim_pending ? s->loss_g.as<float>() : nullptr;
    r.target = s->tgt().as<float>();
    r.ssim_k = s->prep.ssim_k;
    r.inv_n = s->prep.inv_n;
    for (int t = 0; t < 11; ++t) r.w[t] = s->prep.w[t];
    r.bucket_tab = nullptr;
    r.ngroups = (unsigned)decide_group_count(s->n);
    r.gstride = bucket_gstride(s);
    r.vals_in = s->vals[0].as<uint32_t>();
    r.vals_out = s->vals[1].as<uint32_t>();
    r.pairs = s->pair_recs.as<PairRecord>();
    r.fin = s->prep.ssim_pending ? s->prep.fin : LossFinish{};
    return r;
}

GatherLaunch gather_args(gpk_session* s) {
    GatherLaunch gl;
    gl.bucket_tab = s->bucket_tab.as<unsigned>();
    gl.ngroups = (unsigned)decide_group_count(s->n);
    gl.ntiles = (unsigned)s->prep.tiles;
    gl.gstride = bucket_gstride(s);
    gl.tile_begin = s->grp_begin();
    gl.vals_in = s->vals[0].as<uint32_t>();
    gl.vals_out = s->vals[1].as<uint32_t>();
    gl.ctrl = s->ctrl();
    gl.pair_cap = s->pair_cap;
    gl.records = s->records.as<SurvivorRecord>();
    gl.pairs = s->pair_recs.as<PairRecord>();
    gl.slice = s->prep.slice;
    return gl;
}

// The tile lists exist (a fused-gather prepare left them to the forward).
int ensure_lists(gpk_session* s) {
    if (!s->prep.lists_pending) return GPK_OK;
    s->prep.lists_pending = false;
    StageScope scope(s, GPK_STAGE_SORT);
    launch_gather(gather_args(s), s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

int run_rasterize(gpk_session* s, cudaStream_t on = nullptr) {
    if (!s->prep.valid) return fail(GPK_ERR_STATE, "rasterize: no prepared slice");
    const size_t px = (size_t)s->img_w * s->img_h;
    cudaStream_t st = on ? on : s->stream;
    StageScope scope(s, GPK_STAGE_RASTER, st);
    if (s->n == 0) {
        CK(cudaMemsetAsync(s->image.p, 0, px * 4, st));
    } else {
        RasterLaunch r = raster_args(s);
        if (s->prep.lists_pending) {
            if (st != s->stream) return fail(GPK_ERR_STATE, "rasterize: tile lists pending on another stream");
            r.bucket_tab = s->bucket_tab.as<unsigned>();  // the forward gathers its lists
            s->prep.lists_pending = false;
        }
        launch_raster_fwd(r, st);
        CK(cudaGetLastError());
    }
    s->prep.rasterized = true;
    return GPK_OK;
}

// slots: the chain writes the gradient by survivor slot (single-GPU training
// step: Adam reads it there) instead of into the dense planes.
// union: the chain writes the data-parallel union rows (train_dp_body).
int run_backward(gpk_session* s, bool stats, bool slots = false, bool urows = false) {
    if (!s->prep.valid) return fail(GPK_ERR_STATE, "backward: no prepared slice");
    s->prefilter.valid = false;  // the chain writes gradients
    TRY(clear_gmap(s));
    TRY(ensure_lists(s));
    s->grads_in_union = urows && s->n;
    s->grads_in_slots = slots && !urows && s->n;
    s->gmap_dirty = s->grads_in_slots;
    if (s->n == 0) return GPK_OK;
    if (!slots && !s->prep.grads_zeroed) {
        CK(cudaMemsetAsync(s->grads.p, 0, s->cap * 11 * 4, s->stream));
        CK(cudaMemsetAsync(s->grads_dirty(), 0, 4, s->stream));
    }
    if (stats) {
        CK(s->stat_norm.ensure(s->cap * 4));
        CK(s->stat_obs.ensure(s->cap));
        CK(s->stat_world.ensure(s->cap * 12));
        CK(cudaMemsetAsync(s->stat_norm.p, 0, s->cap * 4, s->stream));
        CK(cudaMemsetAsync(s->stat_obs.p, 0, s->cap, s->stream));
        CK(cudaMemsetAsync(s->stat_world.p, 0, s->cap * 12, s->stream));
    }
    {
        StageScope scope(s, GPK_STAGE_BACKWARD);
        const bool reads_target = s->prep.ssim_pending;
        launch_raster_bwd(raster_args(s), s->stream);
        CK(cudaGetLastError());
        s->prep.ssim_pending = false;
        s->prep.fin = LossFinish{};
        if (reads_target) TRY(target_release(s));
    }
    StageScope scope(s, GPK_STAGE_CHAIN);
    ChainLaunch c;
    c.sparams = s->surv_params.as<CandParams>();
    c.dirty_idx = s->dirty_idx.as<uint32_t>();
    c.grads_dirty = s->grads_dirty();
    c.cap = s->cap;
    c.records = s->records.as<SurvivorRecord>();
    c.survivor_list = s->survivors.as<uint32_t>();
    c.partials = s->partials.as<float>();
    c.ctrl = s->ctrl();
    c.grads = s->grads.as<float>();
    c.slot_grads = slots ? s->slot_grads.as<float>() : nullptr;
    c.gmap = s->gmap.as<uint16_t>();
    c.umap = urows ? s->umap.as<uint32_t>() : nullptr;
    c.urows = urows ? s->urows.as<float>() : nullptr;
    c.ucap = s->ucap;
    c.stat_norm = stats ? s->stat_norm.as<float>() : nullptr;
    c.stat_observed = stats ? s->stat_obs.as<uint8_t>() : nullptr;
    c.stat_world = stats ? s->stat_world.as<float>() : nullptr;
    c.acc_norm = s->accum_on ? s->acc_norm.as<double>() : nullptr;
    c.acc_obs = s->accum_on ? s->acc_obs.as<int>() : nullptr;
    c.acc_world = s->accum_on ? s->acc_world.as<double>() : nullptr;
    c.exact_list = s->cand_list.as<uint32_t>();  // deferral list (record slots)
    c.exact_count = &s->ctrl()->chain_exact;
    c.grp_surv = s->grp_surv();
    c.dirty_ctr = &s->ctrl()->dirty_ctr;
    c.err = s->err();
    c.slice = s->prep.slice;
    // K_chain_exact (the few fp64-decided survivors) beside K_chain
    const int groups = (int)decide_group_count(s->n);
    CK(cudaEventRecord(s->ev_xfork, s->stream));
    CK(cudaStreamWaitEvent(s->side, s->ev_xfork, 0));
    launch_chain_exact(c, groups, s->side);
    CK(cudaGetLastError());
    CK(cudaEventRecord(s->ev_xjoin, s->side));
    launch_chain(c, groups, s->num_sms, s->stream);
    CK(cudaGetLastError());
    CK(cudaStreamWaitEvent(s->stream, s->ev_xjoin, 0));
    return GPK_OK;
}

// U1 with dL/dI already in GPK_BUF_DL_DI: the forward does not feed the
// backward, so it runs on the side stream while the backward (+ chain) runs on
// the session stream; the session stream then waits for the forward.
int run_fwd_bwd_forked(gpk_session* s, bool slots = false) {
    CK(cudaEventRecord(s->ev_fork, s->stream));
    CK(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    TRY(run_rasterize(s, s->side));
    CK(cudaEventRecord(s->ev_join, s->side));
    TRY(run_backward(s, false, slots));
    CK(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
    return GPK_OK;
}

// Synchronize; if the slice produced more pairs than the buffers hold, grow
// them and replay prepare (+ rasterize). Returns GPK_OK when the prepared
// state is complete.
int settle_pairs(gpk_session* s) {
    CK(cudaStreamSynchronize(s->stream));
    Control c;
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    if (!c.pair_overflow) return GPK_OK;
    TRY(ensure_pairs(s, (uint64_t)c.pairs + c.pairs / 4 + 1024));
    const bool ras = s->prep.rasterized;
    const PrepState saved = s->prep;
    TRY(run_prepare(s, &saved.pose, &saved.psf, &saved.cfg, saved.grads_zeroed));
    if (ras) TRY(run_rasterize(s));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    if (c.pair_overflow) return fail(GPK_ERR_STATE, "pair capacity still exceeded after growth");
    return GPK_OK;
}

// Host records (n x 11 f32) -> 11 device planes of stride cap: one H2D copy of
// the record block into a staging buffer, then the transpose kernel.
int copy_records_in(gpk_session* s, uint64_t n, const float* rec, float* planes) {
    DevBuf stage;
    CK(stage.ensure(n * 44));
    CK(cudaMemcpyAsync(stage.p, rec, n * 44, cudaMemcpyHostToDevice, s->stream));
    launch_records_to_planes(stage.as<float>(), n, planes, s->cap, s->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));  // before the staging buffer is freed
    return GPK_OK;
}

int copy_params_in(gpk_session* s, uint64_t n, const float* rec) {
    return copy_records_in(s, n, rec, s->params.as<float>());
}

// 11 device planes -> host records: transpose into a staging buffer, one D2H copy.
int copy_planes_out(gpk_session* s, const float* dev, float* rec) {
    const uint64_t n = s->n;
    DevBuf stage;
    CK(stage.ensure(n * 44));
    launch_planes_to_records(dev, s->cap, n, stage.as<float>(), s->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(rec, stage.p, n * 44, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return GPK_OK;
}

// DensifyAccum::reset(n) on the device (optimize.hpp:234-238)
int accum_alloc_zero(gpk_session* s) {
    CK(s->acc_norm.ensure(s->cap * 8));
    CK(s->acc_obs.ensure(s->cap * 4));
    CK(s->acc_world.ensure(s->cap * 24));
    CK(cudaMemsetAsync(s->acc_norm.p, 0, s->cap * 8, s->stream));
    CK(cudaMemsetAsync(s->acc_obs.p, 0, s->cap * 4, s->stream));
    CK(cudaMemsetAsync(s->acc_world.p, 0, s->cap * 24, s->stream));
    return GPK_OK;
}

// Per-slice buffers sized for a plane stride `cap` (survivor records, candidates,
// K_decide tables, slot gradients and their map, the control head).
int alloc_slice_bufs(gpk_session* s, uint64_t cap) {
    const uint64_t nbf = filter_blocks(cap);
    CK(s->records.ensure(cap * sizeof(SurvivorRecord)));
    CK(s->cand_list.ensure(cap * 4));
    CK(s->surv_params.ensure(cap * sizeof(CandParams)));
    CK(s->grp_table.ensure((cap / kDecideGroupSize + 2) * 12));
    CK(s->bucket_tab.ensure((cap / kDecideGroupSize + 2) * (kMaxBuckets + 1) * 4));
    s->bucket_gs = (unsigned)(cap / kDecideGroupSize + 2);
    CK(s->cand.ensure(cap * sizeof(CandParams)));
    CK(s->cand_count.ensure(nbf * 4));
    CK(s->dirty_idx.ensure(cap * 4));
    CK(s->slot_grads.ensure(cap * 11 * 4));
    CK(s->gmap.ensure(cap * 2));
    CK(cudaMemsetAsync(s->gmap.p, 0, cap * 2, s->stream));
    s->grads_in_slots = false;
    s->grads_in_union = false;
    s->gmap_dirty = false;
    TRY(mark_grads_dense(s));
    CK(s->survivors.ensure(cap * 4));
    CK(s->surv_bits.ensure(cap / 8 + 512));
    CK(s->head.ensure(head_size(cap)));
    s->cap = cap;
    ++s->alloc_epoch;
    if (s->keys[0].p) TRY(size_sort_status(s));  // more K_decide groups than sort-tile rows
    return GPK_OK;
}

int alloc_for_n(gpk_session* s, uint64_t n) {
    if (s->owner) return fail(GPK_ERR_STATE, "slice context: the Gaussian set belongs to its session");
    // plane stride: a multiple of the K_filter chunk, so every chunk's plane
    // slice is a 4 KB, 16 B-aligned TMA bulk-copy source/destination
    const uint64_t cap = (std::max<uint64_t>(n, 1) + kParamAlign - 1) / kParamAlign * kParamAlign;
    if (cap > s->cap || !s->params.p) {
        CK(s->params.ensure(cap * 11 * 4));
        CK(s->grads.ensure(cap * 11 * 4));
        CK(s->adam_m.ensure(cap * 11 * 4));
        CK(s->adam_v.ensure(cap * 11 * 4));
        CK(s->t_done.ensure(cap * 4));
        TRY(alloc_slice_bufs(s, cap));
    }
    if (n != s->n) ++s->alloc_epoch;  // captured graphs bake the set size
    s->lazy_live = false;  // (callers flushed what was deferred)
    s->lazy_pending = false;
    s->n = n;
    if (s->accum_on) TRY(accum_alloc_zero(s));
    return GPK_OK;
}

int adam_reset(gpk_session* s) {
    CK(cudaMemsetAsync(s->adam_m.p, 0, s->cap * 11 * 4, s->stream));
    CK(cudaMemsetAsync(s->adam_v.p, 0, s->cap * 11 * 4, s->stream));
    CK(cudaMemsetAsync(s->adam_step(), 0, 16, s->stream));
    return GPK_OK;
}

int materialize_dense_grads(gpk_session* s);

// Adam's gradient: the slot planes of the last training step's backward while
// its map is intact (Adam consumes the map), else the dense planes (the slot
// gradient scattered into them first if it is the latest).
int adam_grad_source(gpk_session* s, AdamLaunch& a) {
    const bool slots = s->grads_in_slots && s->gmap_dirty && s->prep.valid;
    if (!slots) TRY(materialize_dense_grads(s));
    a.slot_grads = slots ? s->slot_grads.as<float>() : nullptr;
    a.gmap = s->gmap.as<uint16_t>();
    a.surv_gidx = s->survivors.as<uint32_t>();
    a.grp_surv = s->grp_surv();
    if (slots) s->gmap_dirty = false;
    return GPK_OK;
}

// Make the dense planes hold the latest gradient (API readers and writers of
// GPK_BUF_GRADS, the all-reduce): scatter the slot gradient if it lives there.
int materialize_dense_grads(gpk_session* s) {
    if (s->grads_in_union) {  // a data-parallel step's summed gradient: its union rows, densely
        s->grads_in_union = false;
        if (s->capturing) return fail(GPK_ERR_STATE, "gradient layout change during capture");
        launch_union_to_dense(s->umap.as<uint32_t>(), s->urows.as<float>(), s->cap, (uint32_t)s->n, s->ucap,
                              s->grads.as<float>(), s->stream);
        CK(cudaGetLastError());
        return mark_grads_dense(s);
    }
    if (!s->grads_in_slots) return GPK_OK;
    s->grads_in_slots = false;
    if (!s->prep.valid || s->n == 0) return GPK_OK;
    if (s->capturing) return fail(GPK_ERR_STATE, "gradient layout change during capture");
    CK(cudaMemsetAsync(s->grads.p, 0, s->cap * 11 * 4, s->stream));
    AdamLaunch a{};
    a.grads = s->grads.as<float>();
    a.cap = s->cap;
    a.slot_grads = s->slot_grads.as<float>();
    a.surv_gidx = s->survivors.as<uint32_t>();
    a.grp_surv = s->grp_surv();
    launch_scatter_slot_grads(a, (unsigned)decide_group_count(s->n), kScatterSet, s->stream);
    CK(cudaGetLastError());
    return mark_grads_dense(s);
}

LazyAdam lazy_args(gpk_session* s) {
    LazyAdam L{};
    L.t_done = s->t_done.as<uint32_t>();
    L.ring = s->lazy_on ? s->lazy_ring() : nullptr;  // (k_adam_consts fills it in lazy mode only)
    L.step = s->adam_step();
    L.m = s->adam_m.as<float>();
    L.v = s->adam_v.as<float>();
    L.bad = s->lazy_bad();
    for (int d = 0; d < 3; ++d) {
        L.bbox_min[d] = (float)s->bbox.min[d];
        L.bbox_max[d] = (float)s->bbox.max[d];
    }
    return L;
}

AdamLaunch adam_launch(gpk_session* s, const double lr[4], bool scheduled, int total, const gpk_adam_hparams* hp) {
    AdamLaunch a{};
    a.params = s->params.as<float>();
    a.grads = s->grads.as<float>();
    a.m = s->adam_m.as<float>();
    a.v = s->adam_v.as<float>();
    a.cap = s->cap;
    a.n = (uint32_t)s->n;
    for (int d = 0; d < 3; ++d) {
        a.bbox_min[d] = (float)s->bbox.min[d];
        a.bbox_max[d] = (float)s->bbox.max[d];
    }
    for (int k = 0; k < 4; ++k) a.lr[k] = lr[k];
    a.scheduled = scheduled ? 1 : 0;
    a.total = total;
    a.beta1 = hp ? hp->beta1 : 0.9;
    a.beta2 = hp ? hp->beta2 : 0.999;
    a.eps = hp ? hp->eps : 1e-8;
    a.step = s->adam_step();
    a.consts = s->adam_consts();
    a.ctrl = s->prep.valid ? s->ctrl() : nullptr;
    a.lazy = lazy_args(s);
    return a;
}

// ---- lazy training steps (LazyAdam, common.cuh) ---------------------------------
// Host rules: lazy_sync before anything reads the parameters or moments
// directly (every deferred step replayed), lazy_kill before anything writes
// them or runs an eager Adam step (t_done is then no longer maintained), and
// lazy_ensure_live before a lazy step. Under capture nothing changes on the
// host: the graph records whether it runs lazily and gpk_graph_launch applies
// the rules at launch.
int lazy_flush_dev(gpk_session* s) {
    if (!s->n) return GPK_OK;
    const double lr[4] = {0, 0, 0, 0};
    launch_lazy_flush(adam_launch(s, lr, false, 1, nullptr), s->stream);
    CK(cudaGetLastError());
    if (s->capturing) s->cap_lazy_used = true;
    return GPK_OK;
}

int lazy_sync(gpk_session* s) {
    if (s->owner) return lazy_sync(s->owner);
    if (s->capturing || !s->lazy_live || !s->lazy_pending) return GPK_OK;
    TRY(lazy_flush_dev(s));
    s->lazy_pending = false;
    return GPK_OK;
}

int lazy_kill(gpk_session* s) {
    if (s->owner) return lazy_kill(s->owner);
    if (s->capturing) return GPK_OK;
    TRY(lazy_sync(s));
    s->lazy_live = false;
    return GPK_OK;
}

int lazy_ensure_live(gpk_session* s) {
    if (s->capturing || s->lazy_live) return GPK_OK;
    if (s->n) {
        CK(cudaMemsetAsync(s->lazy_bad(), 0, 4, s->stream));
        const double lr[4] = {0, 0, 0, 0};
        launch_lazy_begin(adam_launch(s, lr, false, 1, nullptr), s->stream);
        CK(cudaGetLastError());
    }
    s->lazy_live = true;
    s->lazy_pending = false;
    return GPK_OK;
}

// K_filter of this prepare runs lazily
bool lazy_now(gpk_session* s) { return !s->owner && (s->capturing ? s->cap_lazy : s->lazy_live); }

// The training step evaluates the Adam constants (fp64 pow latency) on the
// side stream while the slice renders; the update waits on ev_cjoin.
int adam_consts_ahead(gpk_session* s, const AdamLaunch& a) {
    CK(cudaEventRecord(s->ev_cfork, s->stream));
    CK(cudaStreamWaitEvent(s->side, s->ev_cfork, 0));
    launch_adam_consts(a, s->side);
    CK(cudaGetLastError());
    CK(cudaEventRecord(s->ev_cjoin, s->side));
    s->consts_pending = true;
    return GPK_OK;
}

int adam_consts_ready(gpk_session* s, const AdamLaunch& a) {
    if (s->consts_pending) {
        s->consts_pending = false;
        CK(cudaStreamWaitEvent(s->stream, s->ev_cjoin, 0));
        return GPK_OK;
    }
    launch_adam_consts(a, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

// lo, hi: the primitives to update (a data-parallel rank's shard), default all
int run_adam(gpk_session* s, const double lr[4], bool scheduled, int total,
             const gpk_adam_hparams* hp, uint64_t lo = 0, uint64_t hi = ~0ull) {
    if (s->owner) return fail(GPK_ERR_STATE, "slice context: Adam runs on its session");
    TRY(lazy_kill(s));  // the eager update over all N
    if (s->n == 0) {
        s->consts_pending = false;
        long long st = 0;
        CK(cudaMemcpyAsync(&st, s->adam_step(), 8, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        ++st;
        CK(cudaMemcpyAsync(s->adam_step(), &st, 8, cudaMemcpyHostToDevice, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        return GPK_OK;
    }
    AdamLaunch a = adam_launch(s, lr, scheduled, total, hp);
    a.lo = (uint32_t)std::min<uint64_t>(lo, s->n);
    a.n = (uint32_t)std::min<uint64_t>(hi, s->n);
    TRY(adam_grad_source(s, a));
    s->prefilter.valid = false;  // the parameters change
    StageScope scope(s, GPK_STAGE_ADAM);
    TRY(adam_consts_ready(s, a));
    launch_adam(a, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

// Adam fused with the next slice's K_filter (the training step's last kernel):
// leaves `next` culled for the following prepare and every gradient zero.
int run_adam_cull(gpk_session* s, const double lr[4], int total, const gpk_slice_pose* next,
                  const gpk_psf* psf, const gpk_raster_config* cfg) {
    TRY(lazy_kill(s));
    SliceArgs na;
    TRY(make_slice(s, next, psf, cfg, na));
    if (s->n == 0) return run_adam(s, lr, true, total, nullptr);
    int passes = 0, digit_bits = 0;
    sort_plan(na.tiles_x * na.tiles_y, passes, digit_bits);
    const PrepLaunch f = prep_launch(s, na, passes, digit_bits, true);
    AdamLaunch a = adam_launch(s, lr, true, total, nullptr);
    TRY(adam_grad_source(s, a));
    StageScope scope(s, GPK_STAGE_ADAM);
    TRY(adam_consts_ready(s, a));
    launch_adam_cull(a, f, s->stream);
    CK(cudaGetLastError());
    set_prefilter(s, next, psf, cfg);
    return GPK_OK;
}

// Before the session stream reads or writes the target: the uploaded slice
// target has landed. Captured graphs always wait on ev_tgt_ready (an external
// event node: resolved at each launch against the latest upload).
int target_wait(gpk_session* s) {
    if (s->capturing) {
        CK(cudaStreamWaitEvent(s->stream, s->ev_tgt_ready(), cudaEventWaitExternal));
        return GPK_OK;
    }
    if (s->tgt_pending()) {
        CK(cudaStreamWaitEvent(s->stream, s->ev_tgt_ready(), 0));
        s->tgt_pending() = false;
    }
    return GPK_OK;
}

// Everything queued so far that reads the target is done when ev_tgt_free
// completes (an external record node under capture: each launch re-records it).
int target_release(gpk_session* s) {
    if (!s->capturing) {
        CK(cudaEventRecord(s->ev_tgt_free(), s->stream));
        return GPK_OK;
    }
    CK(cudaEventRecord(s->ev_rel_fork, s->stream));
    CK(cudaStreamWaitEvent(s->rel_stream, s->ev_rel_fork, 0));
    CK(cudaEventRecordWithFlags(s->ev_tgt_free(), s->rel_stream, cudaEventRecordExternal));
    CK(cudaEventRecord(s->ev_rel_join, s->rel_stream));
    s->rel_join_pending = true;
    return GPK_OK;
}

int run_loss(gpk_session* s, double lambda, double dssim_scale, bool fuse_into_backward = false) {
    if (!s->prep.rasterized) return fail(GPK_ERR_STATE, "photometric_loss: no rendered image");
    const int W = s->img_w, H = s->img_h;
    const size_t px = (size_t)W * H;
    const void* before[2] = {s->loss_g.p, s->loss_partial.p};
    if (lambda != 0.0) CK(s->loss_g.ensure(px * 12));
    CK(s->loss_partial.ensure((size_t)loss_partial_blocks(W, H, lambda) * 16));
    if (before[0] != s->loss_g.p || before[1] != s->loss_partial.p) {
        if (s->capturing) return fail(GPK_ERR_STATE, "loss buffers must be sized before capture");
        ++s->alloc_epoch;
    }
    LossLaunch l;
    l.image = s->image.as<float>();
    l.target = s->tgt().as<float>();
    l.dl_di = s->dl_di.as<float>();
    l.g = s->loss_g.as<float>();
    l.partial = s->loss_partial.as<double>();
    l.loss = s->loss();
    l.loss_host = s->loss_sink;
    l.done_ctr = s->loss_done();
    l.W = W;
    l.H = H;
    l.lambda = lambda;
    l.dssim_scale = dssim_scale;
    // gaussian_window(5, 1.5) (metrics.hpp:66-75)
    double w[11], sum = 0.0;
    for (int t = -5; t <= 5; ++t) {
        w[t + 5] = std::exp(-0.5 * t * t / (1.5 * 1.5));
        sum += w[t + 5];
    }
    for (int t = 0; t < 11; ++t) l.w[t] = (float)(w[t] / sum);
    TRY(target_wait(s));
    StageScope scope(s, GPK_STAGE_LOSS);
    const bool fuse = fuse_into_backward && lambda != 0.0;
    // the raster backward (which follows at once) finishes the loss: no
    // last-CTA ticket in k_ssim_fwd (an empty set runs no backward kernel)
    l.finish_in_fwd = fuse && (s->n == 0 || s->loss_in_fwd) ? 1 : 0;
    s->prep.fin = LossFinish{};
    if (fuse) {
        launch_loss_fwd_only(l, s->stream);
        if (!l.finish_in_fwd) {
            LossFinish& f = s->prep.fin;
            f.partial = l.partial;
            f.nblk = loss_partial_blocks(W, H, lambda);
            f.with_ssim = 1;
            f.inv_n = 1.0 / ((double)W * (double)H);
            f.lambda = lambda;
            f.dssim_scale = dssim_scale;
            f.loss = l.loss;
            f.loss_host = l.loss_host;
        }
        s->prep.ssim_pending = true;
        s->prep.ssim_k = (float)(lambda * dssim_scale);
        s->prep.inv_n = (float)(1.0 / (double)px);
        for (int t = 0; t < 11; ++t) s->prep.w[t] = l.w[t];
    } else {
        launch_loss(l, s->stream);
    }
    CK(cudaGetLastError());
    if (!fuse) TRY(target_release(s));  // (fused: the raster backward reads it last)
    return GPK_OK;
}


// ---- voxelizer (voxelize.hpp:16-240) --------------------------------------------

// VoxelizerConfig::validate (voxelize.hpp:24-37) + this backend's index limits.
int make_vox(gpk_session* s, const gpk_voxelizer_config* cfg, VoxArgs& v) {
    if (!cfg) return fail(GPK_ERR_INVALID_ARGUMENT, "null voxelizer config");
    if (cfg->dims[0] < 1 || cfg->dims[1] < 1 || cfg->dims[2] < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: dims must be >= 1");
    if (cfg->tile_dims[0] < 1 || cfg->tile_dims[1] < 1 || cfg->tile_dims[2] < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: tile_dims must be >= 1");
    if (!(cfg->support_sigmas > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: support_sigmas must be > 0");
    if (!(cfg->spacing[0] > 0.0) || !(cfg->spacing[1] > 0.0) || !(cfg->spacing[2] > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: spacing must be positive");
    const uint64_t voxels = (uint64_t)cfg->dims[0] * cfg->dims[1] * cfg->dims[2];
    if (voxels > (1ull << 31)) return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: refusing > 2^31 voxels");
    if (cfg->dims[0] > 65535 || cfg->dims[1] > 65535 || cfg->dims[2] > 65535)
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: dims above 65535 unsupported");
    if (s->n > 0 && !(cfg->scale_modifier > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT, "covariance_from_scale_rotation: scale and mod must be > 0", 0);
    memset(&v, 0, sizeof v);
    uint64_t tiles = 1;
    for (int d = 0; d < 3; ++d) {
        v.dims[d] = cfg->dims[d];
        v.tile[d] = std::min(cfg->tile_dims[d], cfg->dims[d]);  // same tiling, fewer empty lanes
        v.ntiles[d] = (cfg->dims[d] + cfg->tile_dims[d] - 1) / cfg->tile_dims[d];
        v.spacing[d] = cfg->spacing[d];
        v.origin[d] = cfg->origin[d];
        tiles *= (uint64_t)v.ntiles[d];
    }
    if (tiles > (1ull << (kMaxDigitBits * kMaxSortPasses)))
        return fail(GPK_ERR_INVALID_ARGUMENT, "VoxelizerConfig: more than 2^20 voxel tiles unsupported");
    v.support = cfg->support_sigmas;
    v.mod = cfg->scale_modifier;
    return GPK_OK;
}

// prepare_voxel_prims + VoxelTiles (voxelize.hpp:52-105): records, survivor
// list, (tile, primitive) pairs sorted stably by tile.
int run_vox_prep(gpk_session* s, const gpk_voxelizer_config* cfg) {
    VoxArgs v;
    TRY(make_vox(s, cfg, v));
    TRY(lazy_sync(s));  // the voxelizer reads the parameters directly
    if (!s->keys[0].p) TRY(ensure_pairs(s, std::max<uint64_t>(1ull << 20, 8 * s->n)));
    s->prep.valid = false;  // the pair buffers now hold voxel tiles
    s->prep.rasterized = false;
    auto& vs = s->vox;
    vs.v = v;
    vs.tiles = (uint64_t)v.ntiles[0] * v.ntiles[1] * v.ntiles[2];
    vs.voxels = (uint64_t)v.dims[0] * v.dims[1] * v.dims[2];
    sort_plan((int)vs.tiles, vs.passes, vs.digit_bits);
    vs.final_buf = vs.passes & 1;
    vs.valid = true;
    CK(s->vox_records.ensure(s->cap * sizeof(VoxRecord)));
    CK(s->vox_tile_start.ensure((vs.tiles + 1) * 4));
    CK(s->volume.ensure(vs.voxels * 4));
    CK(s->dl_dv_vol.ensure(vs.voxels * 4));
    StageScope scope(s, GPK_STAGE_VOXEL);
    CK(cudaMemsetAsync(s->head.p, 0, head_size(s->n), s->stream));
    // the slice path clears only the histogram rows its previous sort used
    CK(cudaMemsetAsync(s->sort_status.p, 0, s->sort_status.bytes, s->stream));
    if (s->n == 0) {  // every tile empty
        CK(cudaMemsetAsync(s->vox_tile_start.p, 0, (vs.tiles + 1) * 4, s->stream));
        return GPK_OK;
    }
    VoxPrepLaunch p;
    p.params = s->params.as<float>();
    p.cap = s->cap;
    p.n = (uint32_t)s->n;
    p.records = s->vox_records.as<VoxRecord>();
    p.survivor_list = s->survivors.as<uint32_t>();
    p.keys = s->keys[0].as<uint32_t>();
    p.vals = s->vals[0].as<uint32_t>();
    p.pair_cap = s->pair_cap;
    p.hist = s->hist();
    p.tile_hist0 = s->sort_status.as<unsigned>();
    p.sort_tiles_cap = s->sort_tiles_cap;
    p.passes = vs.passes;
    p.digit_bits = vs.digit_bits;
    p.tile_shift = sort_tile_shift(s->pair_cap);
    p.chunk_words = reinterpret_cast<unsigned long long*>(s->filter_flags());
    p.ctrl = s->ctrl();
    p.err = s->err();
    p.v = v;
    p.grid = (int)std::min<uint64_t>(exact_chunks(s->n), (uint64_t)s->num_sms * 4);
    launch_vox_prep(p, s->stream);
    CK(cudaGetLastError());
    TRY(launch_sorts(s, vs.passes, vs.digit_bits, nullptr, 0, p.tile_shift));
    launch_key_starts(s->keys[vs.final_buf].as<uint32_t>(), s->ctrl(), s->pair_cap, (unsigned)vs.tiles,
                      s->vox_tile_start.as<unsigned>(), s->num_sms, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

VoxEvalLaunch vox_eval_args(gpk_session* s) {
    VoxEvalLaunch e;
    e.records = s->vox_records.as<VoxRecord>();
    e.keys = s->keys[s->vox.final_buf].as<uint32_t>();
    e.vals = s->vals[s->vox.final_buf].as<uint32_t>();
    e.tile_start = s->vox_tile_start.as<unsigned>();
    e.ctrl = s->ctrl();
    e.pair_cap = s->pair_cap;
    e.volume = s->volume.as<float>();
    e.dl_dv = s->dl_dv_vol.as<float>();
    e.partials = s->vox_partials.as<float>();
    e.v = s->vox.v;
    e.dl_global = (size_t)e.v.tile[0] * e.v.tile[1] * e.v.tile[2] * 4 > 96 * 1024 ? 1 : 0;
    return e;
}

// Prepare; on pair overflow grow the pair buffers and prepare again.
int vox_prep_settled(gpk_session* s, const gpk_voxelizer_config* cfg) {
    for (int attempt = 0; attempt < 2; ++attempt) {
        TRY(run_vox_prep(s, cfg));
        TRY(sync_and_check(s, "voxelize"));
        Control c;
        CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
        if (!c.pair_overflow) return GPK_OK;
        TRY(ensure_pairs(s, (uint64_t)c.pairs + c.pairs / 4 + 1024));
    }
    return fail(GPK_ERR_STATE, "voxel pair capacity still exceeded after growth");
}

}  // namespace

extern "C" {

int gpk_abi_version(void) { return GPK_ABI_VERSION; }
const char* gpk_last_error_message(void) { return t_err.c_str(); }
int64_t gpk_last_error_index(void) { return t_err_index; }

int gpk_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(GPK_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    *count = c;
    return ok();
}

int gpk_session_create(int device, void* cuda_stream, gpk_session** out) {
    if (!out) return fail(GPK_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    auto* s = new gpk_session;
    s->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete s;
        return fail(GPK_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    if (cuda_stream) {
        s->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete s;
            return fail(GPK_ERR_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
        }
        s->own_stream = true;
    }
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (const char* f = getenv("GPK_FUSE_GATHER")) s->fuse_gather_ok = f[0] != '0';
    if (const char* f = getenv("GPK_ADAM_SPLIT")) s->adam_split = f[0] == '1';
    if (const char* f = getenv("GPK_ADAM_REST_CTAS")) s->adam_rest_ctas = atoi(f);
    if (const char* f = getenv("GPK_LAZY_ADAM")) s->lazy_on = f[0] == '1';
    if (const char* f = getenv("GPK_LOSS_IN_FWD")) s->loss_in_fwd = f[0] == '1';
    if (s->num_sms < 1) s->num_sms = 148;
    e = s->persist.ensure(kPersistBytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->persist.p, 0, kPersistBytes, s->stream);
    if (e == cudaSuccess) {
        ErrorState es;
        for (int k = 0; k < 4; ++k) es.first_index[k] = ~0ull;
        e = cudaMemcpyAsync(s->err(), &es, sizeof es, cudaMemcpyHostToDevice, s->stream);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_cfork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_cjoin, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_xfork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_xjoin, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_tgt_fork, cudaEventDisableTiming);
    for (int k = 0; k < 2; ++k) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_tgt_ready_k[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_tgt_free_k[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_rel_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_rel_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->rel_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_bjoin, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_ord, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->adam_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_rest_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_rest_join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) {
        gpk_session_destroy(s);
        return fail(GPK_ERR_CUDA, std::string("session init: ") + cudaGetErrorString(e));
    }
    if (alloc_for_n(s, 0) != GPK_OK) {
        gpk_session_destroy(s);
        return GPK_ERR_OUT_OF_MEMORY;
    }
    *out = s;
    return ok();
}

static int session_destroy(gpk_session* s);

int gpk_session_destroy(gpk_session* s) {
    if (s && s->owner) return fail(GPK_ERR_STATE, "a slice context is destroyed with its session");
    return session_destroy(s);
}

static int session_destroy(gpk_session* s) {
    if (!s) return ok();
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    for (gpk_session* c : s->ctxs) session_destroy(c);  // their borrowed planes are not freed
    s->ctxs.clear();
    for (auto& g : s->graphs) {
        cudaGraphExecDestroy(g.exec);
        for (auto& p : g.timed) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
    }
    s->graphs.clear();
    DevBuf* bufs[] = {&s->params, &s->grads, &s->adam_m, &s->adam_v, &s->records, &s->survivors,
                      &s->keys[0], &s->keys[1], &s->vals[0], &s->vals[1], &s->partials, &s->pair_recs, &s->tile_start, &s->vox_tile_start,
                      &s->sort_status, &s->head, &s->persist, &s->image,
                      &s->dl_di, &s->target_k[0], &s->target_k[1], &s->loss_g, &s->loss_partial, &s->stat_norm, &s->acc_norm, &s->acc_obs, &s->acc_world,
                      &s->stat_obs, &s->stat_world, &s->cand_list, &s->surv_params, &s->cand, &s->cand_count, &s->grp_table, &s->bucket_tab,
                      &s->dirty_idx, &s->vox_records, &s->slot_grads, &s->gmap, &s->union_words,
                      &s->union_prefix, &s->umap, &s->urows, &s->uctrl, &s->surv_bits,
                      &s->volume, &s->dl_dv_vol, &s->vox_partials};
    for (DevBuf* b : bufs) b->release();
    drain_timing(s);
    for (cudaEvent_t e : s->event_pool) cudaEventDestroy(e);
    if (s->side) {
        cudaStreamSynchronize(s->side);
        cudaStreamDestroy(s->side);
    }
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->ev_cfork) cudaEventDestroy(s->ev_cfork);
    if (s->ev_cjoin) cudaEventDestroy(s->ev_cjoin);
    if (s->ev_xfork) cudaEventDestroy(s->ev_xfork);
    if (s->ev_xjoin) cudaEventDestroy(s->ev_xjoin);
    if (s->copy) {
        cudaStreamSynchronize(s->copy);
        cudaStreamDestroy(s->copy);
    }
    if (s->ev_tgt_fork) cudaEventDestroy(s->ev_tgt_fork);
    for (int k = 0; k < 2; ++k) {
        if (s->ev_tgt_ready_k[k]) cudaEventDestroy(s->ev_tgt_ready_k[k]);
        if (s->ev_tgt_free_k[k]) cudaEventDestroy(s->ev_tgt_free_k[k]);
    }
    if (s->ev_rel_fork) cudaEventDestroy(s->ev_rel_fork);
    if (s->ev_rel_join) cudaEventDestroy(s->ev_rel_join);
    if (s->rel_stream) {
        cudaStreamSynchronize(s->rel_stream);
        cudaStreamDestroy(s->rel_stream);
    }
    if (s->ev_bjoin) cudaEventDestroy(s->ev_bjoin);
    if (s->ev_ord) cudaEventDestroy(s->ev_ord);
    if (s->ev_rest_fork) cudaEventDestroy(s->ev_rest_fork);
    if (s->ev_rest_join) cudaEventDestroy(s->ev_rest_join);
    if (s->adam_stream) {
        cudaStreamSynchronize(s->adam_stream);
        cudaStreamDestroy(s->adam_stream);
    }
    if (s->comm) gpk_comm_destroy(s);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return ok();
}

int gpk_session_set_stream(gpk_session* s, void* cuda_stream) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    if (s->own_stream) cudaStreamDestroy(s->stream);
    s->own_stream = false;
    s->stream = static_cast<cudaStream_t>(cuda_stream);
    return ok();
}

int gpk_session_get_stream(gpk_session* s, void** cuda_stream) {
    if (!s || !cuda_stream) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    *cuda_stream = s->stream;
    return ok();
}

int gpk_session_synchronize(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    if (s->owner) CK(cudaStreamSynchronize(s->owner->stream));  // batched steps run there
    TRY(sync_and_check(s, "session"));
    if (s->prep.valid) {
        Control c;
        CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
        if (c.pair_overflow) {
            char buf[160];
            snprintf(buf, sizeof buf,
                     "tile pair capacity exceeded (%u pairs > %llu); call gpk_session_reserve_pairs",
                     c.pairs, (unsigned long long)s->pair_cap);
            return fail(GPK_ERR_STATE, buf);
        }
    }
    return ok();
}

int gpk_session_reserve_pairs(gpk_session* s, uint64_t pairs) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(ensure_pairs(s, pairs));
    CK(cudaStreamSynchronize(s->stream));
    return ok();
}

int gpk_device_buffer(gpk_session* s, int which, void** ptr, uint64_t* bytes) {
    if (!s || !ptr) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    const size_t px = (size_t)s->img_w * s->img_h;
    void* p = nullptr;
    uint64_t b = 0;
    switch (which) {
        case GPK_BUF_PARAMS:  // the caller may read or write them: current, not maintained lazily
            TRY(lazy_kill(s));
            p = s->params.p;
            b = s->cap * 44;
            s->prefilter.valid = false;
            break;
        case GPK_BUF_GRADS:  // the caller may read or write the dense planes
            TRY(materialize_dense_grads(s));
            TRY(mark_grads_dense(s));
            p = s->grads.p;
            b = s->cap * 44;
            break;
        case GPK_BUF_IMAGE: p = s->image.p; b = px * 4; break;
        case GPK_BUF_DL_DI: p = s->dl_di.p; b = px * 4; break;
        case GPK_BUF_TARGET:
            TRY(target_wait(s));
            if (!s->capturing) TRY(target_release(s));  // (the caller may use it until the next upload)
            p = s->tgt().p;
            b = px * 4;
            break;
        case GPK_BUF_LOSS: p = s->loss(); b = 8; break;
        case GPK_BUF_UNION_ROWS: p = s->urows.p; b = s->urows.p ? s->cap * 44 : 0; break;
        case GPK_BUF_VOLUME: p = s->volume.p; b = s->vox.voxels * 4; break;
        case GPK_BUF_DL_DV: p = s->dl_dv_vol.p; b = s->vox.voxels * 4; break;
        default: return fail(GPK_ERR_INVALID_ARGUMENT, "unknown or unallocated buffer");
    }
    *ptr = p;
    if (bytes) *bytes = b;
    return ok();
}

// A context's stream-ordered copies are ordered on both its own stream (its
// direct calls) and its session's stream (where batched steps and their graphs
// run): the context stream first waits for the session stream, and the
// session stream afterwards waits for the copy.
static int ctx_order_in(gpk_session* s) {
    if (!s->owner || s->capturing) return GPK_OK;
    CK(cudaEventRecord(s->owner->ev_ord, s->owner->stream));
    CK(cudaStreamWaitEvent(s->stream, s->owner->ev_ord, 0));
    return GPK_OK;
}
static int ctx_order_out(gpk_session* s, cudaStream_t copied_on) {
    if (!s->owner || s->capturing) return GPK_OK;
    CK(cudaEventRecord(s->ev_ord, copied_on));
    CK(cudaStreamWaitEvent(s->owner->stream, s->ev_ord, 0));
    return GPK_OK;
}

int gpk_upload(gpk_session* s, int which, const void* host, uint64_t bytes) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    // image-shaped inputs may be staged before the first slice sized them
    DevBuf* grow = which == GPK_BUF_DL_DI ? &s->dl_di : which == GPK_BUF_TARGET ? &s->tgt()
                 : which == GPK_BUF_DL_DV ? &s->dl_dv_vol : nullptr;
    if (grow && host && bytes > grow->bytes) {
        TRY(set_device(s));
        CK(cudaStreamSynchronize(s->stream));
        CK(cudaStreamSynchronize(s->copy));
        CK(grow->ensure(bytes));
        ++s->alloc_epoch;
    }
    void* p = nullptr;
    uint64_t cap = 0;
    TRY(gpk_device_buffer(s, which, &p, &cap));
    if (grow) cap = grow->bytes;
    if (!host || bytes > cap) return fail(GPK_ERR_INVALID_ARGUMENT, "upload: size exceeds buffer");
    TRY(set_device(s));
    TRY(ctx_order_in(s));
    if (which == GPK_BUF_TARGET && !s->capturing) {
        // on the copy stream, after the last queued reader of the target
        // (ev_tgt_free): the transfer overlaps the rest of the step that read
        // it and the next step's prepare and forward, which do not read it
        CK(cudaStreamWaitEvent(s->copy, s->ev_tgt_free(), 0));
        CK(cudaMemcpyAsync(p, host, bytes, cudaMemcpyHostToDevice, s->copy));
        CK(cudaEventRecord(s->ev_tgt_ready(), s->copy));
        s->tgt_pending() = true;
        return ok();
    }
    CK(cudaMemcpyAsync(p, host, bytes, cudaMemcpyHostToDevice, s->stream));
    TRY(ctx_order_out(s, s->stream));
    return ok();
}

int gpk_download(gpk_session* s, int which, void* host, uint64_t bytes) {
    void* p = nullptr;
    uint64_t cap = 0;
    TRY(gpk_device_buffer(s, which, &p, &cap));
    if (!host || bytes > cap) return fail(GPK_ERR_INVALID_ARGUMENT, "download: size exceeds buffer");
    TRY(set_device(s));
    TRY(ctx_order_in(s));
    CK(cudaMemcpyAsync(host, p, bytes, cudaMemcpyDeviceToHost, s->stream));
    TRY(ctx_order_out(s, s->stream));
    return ok();
}

int gpk_set_target_slot(gpk_session* s, int32_t slot) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (slot != 0 && slot != 1) return fail(GPK_ERR_INVALID_ARGUMENT, "target slot must be 0 or 1");
    if (s->capturing) return fail(GPK_ERR_STATE, "target slot: select it before the capture");
    TRY(set_device(s));
    DevBuf& b = s->target_k[slot];
    const size_t px = (size_t)s->img_w * s->img_h;
    if (px && b.bytes < px * 4) {
        const void* before = b.p;
        CK(cudaStreamSynchronize(s->copy));
        CK(b.ensure(px * 4));
        if (before) ++s->alloc_epoch;  // (a first allocation: no graph holds it yet)
    }
    s->tgt_slot = slot;
    return ok();
}

int gpk_set_loss_sink(gpk_session* s, double* host) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    void* d = nullptr;
    if (host) {
        const cudaError_t e = cudaHostGetDevicePointer(&d, host, 0);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(GPK_ERR_INVALID_ARGUMENT, "loss sink: not page-locked host memory");
        }
    }
    CK(cudaStreamSynchronize(s->stream));
    if (d != (void*)s->loss_sink) ++s->alloc_epoch;  // captured graphs bake the sink
    s->loss_sink = static_cast<double*>(d);
    return ok();
}

int gpk_set_lazy_adam(gpk_session* s, int on) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (s->owner) return fail(GPK_ERR_STATE, "slice context: the mode belongs to its session");
    TRY(set_device(s));
    if (!on) TRY(lazy_kill(s));
    if ((on != 0) != s->lazy_on) ++s->alloc_epoch;  // graphs captured in the other mode
    s->lazy_on = on != 0;
    return ok();
}

int gpk_stage_timing(gpk_session* s, int enable) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    s->timing = enable != 0;
    return ok();
}

int gpk_stage_times(gpk_session* s, double* ms, uint64_t* counts, int reset) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    drain_timing(s);
    for (int k = 0; k < GPK_NUM_STAGES; ++k) {
        if (ms) ms[k] = s->stage_ms[k];
        if (counts) counts[k] = s->stage_cnt[k];
        if (reset) {
            s->stage_ms[k] = 0.0;
            s->stage_cnt[k] = 0;
        }
    }
    return ok();
}

int gpk_set_gaussians(gpk_session* s, uint64_t n, const float* records, const gpk_bounds* bbox) {
    if (!s || (n && !records) || !bbox) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (n >= (1ull << 31)) return fail(GPK_ERR_INVALID_ARGUMENT, "set size must be < 2^31");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    TRY(alloc_for_n(s, n));
    s->bbox = *bbox;
    if (n) TRY(copy_params_in(s, n, records));
    s->prep.valid = false;
    s->prefilter.valid = false;
    TRY(adam_reset(s));
    CK(cudaStreamSynchronize(s->stream));
    return ok();
}

int gpk_set_gaussians_f64(gpk_session* s, uint64_t n, const double* records,
                          const gpk_bounds* bbox) {
    std::vector<float> f(n * 11);
    for (uint64_t i = 0; i < n * 11; ++i) f[i] = (float)records[i];
    return gpk_set_gaussians(s, n, f.data(), bbox);
}

int gpk_get_bounds(gpk_session* s, gpk_bounds* out) {
    if (!s || !out) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    *out = s->bbox;
    return ok();
}

int gpk_get_gaussians(gpk_session* s, float* records) {
    if (!s || (s->n && !records)) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    TRY(lazy_sync(s));
    CK(cudaStreamSynchronize(s->stream));
    if (s->n) TRY(copy_planes_out(s, s->params.as<float>(), records));
    return ok();
}

int gpk_set_gradients(gpk_session* s, const float* grads) {
    if (!s || (s->n && !grads)) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    if (s->n) TRY(copy_records_in(s, s->n, grads, s->grads.as<float>()));
    s->grads_in_slots = false;
    s->grads_in_union = false;
    TRY(mark_grads_dense(s));
    CK(cudaStreamSynchronize(s->stream));
    return ok();
}

int gpk_get_gradients(gpk_session* s, float* grads) {
    if (!s || (s->n && !grads)) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    TRY(materialize_dense_grads(s));
    TRY(sync_and_check(s, "gradients"));
    if (s->n) TRY(copy_planes_out(s, s->grads.as<float>(), grads));
    return ok();
}

int gpk_gaussian_count(gpk_session* s, uint64_t* n) {
    if (!s || !n) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    *n = s->n;
    return ok();
}

int gpk_prepare(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                const gpk_raster_config* cfg) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(run_prepare(s, pose, psf, cfg, false));
    return ok();
}

int gpk_prepared_count(gpk_session* s, uint64_t* survivors, uint64_t* pairs) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->prep.valid) return fail(GPK_ERR_STATE, "no prepared slice");
    TRY(set_device(s));
    TRY(settle_pairs(s));
    TRY(sync_and_check(s, "prepare_gaussians"));
    Control c;
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    if (survivors) *survivors = s->n ? c.survivors : 0;
    if (pairs) *pairs = s->n ? c.pairs : 0;
    return ok();
}

int gpk_prepare_stats(gpk_session* s, uint64_t* candidates, uint64_t* survivors, uint64_t* pairs,
                      uint64_t* fp64_decided) {
    uint64_t S = 0, T = 0;
    TRY(gpk_prepared_count(s, &S, &T));
    Control c;
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    if (candidates) *candidates = s->n ? c.candidates : 0;
    if (survivors) *survivors = S;
    if (pairs) *pairs = T;
    if (fp64_decided) *fp64_decided = s->n ? c.exact_decided : 0;
    return ok();
}

int gpk_get_prepared(gpk_session* s, uint32_t* index, int32_t* bounds, double* fields) {
    uint64_t S = 0, T = 0;
    TRY(gpk_prepared_count(s, &S, &T));
    if (S == 0) return ok();
    // survivors in set order: K_decide groups in order, slots g*4096 + [0, S_g)
    const uint64_t ng = decide_group_count(s->n);
    std::vector<uint32_t> per(ng), list;
    CK(cudaMemcpy(per.data(), s->grp_surv(), ng * 4, cudaMemcpyDeviceToHost));
    list.reserve(S);
    for (uint64_t g = 0; g < ng; ++g)
        for (uint32_t j = 0; j < per[g]; ++j) list.push_back((uint32_t)(g * kDecideGroupSize + j));
    if (list.size() != S) return fail(GPK_ERR_STATE, "prepared: survivor bookkeeping mismatch");
    std::vector<SurvivorRecord> recs(s->records.bytes / sizeof(SurvivorRecord));
    CK(cudaMemcpy(recs.data(), s->records.p, recs.size() * sizeof(SurvivorRecord),
                  cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < S; ++k) {
        const SurvivorRecord& r = recs[list[k]];
        if (index) index[k] = r.gidx & 0x7fffffffu;  // bit 31: decided on the fp64 path
        if (bounds) {
            bounds[4 * k + 0] = r.lo_x;
            bounds[4 * k + 1] = r.hi_x;
            bounds[4 * k + 2] = r.lo_y;
            bounds[4 * k + 3] = r.hi_y;
        }
        if (fields) {
            double* f = fields + 6 * k;
            f[0] = r.alpha_tilde;
            f[1] = r.mu2d_x;
            f[2] = r.mu2d_y;
            f[3] = r.conic_a;
            f[4] = r.conic_b;
            f[5] = r.conic_d;
        }
    }
    return ok();
}

int gpk_get_prepared_fields(gpk_session* s, double* fields) {
    uint64_t S = 0, T = 0;
    TRY(gpk_prepared_count(s, &S, &T));
    if (S == 0 || !fields) return ok();
    const uint64_t ng = decide_group_count(s->n);
    std::vector<uint32_t> per(ng), list;
    CK(cudaMemcpy(per.data(), s->grp_surv(), ng * 4, cudaMemcpyDeviceToHost));
    list.reserve(S);
    for (uint64_t g = 0; g < ng; ++g)
        for (uint32_t j = 0; j < per[g]; ++j) list.push_back((uint32_t)(g * kDecideGroupSize + j));
    if (list.size() != S) return fail(GPK_ERR_STATE, "prepared: survivor bookkeeping mismatch");
    DevBuf slots, out;
    CK(slots.ensure(S * 4));
    CK(out.ensure(S * GPK_PREPARED_FIELDS * 8));
    CK(cudaMemcpyAsync(slots.p, list.data(), S * 4, cudaMemcpyHostToDevice, s->stream));
    launch_prepared_full(s->surv_params.as<CandParams>(), slots.as<uint32_t>(), (unsigned)S, s->prep.slice,
                         out.as<double>(), s->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(fields, out.p, S * GPK_PREPARED_FIELDS * 8, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return ok();
}

int gpk_get_tile_lists(gpk_session* s, uint32_t* offsets, uint32_t* entries) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(ensure_lists(s));
    uint64_t S = 0, T = 0;
    TRY(gpk_prepared_count(s, &S, &T));
    const int tiles = s->prep.tiles;
    std::vector<uint32_t> keys(T), vals(T);
    if (T) {
        CK(cudaMemcpy(vals.data(), s->vals[s->prep.final_buf].p, T * 4, cudaMemcpyDeviceToHost));
        if (s->prep.passes == 1) {  // gathered lists: tile starts from the published table
            std::vector<uint32_t> begin(tiles + 1);
            CK(cudaMemcpy(begin.data(), s->grp_begin(), (tiles + 1) * 4, cudaMemcpyDeviceToHost));
            for (int t = 0; t < tiles; ++t)
                for (uint32_t k = begin[t]; k < begin[t + 1] && k < T; ++k) keys[k] = (uint32_t)t;
        } else {
            CK(cudaMemcpy(keys.data(), s->keys[s->prep.final_buf].p, T * 4, cudaMemcpyDeviceToHost));
        }
    }
    std::vector<SurvivorRecord> recs;
    if (T) {
        recs.resize(s->records.bytes / sizeof(SurvivorRecord));
        CK(cudaMemcpy(recs.data(), s->records.p, recs.size() * sizeof(SurvivorRecord),
                      cudaMemcpyDeviceToHost));
    }
    if (offsets) {
        uint64_t k = 0;
        for (int t = 0; t <= tiles; ++t) {
            while (k < T && keys[k] < (uint32_t)t) ++k;
            offsets[t] = (uint32_t)k;
        }
    }
    if (entries)
        for (uint64_t k = 0; k < T; ++k) entries[k] = recs[vals[k]].gidx & 0x7fffffffu;
    return ok();
}

int gpk_rasterize(gpk_session* s, float* image_out) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(run_rasterize(s));
    if (image_out) {
        TRY(settle_pairs(s));
        TRY(sync_and_check(s, "rasterize_prepared"));
        CK(cudaMemcpy(image_out, s->image.p, (size_t)s->img_w * s->img_h * 4,
                      cudaMemcpyDeviceToHost));
    }
    return ok();
}

int gpk_backward(gpk_session* s, const float* dl_di, float* grads_out, gpk_screen_stats* stats) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->prep.valid) return fail(GPK_ERR_STATE, "backward: no prepared slice");
    TRY(set_device(s));
    const size_t px = (size_t)s->img_w * s->img_h;
    if (dl_di) CK(cudaMemcpyAsync(s->dl_di.p, dl_di, px * 4, cudaMemcpyHostToDevice, s->stream));
    const bool host = grads_out || stats;
    if (host) TRY(settle_pairs(s));
    TRY(run_backward(s, stats != nullptr));
    if (host) {
        TRY(sync_and_check(s, "backward_slice"));
        if (grads_out && s->n) TRY(copy_planes_out(s, s->grads.as<float>(), grads_out));
        if (stats && s->n) {
            std::vector<float> nrm(s->n), wld(3 * s->n);
            CK(cudaMemcpy(nrm.data(), s->stat_norm.p, s->n * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(wld.data(), s->stat_world.p, s->n * 12, cudaMemcpyDeviceToHost));
            if (stats->observed)
                CK(cudaMemcpy(stats->observed, s->stat_obs.p, s->n, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < s->n; ++i) {
                if (stats->mu2d_grad_norm) stats->mu2d_grad_norm[i] = nrm[i];
                if (stats->world_pos_grad)
                    for (int d = 0; d < 3; ++d) stats->world_pos_grad[3 * i + d] = wld[3 * i + d];
            }
        }
    }
    return ok();
}

int gpk_photometric_loss(gpk_session* s, const float* target, double lambda, double dssim_scale,
                         double* loss_out, float* dl_di_out) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (lambda < 0.0 || !std::isfinite(lambda))
        return fail(GPK_ERR_INVALID_ARGUMENT, "photometric_loss: lambda must be >= 0");
    TRY(set_device(s));
    const size_t px = (size_t)s->img_w * s->img_h;
    // host results: the render must be complete first (a slice whose tile pairs
    // overflowed is re-prepared and re-rendered before the loss reads it)
    if ((loss_out || dl_di_out) && s->prep.valid && s->prep.rasterized) TRY(settle_pairs(s));
    TRY(target_wait(s));
    if (target) CK(cudaMemcpyAsync(s->tgt().p, target, px * 4, cudaMemcpyHostToDevice, s->stream));
    TRY(run_loss(s, lambda, dssim_scale));
    if (loss_out || dl_di_out) {
        TRY(sync_and_check(s, "photometric_loss"));
        if (loss_out) CK(cudaMemcpy(loss_out, s->loss(), 8, cudaMemcpyDeviceToHost));
        if (dl_di_out) CK(cudaMemcpy(dl_di_out, s->dl_di.p, px * 4, cudaMemcpyDeviceToHost));
    }
    return ok();
}

int gpk_photometric_loss_images(gpk_session* s, int32_t width, int32_t height,
                                const float* rendered, const float* target, double lambda,
                                double dssim_scale, double* loss_out, float* dl_di_out) {
    if (!s || !rendered || !target) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (width < 1 || height < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, "photometric_loss: image shape mismatch");
    if (lambda < 0.0 || !std::isfinite(lambda))
        return fail(GPK_ERR_INVALID_ARGUMENT, "photometric_loss: lambda must be >= 0");
    TRY(set_device(s));
    TRY(ensure_image(s, width, height));
    const size_t px = (size_t)width * height;
    TRY(target_wait(s));
    CK(cudaMemcpyAsync(s->image.p, rendered, px * 4, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemcpyAsync(s->tgt().p, target, px * 4, cudaMemcpyHostToDevice, s->stream));
    // the prepared slice survives when the images have its shape (only the
    // rendered image buffer is overwritten), as the reference's loss leaves
    // the caller's prepared vector alone
    const bool keep = s->prep.valid && s->prep.slice.W == width && s->prep.slice.H == height;
    s->prep.rasterized = true;
    TRY(run_loss(s, lambda, dssim_scale));
    s->prep.rasterized = false;
    s->prep.valid = keep;
    TRY(sync_and_check(s, "photometric_loss"));
    if (loss_out) CK(cudaMemcpy(loss_out, s->loss(), 8, cudaMemcpyDeviceToHost));
    if (dl_di_out) CK(cudaMemcpy(dl_di_out, s->dl_di.p, px * 4, cudaMemcpyDeviceToHost));
    return ok();
}

int gpk_adam_step(gpk_session* s, const gpk_learning_rates* lrs, const gpk_adam_hparams* hp) {
    if (!s || !lrs) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    const double lr[4] = {lrs->position, lrs->opacity, lrs->scale, lrs->rotation};
    TRY(run_adam(s, lr, false, 1, hp));
    return ok();
}

int gpk_adam_step_scheduled(gpk_session* s, const gpk_learning_rates* lr0, int32_t total,
                            const gpk_adam_hparams* hp) {
    if (!s || !lr0) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (total < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "total iterations must be >= 1");
    TRY(set_device(s));
    const double lr[4] = {lr0->position, lr0->opacity, lr0->scale, lr0->rotation};
    TRY(run_adam(s, lr, true, total, hp));
    return ok();
}

int gpk_adam_reset(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(lazy_kill(s));  // the deferred steps' parameter updates first
    TRY(adam_reset(s));
    return ok();
}

int gpk_get_adam_state(gpk_session* s, float* m, float* v, int64_t* step) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(lazy_sync(s));
    CK(cudaStreamSynchronize(s->stream));
    if (m && s->n) TRY(copy_planes_out(s, s->adam_m.as<float>(), m));
    if (v && s->n) TRY(copy_planes_out(s, s->adam_v.as<float>(), v));
    if (step) {
        long long st = 0;
        CK(cudaMemcpy(&st, s->adam_step(), 8, cudaMemcpyDeviceToHost));
        *step = st;
    }
    return ok();
}

int gpk_set_adam_state(gpk_session* s, const float* m, const float* v, int64_t step) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(lazy_kill(s));
    CK(cudaStreamSynchronize(s->stream));
    const uint64_t n = s->n;
    if (m && n) TRY(copy_records_in(s, n, m, s->adam_m.as<float>()));
    if (v && n) TRY(copy_records_in(s, n, v, s->adam_v.as<float>()));
    long long st = step;
    CK(cudaMemcpy(s->adam_step(), &st, 8, cudaMemcpyHostToDevice));
    return ok();
}

int gpk_fwd_bwd_slice(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                      const gpk_raster_config* cfg) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(run_prepare(s, pose, psf, cfg, true));
    TRY(run_fwd_bwd_forked(s));
    return ok();
}

// Data-parallel training (defined with the NCCL code): the dense gradient
// planes are reduce-scattered, each rank updates its shard, the parameter
// shards are all-gathered; a plain all-reduce when the shards would not tile
// the planes.
static void*& session_comm(gpk_session* s);
static uint64_t dp_chunk(gpk_session* s);
static int dp_reduce_scatter(gpk_session* s);
static int dp_all_gather_params(gpk_session* s);
static int dp_all_reduce(gpk_session* s);

// One training step (optimize.hpp:385-402): prepare, rasterize, photometric
// loss, backward, (all-reduce), scheduled Adam. The gradient is kept by
// survivor slot on a single GPU (AdamLaunch) and dense under a communicator.
// With `next`, Adam is fused with the cull of the next slice (same PSF and
// raster config) and the following step on `next` skips K_filter.
static int train_body_(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                       const gpk_raster_config* cfg, double lambda, double dssim_scale,
                       const gpk_learning_rates* lr0, int32_t total, const gpk_slice_pose* next) {
    const double lr[4] = {lr0->position, lr0->opacity, lr0->scale, lr0->rotation};
    const bool dp = session_comm(s) != nullptr;
    // lazy step (LazyAdam): the single-GPU step with the default betas; the
    // pipelined form (Adam fused with the next slice's cull) does not apply
    const bool lazy = s->lazy_on && !dp && !s->owner && s->n;
    if (lazy) {
        TRY(lazy_ensure_live(s));
        next = nullptr;
        if (s->capturing) s->cap_lazy = s->cap_lazy_used = s->cap_lazy_writes = true;
    } else {
        TRY(lazy_kill(s));
    }
    if (s->n) TRY(adam_consts_ahead(s, adam_launch(s, lr, true, total, nullptr)));
    s->fuse_gather = s->fuse_gather_ok;  // the forward builds the tile lists (gather_tile)
    const int pst = run_prepare(s, pose, psf, cfg, true);
    s->fuse_gather = false;
    TRY(pst);
    s->assume_prefiltered = false;
    // the non-survivors' Adam beside the render (see gpk_session::adam_split)
    const bool split = s->adam_split && !lazy && !dp && !next && s->n && s->consts_pending;
    if (split) {
        const AdamLaunch ar = adam_launch(s, lr, true, total, nullptr);
        CK(cudaEventRecord(s->ev_rest_fork, s->stream));
        CK(cudaStreamWaitEvent(s->adam_stream, s->ev_rest_fork, 0));
        CK(cudaStreamWaitEvent(s->adam_stream, s->ev_cjoin, 0));  // the step's constants
        s->consts_pending = false;
        {
            StageScope scope(s, GPK_STAGE_ADAM_REST, s->adam_stream);
            launch_adam_rest(ar, s->surv_bits.as<unsigned>(), s->adam_rest_ctas, s->adam_stream);
            CK(cudaGetLastError());
        }
        CK(cudaEventRecord(s->ev_rest_join, s->adam_stream));
    }
    TRY(run_rasterize(s));
    TRY(run_loss(s, lambda, dssim_scale, true));
    TRY(run_backward(s, false, /*slots=*/!dp));  // dense planes for the collectives
    if (lazy) {
        // the survivors (their deferred steps first), then the step's window
        AdamLaunch a = adam_launch(s, lr, true, total, nullptr);
        a.slot_grads = s->slot_grads.as<float>();
        a.gmap = s->gmap.as<uint16_t>();
        a.surv_gidx = s->survivors.as<uint32_t>();
        a.grp_surv = s->grp_surv();
        s->gmap_dirty = false;  // k_lazy_survivors clears the survivors' map entries
        s->prefilter.valid = false;
        StageScope scope(s, GPK_STAGE_ADAM);
        TRY(adam_consts_ready(s, a));
        launch_lazy_survivors(a, (unsigned)decide_group_count(s->n), s->stream);
        CK(cudaGetLastError());
        launch_lazy_window(a, s->stream);
        CK(cudaGetLastError());
        if (!s->capturing) s->lazy_pending = true;
        return GPK_OK;
    }
    if (split) {
        CK(cudaStreamWaitEvent(s->stream, s->ev_rest_join, 0));
        AdamLaunch a = adam_launch(s, lr, true, total, nullptr);
        a.slot_grads = s->slot_grads.as<float>();
        a.gmap = s->gmap.as<uint16_t>();
        a.surv_gidx = s->survivors.as<uint32_t>();
        a.grp_surv = s->grp_surv();
        s->gmap_dirty = false;  // k_adam_final clears the survivors' map entries
        s->prefilter.valid = false;
        StageScope scope(s, GPK_STAGE_ADAM);
        launch_adam_final(a, (unsigned)decide_group_count(s->n), s->stream);
        CK(cudaGetLastError());
        return GPK_OK;
    }
    if (dp && s->n && s->cap % (uint64_t)s->comm_world == 0) {
        TRY(dp_reduce_scatter(s));
        const uint64_t chunk = dp_chunk(s), lo = (uint64_t)s->comm_rank * chunk;
        TRY(run_adam(s, lr, true, total, nullptr, lo, lo + chunk));
        return dp_all_gather_params(s);
    }
    if (dp) TRY(dp_all_reduce(s));
    if (next && !dp) return run_adam_cull(s, lr, total, next, psf, cfg);
    return run_adam(s, lr, true, total, nullptr);
}

static int train_body(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf, const gpk_raster_config* cfg,
                      double lambda, double dssim_scale, const gpk_learning_rates* lr0, int32_t total,
                      const gpk_slice_pose* next) {
    const int st = train_body_(s, pose, psf, cfg, lambda, dssim_scale, lr0, total, next);
    if (st != GPK_OK) s->consts_pending = false;  // constants of an abandoned step
    return st;
}

int gpk_train_step(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                   const gpk_raster_config* cfg, double lambda, double dssim_scale,
                   const gpk_learning_rates* lr0, int32_t total_iterations) {
    if (!s || !lr0) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "total iterations must be >= 1");
    TRY(set_device(s));
    TRY(train_body(s, pose, psf, cfg, lambda, dssim_scale, lr0, total_iterations, nullptr));
    return ok();
}

// Pipelined training step: as gpk_train_step, with Adam fused with the cull of
// `next_pose` (same PSF and raster config), so the next step on next_pose skips
// K_filter. Bitwise the same results as gpk_train_step.
int gpk_train_step_next(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, double lambda, double dssim_scale,
                        const gpk_learning_rates* lr0, int32_t total_iterations,
                        const gpk_slice_pose* next_pose) {
    if (!s || !lr0 || !next_pose) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "total iterations must be >= 1");
    TRY(set_device(s));
    TRY(train_body(s, pose, psf, cfg, lambda, dssim_scale, lr0, total_iterations, next_pose));
    return ok();
}

// ---- slice contexts and batched steps -----------------
// A batched step renders B slices of the resident set concurrently — slice k on
// context k (its own stream and per-slice buffers; context 0 is the session
// itself) — and sums their gradients per primitive in slice order: inside the
// one Adam of the training step (k_adam_batch reads every slice's slot map), or
// into the dense planes for the fwd+bwd unit. Launch-latency-bound slice
// kernels (a 512^2 slice is 1024 tiles, ~7 CTAs per SM) of different slices
// then overlap on the GPU instead of running one after another.

static int ctx_sync(gpk_session* s, gpk_session* c) {
    if (c->params.p != s->params.p || c->adam_m.p != s->adam_m.p) {
        c->params.borrow(s->params);
        c->grads.borrow(s->grads);
        c->adam_m.borrow(s->adam_m);
        c->adam_v.borrow(s->adam_v);
        ++c->alloc_epoch;
    }
    c->bbox = s->bbox;
    if (c->n != s->n) {
        TRY(clear_gmap(c));  // the old slots' map entries (before the set size changes)
        c->prep.valid = false;
        c->n = s->n;
        ++c->alloc_epoch;
    }
    if (c->cap != s->cap) TRY(alloc_slice_bufs(c, s->cap));
    return GPK_OK;
}

static int ctx_get(gpk_session* s, int k, gpk_session** out) {
    if (s->owner) return fail(GPK_ERR_STATE, "slice contexts belong to a session, not to a context");
    if (k < 0 || k >= kMaxBatch) return fail(GPK_ERR_INVALID_ARGUMENT, "slice context index out of range [0, 8)");
    if (k == 0) {
        *out = s;
        return GPK_OK;
    }
    while ((int)s->ctxs.size() < k) {
        if (s->capturing) return fail(GPK_ERR_STATE, "slice contexts must exist before capture");
        gpk_session* c = nullptr;
        TRY(gpk_session_create(s->device, nullptr, &c));
        c->owner = s;
        s->ctxs.push_back(c);
    }
    gpk_session* c = s->ctxs[k - 1];
    if (s->capturing && (c->params.p != s->params.p || c->n != s->n || c->cap != s->cap))
        return fail(GPK_ERR_STATE, "slice context out of date during capture");
    TRY(ctx_sync(s, c));
    *out = c;
    return GPK_OK;
}

static uint64_t epoch_total(gpk_session* s) {
    uint64_t e = s->alloc_epoch;
    for (gpk_session* c : s->ctxs) e += c->alloc_epoch;
    return e;
}

static int batch_check(gpk_session* s, int B, const gpk_slice_pose* poses) {
    if (!s || !poses) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (s->owner) return fail(GPK_ERR_STATE, "batched steps run on the session, not on a context");
    if (B < 1 || B > kMaxBatch) return fail(GPK_ERR_INVALID_ARGUMENT, "batch of 1..8 slices");
    if (s->accum_on && B > 1)
        return fail(GPK_ERR_STATE, "densify accumulation is per slice: batched steps need it disabled");
    return GPK_OK;
}

static int presize_step(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, bool loss, double lambda);

// The batch's K_filter work in one pass over the parameters (k_filter_multi),
// on the session stream before the fork: every slice's candidates, control
// head and sort rows. Buffers are sized first (outside capture).
static int batch_filter(gpk_session* s, gpk_session* const* cx, int B, const gpk_slice_pose* poses,
                        const gpk_psf* psf, const gpk_raster_config* cfg, bool loss, double lambda) {
    if (!s->capturing)  // the contexts' own queued work (direct calls) precedes the batch
        for (int k = 1; k < B; ++k) {
            CK(cudaEventRecord(cx[k]->ev_bjoin, cx[k]->stream));
            CK(cudaStreamWaitEvent(s->stream, cx[k]->ev_bjoin, 0));
        }
    PrepLaunch pl[kMaxBatch];
    for (int k = 0; k < B; ++k) {
        gpk_session* c = cx[k];
        TRY(presize_step(c, &poses[k], psf, cfg, loss, lambda));
        SliceArgs a;
        TRY(make_slice(c, &poses[k], psf, cfg, a));
        int passes = 0, bits = 0;
        sort_plan(a.tiles_x * a.tiles_y, passes, bits);
        if (a.tiles_x * a.tiles_y > (1 << (kMaxDigitBits * kMaxSortPasses)))
            return fail(GPK_ERR_INVALID_ARGUMENT, "SlicePose: more than 2^20 tiles unsupported");
        pl[k] = prep_launch(c, a, passes, bits, false);
        pl[k].head = c->head.as<unsigned>();
        pl[k].head_words = (unsigned)(head_size(c->n) / 4);
    }
    if (s->n == 0) return GPK_OK;
    StageScope scope(s, GPK_STAGE_PREPARE);
    launch_prep_multi(pl, B, s->num_sms, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

// Fork the contexts of slices 1..B-1 off the session stream.
static int batch_fork(gpk_session* s, gpk_session* const* cx, int B) {
    CK(cudaEventRecord(s->ev_fork, s->stream));
    for (int k = 1; k < B; ++k) {
        CK(cudaStreamWaitEvent(cx[k]->stream, s->ev_fork, 0));
        cx[k]->capturing = s->capturing;
    }
    return GPK_OK;
}

static int batch_join(gpk_session* s, gpk_session* const* cx, int B) {
    for (int k = 1; k < B; ++k) {
        CK(cudaEventRecord(cx[k]->ev_bjoin, cx[k]->stream));
        CK(cudaStreamWaitEvent(s->stream, cx[k]->ev_bjoin, 0));
        cx[k]->capturing = false;
    }
    return GPK_OK;
}

// The B slices' gradients summed into the dense planes in slice order
// (k_sum_slots: every entry written, every map read cleared).
static AdamLaunch batch_sources(gpk_session* s, gpk_session* const* cx, int B) {
    AdamLaunch a{};
    a.grads = s->grads.as<float>();
    a.cap = s->cap;
    a.n = (uint32_t)s->n;
    a.slot_grads = cx[0]->slot_grads.as<float>();
    a.gmap = cx[0]->gmap.as<uint16_t>();
    a.ctrl = cx[0]->ctrl();
    a.nsrc = B - 1;
    for (int k = 1; k < B; ++k) {
        a.src_slot[k - 1] = cx[k]->slot_grads.as<float>();
        a.src_gmap[k - 1] = cx[k]->gmap.as<uint16_t>();
        a.src_ctrl[k - 1] = cx[k]->ctrl();
    }
    return a;
}

static int batch_dense_sum(gpk_session* s, gpk_session* const* cx, int B) {
    if (s->n) {
        launch_sum_slots(batch_sources(s, cx, B), s->stream);
        CK(cudaGetLastError());
    }
    for (int k = 0; k < B; ++k) {
        cx[k]->gmap_dirty = false;
        cx[k]->grads_in_slots = false;
    }
    s->grads_in_slots = false;
    s->grads_in_union = false;
    return mark_grads_dense(s);
}

// U1 x B: per slice prepare, then its forward (context side stream) beside its
// backward of the slice's GPK_BUF_DL_DI (slot gradients); the dense gradient
// is the sum over the slices.
static int fwd_bwd_batch_body(gpk_session* s, int B, const gpk_slice_pose* poses, const gpk_psf* psf,
                              const gpk_raster_config* cfg) {
    TRY(lazy_kill(s));  // k_filter_multi reads current parameters
    gpk_session* cx[kMaxBatch];
    for (int k = 0; k < B; ++k) TRY(ctx_get(s, k, &cx[k]));
    s->ctx_used = B - 1;
    TRY(batch_filter(s, cx, B, poses, psf, cfg, false, 0.0));
    TRY(batch_fork(s, cx, B));
    for (int k = 0; k < B; ++k) {
        TRY(run_prepare(cx[k], &poses[k], psf, cfg, false, /*filtered=*/true));
        TRY(run_fwd_bwd_forked(cx[k], /*slots=*/true));
    }
    TRY(batch_join(s, cx, B));
    return batch_dense_sum(s, cx, B);
}

// U2 x B: every slice prepared, rendered, its loss (its context's target) and
// backward taken; one Adam over the summed gradient (k_adam_batch).
static int train_batch_body(gpk_session* s, int B, const gpk_slice_pose* poses, const gpk_psf* psf,
                            const gpk_raster_config* cfg, double lambda, double dssim_scale,
                            const gpk_learning_rates* lr0, int32_t total) {
    const double lr[4] = {lr0->position, lr0->opacity, lr0->scale, lr0->rotation};
    TRY(lazy_kill(s));  // eager: k_filter_multi + the dense Adam
    gpk_session* cx[kMaxBatch];
    for (int k = 0; k < B; ++k) TRY(ctx_get(s, k, &cx[k]));
    s->ctx_used = B - 1;
    if (s->n) TRY(adam_consts_ahead(s, adam_launch(s, lr, true, total, nullptr)));
    TRY(batch_filter(s, cx, B, poses, psf, cfg, true, lambda));
    TRY(batch_fork(s, cx, B));
    for (int k = 0; k < B; ++k) {
        gpk_session* c = cx[k];
        c->fuse_gather = s->fuse_gather_ok;
        const int pst = run_prepare(c, &poses[k], psf, cfg, false, /*filtered=*/true);
        c->fuse_gather = false;
        TRY(pst);
        TRY(run_rasterize(c));
        TRY(run_loss(c, lambda, dssim_scale, true));
        TRY(run_backward(c, false, /*slots=*/true));
    }
    TRY(batch_join(s, cx, B));
    // the summed gradient into the dense planes, then the dense Adam (an
    // overflowed slice anywhere skips the update, as k_adam checks every
    // slice's control head)
    TRY(batch_dense_sum(s, cx, B));
    if (s->n == 0) return run_adam(s, lr, true, total, nullptr);
    AdamLaunch a = adam_launch(s, lr, true, total, nullptr);
    const AdamLaunch src = batch_sources(s, cx, B);
    a.ctrl = src.ctrl;
    a.nsrc = src.nsrc;
    for (int k = 0; k + 1 < B; ++k) a.src_ctrl[k] = src.src_ctrl[k];
    s->prefilter.valid = false;
    StageScope scope(s, GPK_STAGE_ADAM);
    TRY(adam_consts_ready(s, a));
    launch_adam(a, s->stream);
    CK(cudaGetLastError());
    return GPK_OK;
}

// ---- data-parallel step with the union-compacted exchange (dp.cu) -----------------
static int dp_union_allreduce(gpk_session* s);

// Buffers of the union exchange (sized by the plane stride; outside capture).
static int dp_union_alloc(gpk_session* s) {
    const void* before[3] = {s->union_words.p, s->umap.p, s->urows.p};
    const uint64_t fb = filter_blocks(s->cap);
    CK(s->union_words.ensure(fb * kFilterItems * 4));
    CK(s->union_prefix.ensure((fb + 2 * (fb / 1024 + 1)) * 4));  // chunk prefixes, block totals, block offsets
    CK(s->umap.ensure(s->cap * 4));
    CK(s->urows.ensure(s->cap * 44));
    const void* uc = s->uctrl.p;
    CK(s->uctrl.ensure(16));  // M, overflow, the scan's ticket
    if (uc != s->uctrl.p) CK(cudaMemsetAsync(s->uctrl.p, 0, 16, s->stream));
    if (before[0] != s->union_words.p || before[1] != s->umap.p || before[2] != s->urows.p) {
        if (s->capturing) return fail(GPK_ERR_STATE, "union buffers must be sized before capture");
        ++s->alloc_epoch;
    }
    if (s->ucap == 0 || s->ucap > s->cap) s->ucap = std::min<uint64_t>(s->cap, std::max<uint64_t>(1u << 16, s->n / 8));
    return GPK_OK;
}

// One data-parallel training step, rank `rank` of `world`, rendering
// poses[rank] (optimize.hpp:385-402 per rank). phases: GPK_DP_RENDER (union,
// prepare, render, loss, backward into the union rows), GPK_DP_EXCHANGE (the
// grouped all-reduce of the rows), GPK_DP_UPDATE (Adam on every Gaussian from
// its summed row).
static int train_dp_body(gpk_session* s, int world, int rank, const gpk_slice_pose* poses, const gpk_psf* psf,
                         const gpk_raster_config* cfg, double lambda, double dssim_scale,
                         const gpk_learning_rates* lr0, int32_t total, int phases) {
    const double lr[4] = {lr0->position, lr0->opacity, lr0->scale, lr0->rotation};
    TRY(lazy_kill(s));  // eager: every rank's Adam over all N
    if (phases & GPK_DP_RENDER) {
        TRY(dp_union_alloc(s));
        if (s->n) TRY(adam_consts_ahead(s, adam_launch(s, lr, true, total, nullptr)));
        TRY(presize_step(s, &poses[rank], psf, cfg, true, lambda));
        if (s->n) {
            PrepLaunch pl[kMaxBatch];
            for (int k = 0; k < world; ++k) {
                SliceArgs a;
                TRY(make_slice(s, &poses[k], psf, cfg, a));
                int passes = 0, bits = 0;
                sort_plan(a.tiles_x * a.tiles_y, passes, bits);
                pl[k] = prep_launch(s, a, passes, bits, false);
            }
            pl[rank].head = s->head.as<unsigned>();
            pl[rank].head_words = (unsigned)(head_size(s->n) / 4);
            {
                StageScope scope(s, GPK_STAGE_PREPARE);
                launch_prep_multi(pl, world, s->num_sms, s->stream, rank, s->union_words.as<unsigned>());
                CK(cudaGetLastError());
                launch_union_scan(s->union_words.as<unsigned>(), (unsigned)filter_blocks(s->n),
                                  s->union_prefix.as<unsigned>(), s->uctrl.as<unsigned>(), s->ucap, s->stream);
                CK(cudaGetLastError());
                launch_union_map(s->union_words.as<unsigned>(), s->union_prefix.as<unsigned>(), (uint32_t)s->n,
                                 s->umap.as<uint32_t>(), s->urows.as<float>(), s->cap, s->ucap, s->stream);
                CK(cudaGetLastError());
            }
            if (!s->capturing) {
                // direct call: the union size decides the exchange count; every
                // rank computes the same union, so every rank grows alike
                unsigned u[2];
                CK(cudaMemcpyAsync(u, s->uctrl.p, 8, cudaMemcpyDeviceToHost, s->stream));
                CK(cudaStreamSynchronize(s->stream));
                if (u[1]) {
                    s->ucap = std::min<uint64_t>(s->cap, (uint64_t)u[0] + u[0] / 4 + 1024);
                    CK(cudaMemsetAsync(s->uctrl.as<unsigned>() + 1, 0, 4, s->stream));
                    // (k_union_map cleared the old capacity's rows only)
                    for (int k = 0; k < 11; ++k)
                        CK(cudaMemsetAsync(s->urows.as<float>() + (size_t)k * s->cap, 0, s->ucap * 4, s->stream));
                } else if (2 * (uint64_t)u[0] + 2048 < s->ucap) {
                    // far below the capacity: shrink it (the all-reduce count and
                    // the rows' clearing scale with it; graphs are recaptured)
                    s->ucap = std::min<uint64_t>(s->cap, (uint64_t)u[0] + u[0] / 4 + 1024);
                    ++s->alloc_epoch;
                }
            }
        }
        s->fuse_gather = s->fuse_gather_ok;
        const int pst = run_prepare(s, &poses[rank], psf, cfg, false, /*filtered=*/s->n != 0);
        s->fuse_gather = false;
        TRY(pst);
        TRY(run_rasterize(s));
        TRY(run_loss(s, lambda, dssim_scale, true));
        TRY(run_backward(s, false, /*slots=*/true, /*urows=*/true));
    }
    if (phases & GPK_DP_EXCHANGE) TRY(dp_union_allreduce(s));
    if (phases & GPK_DP_UPDATE) {
        if (!s->urows.p) return fail(GPK_ERR_STATE, "data-parallel update before its render phase");
        if (s->n == 0) return run_adam(s, lr, true, total, nullptr);
        AdamLaunch a = adam_launch(s, lr, true, total, nullptr);
        a.slot_grads = s->urows.as<float>();
        a.umap = s->umap.as<uint32_t>();
        a.uctrl = s->uctrl.as<unsigned>();
        s->prefilter.valid = false;
        StageScope scope(s, GPK_STAGE_ADAM);
        TRY(adam_consts_ready(s, a));
        launch_adam(a, s->stream);
        CK(cudaGetLastError());
        s->grads_in_union = true;
    }
    return GPK_OK;
}

// ---- CUDA graphs -------------------------------------------------------------
static int capture_graph(gpk_session* s, int32_t* graph_id, int (*body)(gpk_session*, const void*),
                         const void* arg) {
    if (!s || !graph_id) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    const gpk_session::CaptureMeta meta = s->capture_meta;  // set by the caller for this capture
    s->capture_meta = gpk_session::CaptureMeta{};
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    drain_timing(s);
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    s->capturing = true;
    s->ctx_used = 0;
    s->cap_lazy = s->cap_lazy_used = s->cap_lazy_writes = false;
    int st = body(s, arg);
    // join the target-release branches (target_release) at the end of the graph
    for (int k = -1; k < (int)s->ctxs.size(); ++k) {
        gpk_session* c = k < 0 ? s : s->ctxs[k];
        if (!c->rel_join_pending) continue;
        c->rel_join_pending = false;
        if (st == GPK_OK && cudaStreamWaitEvent(s->stream, c->ev_rel_join, 0) != cudaSuccess)
            st = fail(GPK_ERR_CUDA, "graph capture: target release join");
    }
    s->capturing = false;
    const bool lazy = s->cap_lazy_used, lazy_writes = s->cap_lazy_writes;
    s->cap_lazy = s->cap_lazy_used = s->cap_lazy_writes = false;
    for (gpk_session* c : s->ctxs) c->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    // stage events recorded during capture became event-record nodes of the graph
    std::vector<gpk_session::Pending> timed;
    timed.swap(s->pending);
    if (st != GPK_OK || e != cudaSuccess) {
        for (auto& p : timed) {
            s->event_pool.push_back(p.a);
            s->event_pool.push_back(p.b);
        }
    }
    if (st != GPK_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    if (e != cudaSuccess) return fail(GPK_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return fail(GPK_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
    gpk_session::Graph gr;
    gr.exec = ex;
    gr.prep = s->prep;
    gr.grads_in_slots = s->grads_in_slots;
    gr.grads_in_union = s->grads_in_union;
    gr.gmap_dirty = s->gmap_dirty;
    gr.alloc_epoch = epoch_total(s);
    for (int k = 0; k < s->ctx_used; ++k) {
        gpk_session* c = s->ctxs[k];
        gr.ctx_state.push_back({c, c->prep, c->grads_in_slots, c->gmap_dirty});
    }
    gr.timed = std::move(timed);
    gr.needs_prefilter = meta.needs_prefilter;
    gr.sets_prefilter = meta.sets_prefilter;
    gr.writes_params = meta.writes_params;
    gr.lazy = lazy;
    gr.lazy_writes = lazy_writes;
    gr.next_pose = meta.next_pose;
    s->graphs.push_back(std::move(gr));
    *graph_id = (int32_t)s->graphs.size() - 1;
    return ok();
}

struct FwdBwdArgs {
    const gpk_slice_pose* pose;
    const gpk_psf* psf;
    const gpk_raster_config* cfg;
};

struct TrainArgs {
    const gpk_slice_pose* pose;
    const gpk_psf* psf;
    const gpk_raster_config* cfg;
    double lambda, dssim;
    const gpk_learning_rates* lr0;
    int total;
};

// Size every buffer the captured step touches (allocation is illegal under capture).
static int presize_step(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, bool loss, double lambda) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    SliceArgs a;
    TRY(make_slice(s, pose, psf, cfg, a));
    TRY(ensure_image(s, a.W, a.H));
    if (!s->keys[0].p) TRY(ensure_pairs(s, std::max<uint64_t>(1ull << 20, 8 * s->n)));
    TRY(ensure_tile_start(s, (uint64_t)a.tiles_x * a.tiles_y));
    if (loss) {
        const size_t px = (size_t)a.W * a.H;
        const void* before[2] = {s->loss_g.p, s->loss_partial.p};
        if (lambda != 0.0) CK(s->loss_g.ensure(px * 12));
        CK(s->loss_partial.ensure((size_t)loss_partial_blocks(a.W, a.H, lambda) * 16));
        if (before[0] != s->loss_g.p || before[1] != s->loss_partial.p) ++s->alloc_epoch;
    }
    return GPK_OK;
}

int gpk_graph_capture_fwd_bwd(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                              const gpk_raster_config* cfg, int32_t* graph_id) {
    TRY(presize_step(s, pose, psf, cfg, false, 0.0));
    const FwdBwdArgs args{pose, psf, cfg};
    return capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const FwdBwdArgs* a = static_cast<const FwdBwdArgs*>(p);
        TRY(run_prepare(ss, a->pose, a->psf, a->cfg, true));
        TRY(run_fwd_bwd_forked(ss));
        return GPK_OK;
    }, &args);
}

int gpk_graph_capture_train(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                            const gpk_raster_config* cfg, double lambda, double dssim_scale,
                            const gpk_learning_rates* lr0, int32_t total_iterations,
                            int32_t* graph_id) {
    if (!lr0 || total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "bad learning rates");
    TRY(presize_step(s, pose, psf, cfg, true, lambda));
    const TrainArgs args{pose, psf, cfg, lambda, dssim_scale, lr0, total_iterations};
    s->capture_meta.writes_params = true;
    return capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const TrainArgs* a = static_cast<const TrainArgs*>(p);
        return train_body(ss, a->pose, a->psf, a->cfg, a->lambda, a->dssim, a->lr0, a->total, nullptr);
    }, &args);
}

struct TrainNextArgs {
    const gpk_slice_pose* pose;
    const gpk_psf* psf;
    const gpk_raster_config* cfg;
    double lambda, dssim;
    const gpk_learning_rates* lr0;
    int total;
    const gpk_slice_pose* next;
};

int gpk_graph_capture_train_next(gpk_session* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                                 const gpk_raster_config* cfg, double lambda, double dssim_scale,
                                 const gpk_learning_rates* lr0, int32_t total_iterations,
                                 const gpk_slice_pose* next_pose, int32_t* graph_id) {
    if (!lr0 || !next_pose || total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "bad arguments");
    // data parallel: the shard-wise Adam has no fused cull; lazy steps do not
    // fuse it either (their Adam touches the survivors and a window only)
    if (session_comm(s) || (s && s->lazy_on))
        return gpk_graph_capture_train(s, pose, psf, cfg, lambda, dssim_scale, lr0, total_iterations, graph_id);
    TRY(presize_step(s, pose, psf, cfg, true, lambda));
    const TrainNextArgs args{pose, psf, cfg, lambda, dssim_scale, lr0, total_iterations, next_pose};
    s->capture_meta.needs_prefilter = true;
    s->capture_meta.sets_prefilter = true;
    s->capture_meta.writes_params = true;
    s->capture_meta.next_pose = *next_pose;
    const gpk_session::Prefilter saved = s->prefilter;
    s->assume_prefiltered = true;
    const int st = capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const TrainNextArgs* a = static_cast<const TrainNextArgs*>(p);
        return train_body(ss, a->pose, a->psf, a->cfg, a->lambda, a->dssim, a->lr0, a->total, a->next);
    }, &args);
    s->assume_prefiltered = false;
    s->prefilter = saved;  // capture records work, it does not run it
    return st;
}

// ---- batched steps: C-ABI ---------------------------------------------------------
struct BatchArgs {
    int B;
    const gpk_slice_pose* poses;
    const gpk_psf* psf;
    const gpk_raster_config* cfg;
    double lambda, dssim;
    const gpk_learning_rates* lr0;
    int total;
};

static int presize_batch(gpk_session* s, const BatchArgs& b, bool loss) {
    for (int k = 0; k < b.B; ++k) {
        gpk_session* c = nullptr;
        TRY(ctx_get(s, k, &c));
        TRY(presize_step(c, &b.poses[k], b.psf, b.cfg, loss, b.lambda));
    }
    return GPK_OK;
}

int gpk_slice_context(gpk_session* s, int32_t k, gpk_session** ctx) {
    if (!s || !ctx) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    TRY(ctx_get(s, k, ctx));
    return ok();
}

int gpk_fwd_bwd_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses, const gpk_psf* psf,
                      const gpk_raster_config* cfg) {
    TRY(batch_check(s, nslices, poses));
    TRY(set_device(s));
    TRY(fwd_bwd_batch_body(s, nslices, poses, psf, cfg));
    return ok();
}

int gpk_train_step_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses, const gpk_psf* psf,
                         const gpk_raster_config* cfg, double lambda, double dssim_scale,
                         const gpk_learning_rates* lr0, int32_t total_iterations) {
    TRY(batch_check(s, nslices, poses));
    if (!lr0 || total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "bad learning rates");
    if (session_comm(s)) return fail(GPK_ERR_STATE, "batched step under a communicator: not supported");
    TRY(set_device(s));
    const int st = train_batch_body(s, nslices, poses, psf, cfg, lambda, dssim_scale, lr0, total_iterations);
    if (st != GPK_OK) s->consts_pending = false;
    TRY(st);
    return ok();
}

int gpk_graph_capture_fwd_bwd_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses,
                                    const gpk_psf* psf, const gpk_raster_config* cfg, int32_t* graph_id) {
    TRY(batch_check(s, nslices, poses));
    TRY(set_device(s));
    const BatchArgs args{nslices, poses, psf, cfg, 0.0, 0.0, nullptr, 1};
    TRY(presize_batch(s, args, false));
    return capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const BatchArgs* a = static_cast<const BatchArgs*>(p);
        return fwd_bwd_batch_body(ss, a->B, a->poses, a->psf, a->cfg);
    }, &args);
}

int gpk_graph_capture_train_batch(gpk_session* s, int32_t nslices, const gpk_slice_pose* poses,
                                  const gpk_psf* psf, const gpk_raster_config* cfg, double lambda,
                                  double dssim_scale, const gpk_learning_rates* lr0, int32_t total_iterations,
                                  int32_t* graph_id) {
    TRY(batch_check(s, nslices, poses));
    if (!lr0 || total_iterations < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "bad learning rates");
    if (session_comm(s)) return fail(GPK_ERR_STATE, "batched step under a communicator: not supported");
    TRY(set_device(s));
    const BatchArgs args{nslices, poses, psf, cfg, lambda, dssim_scale, lr0, total_iterations};
    TRY(presize_batch(s, args, true));
    s->capture_meta.writes_params = true;
    return capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const BatchArgs* a = static_cast<const BatchArgs*>(p);
        const int st = train_batch_body(ss, a->B, a->poses, a->psf, a->cfg, a->lambda, a->dssim, a->lr0, a->total);
        if (st != GPK_OK) ss->consts_pending = false;
        return st;
    }, &args);
}

static int dp_check(gpk_session* s, int world, int rank, const gpk_slice_pose* poses, const gpk_learning_rates* lr0,
                    int total);

struct DpArgs {
    int world, rank;
    const gpk_slice_pose* poses;
    const gpk_psf* psf;
    const gpk_raster_config* cfg;
    double lambda, dssim;
    const gpk_learning_rates* lr0;
    int total;
};

int gpk_graph_capture_train_dp(gpk_session* s, int32_t world, int32_t rank, const gpk_slice_pose* poses,
                               const gpk_psf* psf, const gpk_raster_config* cfg, double lambda, double dssim_scale,
                               const gpk_learning_rates* lr0, int32_t total_iterations, int32_t* graph_id) {
    TRY(dp_check(s, world, rank, poses, lr0, total_iterations));
    if (!s->comm) return fail(GPK_ERR_STATE, "exchange: communicator not initialized");
    TRY(set_device(s));
    TRY(dp_union_alloc(s));
    TRY(presize_step(s, &poses[rank], psf, cfg, true, lambda));
    const DpArgs args{world, rank, poses, psf, cfg, lambda, dssim_scale, lr0, total_iterations};
    s->capture_meta.writes_params = true;
    return capture_graph(s, graph_id, [](gpk_session* ss, const void* p) -> int {
        const DpArgs* a = static_cast<const DpArgs*>(p);
        const int st = train_dp_body(ss, a->world, a->rank, a->poses, a->psf, a->cfg, a->lambda, a->dssim, a->lr0,
                                     a->total, GPK_DP_RENDER | GPK_DP_EXCHANGE | GPK_DP_UPDATE);
        if (st != GPK_OK) ss->consts_pending = false;
        return st;
    }, &args);
}

int gpk_graph_launch(gpk_session* s, int32_t graph_id) {
    if (!s || graph_id < 0 || graph_id >= (int32_t)s->graphs.size())
        return fail(GPK_ERR_INVALID_ARGUMENT, "unknown graph id");
    TRY(set_device(s));
    gpk_session::Graph& g = s->graphs[graph_id];
    if (g.alloc_epoch != epoch_total(s))
        return fail(GPK_ERR_STATE, "graph invalidated: session buffers were reallocated since capture; recapture");
    // lazy graphs need t_done maintained; any other graph reads or writes
    // current parameters
    TRY(g.lazy ? lazy_ensure_live(s) : lazy_kill(s));
    if (g.needs_prefilter && !prefilter_matches(s, &g.prep.pose, &g.prep.psf, &g.prep.cfg)) {
        // the graph starts at K_decide: cull its slice first (stand-alone K_filter,
        // which also clears the gradient planes)
        SliceArgs a;
        TRY(make_slice(s, &g.prep.pose, &g.prep.psf, &g.prep.cfg, a));
        if (s->n) {
            launch_prep(prep_launch(s, a, g.prep.passes, g.prep.digit_bits, true), s->num_sms, s->stream);
            CK(cudaGetLastError());
        }
    }
    CK(cudaGraphLaunch(g.exec, s->stream));
    if (g.lazy_writes) s->lazy_pending = true;
    if (g.sets_prefilter)
        set_prefilter(s, &g.next_pose, &g.prep.psf, &g.prep.cfg);
    else if (g.writes_params || g.needs_prefilter)
        s->prefilter.valid = false;
    s->prep = g.prep;
    s->grads_in_slots = g.grads_in_slots;
    s->grads_in_union = g.grads_in_union;
    s->gmap_dirty = g.gmap_dirty;
    for (const auto& cs : g.ctx_state) {
        cs.ctx->prep = cs.prep;
        cs.ctx->grads_in_slots = cs.grads_in_slots;
        cs.ctx->gmap_dirty = cs.gmap_dirty;
    }
    if (s->timing && !g.timed.empty()) {
        // graph captured with stage timing: its event nodes bracket each stage
        // on the device, back to back (no host submission gaps)
        CK(cudaStreamSynchronize(s->stream));
        for (auto& p : g.timed) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
                s->stage_ms[p.stage] += ms;
                s->stage_cnt[p.stage] += 1;
            }
        }
    }
    return ok();
}

int gpk_graph_destroy_all(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    for (auto& g : s->graphs) {
        cudaGraphExecDestroy(g.exec);
        for (auto& p : g.timed) {
            s->event_pool.push_back(p.a);
            s->event_pool.push_back(p.b);
        }
    }
    s->graphs.clear();
    return ok();
}

// ---- multi-GPU (NCCL loaded lazily so the library has no hard dependency) ----
struct NcclId {
    char internal[128];  // ncclUniqueId, passed by value
};
struct NcclApi {
    void* lib = nullptr;
    int (*get_unique_id)(void*) = nullptr;
    int (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
    int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*reduce_scatter)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    int (*comm_destroy)(void*) = nullptr;
    const char* (*get_error_string)(int) = nullptr;
};

static NcclApi* nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
        }
        if (api.lib) {
            api.get_unique_id = (int (*)(void*))dlsym(api.lib, "ncclGetUniqueId");
            api.comm_init_rank = (int (*)(void**, int, NcclId, int))dlsym(api.lib, "ncclCommInitRank");
            api.all_reduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
                api.lib, "ncclAllReduce");
            api.comm_destroy = (int (*)(void*))dlsym(api.lib, "ncclCommDestroy");
            api.reduce_scatter = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
                api.lib, "ncclReduceScatter");
            api.all_gather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(
                api.lib, "ncclAllGather");
            api.group_start = (int (*)())dlsym(api.lib, "ncclGroupStart");
            api.group_end = (int (*)())dlsym(api.lib, "ncclGroupEnd");
            api.get_error_string = (const char* (*)(int))dlsym(api.lib, "ncclGetErrorString");
        }
    }
    return (api.get_unique_id && api.comm_init_rank && api.all_reduce) ? &api : nullptr;
}


static void*& session_comm(gpk_session* s) { return s->comm; }

int gpk_nccl_get_unique_id(void* id_out128) {
    NcclApi* api = nccl();
    if (!api) return fail(GPK_ERR_NCCL, "libnccl.so.2 not found");
    const int r = api->get_unique_id(id_out128);
    if (r != 0) return fail(GPK_ERR_NCCL, "ncclGetUniqueId failed");
    return ok();
}

int gpk_comm_init(gpk_session* s, int nranks, int rank, const void* id128) {
    if (!s || !id128) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    NcclApi* api = nccl();
    if (!api) return fail(GPK_ERR_NCCL, "libnccl.so.2 not found");
    TRY(set_device(s));
    NcclId id;
    memcpy(id.internal, id128, 128);
    void* comm = nullptr;
    const int r = api->comm_init_rank(&comm, nranks, id, rank);
    if (r != 0)
        return fail(GPK_ERR_NCCL, std::string("ncclCommInitRank: ") +
                                      (api->get_error_string ? api->get_error_string(r) : "error"));
    session_comm(s) = comm;
    s->comm_rank = rank;
    s->comm_world = nranks;
    return ok();
}

int gpk_comm_destroy(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    NcclApi* api = nccl();
    void*& comm = session_comm(s);
    if (api && comm && api->comm_destroy) api->comm_destroy(comm);
    comm = nullptr;
    s->comm_rank = 0;
    s->comm_world = 1;
    return ok();
}

// Data-parallel training step, ZeRO-style: the summed
// gradient is only needed by the Adam that updates it, so each rank
// reduce-scatters the dense planes (rank r receives the sum over primitives
// [r*chunk, (r+1)*chunk) of every plane), runs Adam on that shard and the
// parameter shards are all-gathered. Same traffic as one all-reduce, Adam work
// / world, and every replica ends bitwise equal (one owner per primitive).
static uint64_t dp_chunk(gpk_session* s) { return s->cap / (uint64_t)s->comm_world; }

static int dp_all_reduce(gpk_session* s) {
    NcclApi* api = nccl();
    if (!api) return fail(GPK_ERR_NCCL, "NCCL not available");
    if (api->all_reduce(s->grads.p, s->grads.p, s->cap * 11, /*ncclFloat32*/ 7, /*ncclSum*/ 0, s->comm, s->stream) != 0)
        return fail(GPK_ERR_NCCL, "ncclAllReduce failed");
    return mark_grads_dense(s);  // non-zero wherever any rank had survivors
}

static int dp_reduce_scatter(gpk_session* s) {
    NcclApi* api = nccl();
    if (!api || !api->reduce_scatter || !api->group_start) return fail(GPK_ERR_NCCL, "NCCL not available");
    const uint64_t chunk = dp_chunk(s);
    float* g = s->grads.as<float>();
    if (api->group_start() != 0) return fail(GPK_ERR_NCCL, "ncclGroupStart failed");
    for (int k = 0; k < 11; ++k) {
        float* plane = g + (size_t)k * s->cap;  // in place: recv = send + rank * chunk
        if (api->reduce_scatter(plane, plane + (size_t)s->comm_rank * chunk, chunk, /*ncclFloat32*/ 7, /*ncclSum*/ 0,
                                s->comm, s->stream) != 0)
            return fail(GPK_ERR_NCCL, "ncclReduceScatter failed");
    }
    if (api->group_end() != 0) return fail(GPK_ERR_NCCL, "ncclGroupEnd failed");
    return GPK_OK;
}

static int dp_all_gather_params(gpk_session* s) {
    NcclApi* api = nccl();
    if (!api || !api->all_gather || !api->group_start) return fail(GPK_ERR_NCCL, "NCCL not available");
    const uint64_t chunk = dp_chunk(s);
    float* p = s->params.as<float>();
    if (api->group_start() != 0) return fail(GPK_ERR_NCCL, "ncclGroupStart failed");
    for (int k = 0; k < 11; ++k) {
        float* plane = p + (size_t)k * s->cap;  // in place: send = recv + rank * chunk
        if (api->all_gather(plane + (size_t)s->comm_rank * chunk, plane, chunk, /*ncclFloat32*/ 7, s->comm,
                            s->stream) != 0)
            return fail(GPK_ERR_NCCL, "ncclAllGather failed");
    }
    if (api->group_end() != 0) return fail(GPK_ERR_NCCL, "ncclGroupEnd failed");
    // the shard of the dense planes now holds other ranks' gradients too:
    // zero it (the sparse clear of the next prepare covers this rank's own
    // survivors elsewhere)
    const uint64_t chunk_bytes = chunk * 4;
    for (int k = 0; k < 11; ++k)
        CK(cudaMemsetAsync(s->grads.as<float>() + (size_t)k * s->cap + (size_t)s->comm_rank * chunk, 0, chunk_bytes,
                           s->stream));
    return GPK_OK;
}

// The union rows' sum over the ranks: one grouped all-reduce of the first
// ucap rows of each of the 11 planes, in place, on the session stream.
static int dp_union_allreduce(gpk_session* s) {
    NcclApi* api = nccl();
    if (!api || !s->comm || !api->group_start) return fail(GPK_ERR_STATE, "exchange: communicator not initialized");
    if (!s->urows.p) return fail(GPK_ERR_STATE, "exchange before the render phase");
    if (api->group_start() != 0) return fail(GPK_ERR_NCCL, "ncclGroupStart failed");
    for (int k = 0; k < 11; ++k) {
        float* plane = s->urows.as<float>() + (size_t)k * s->cap;
        if (api->all_reduce(plane, plane, s->ucap, /*ncclFloat32*/ 7, /*ncclSum*/ 0, s->comm, s->stream) != 0)
            return fail(GPK_ERR_NCCL, "ncclAllReduce (union rows) failed");
    }
    if (api->group_end() != 0) return fail(GPK_ERR_NCCL, "ncclGroupEnd failed");
    return GPK_OK;
}

static int dp_check(gpk_session* s, int world, int rank, const gpk_slice_pose* poses, const gpk_learning_rates* lr0,
                    int total) {
    if (!s || !poses || !lr0) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (s->owner) return fail(GPK_ERR_STATE, "data-parallel steps run on a session, not on a context");
    if (world < 1 || world > kMaxBatch || rank < 0 || rank >= world)
        return fail(GPK_ERR_INVALID_ARGUMENT, "data-parallel step: 1 <= world <= 8, 0 <= rank < world");
    if (total < 1) return fail(GPK_ERR_INVALID_ARGUMENT, "total iterations must be >= 1");
    if (s->accum_on) return fail(GPK_ERR_STATE, "densify accumulation is not gathered across ranks");
    return GPK_OK;
}

int gpk_train_step_dp(gpk_session* s, int32_t world, int32_t rank, const gpk_slice_pose* poses, const gpk_psf* psf,
                      const gpk_raster_config* cfg, double lambda, double dssim_scale, const gpk_learning_rates* lr0,
                      int32_t total_iterations, int32_t phases) {
    TRY(dp_check(s, world, rank, poses, lr0, total_iterations));
    if ((phases & GPK_DP_EXCHANGE) && !s->comm) return fail(GPK_ERR_STATE, "exchange: communicator not initialized");
    TRY(set_device(s));
    const int st = train_dp_body(s, world, rank, poses, psf, cfg, lambda, dssim_scale, lr0, total_iterations, phases);
    if (st != GPK_OK) s->consts_pending = false;
    TRY(st);
    return ok();
}

int gpk_dp_union_rows(gpk_session* s, uint64_t* rows, uint64_t* capacity) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    unsigned u[2] = {0, 0};
    if (s->uctrl.p) CK(cudaMemcpy(u, s->uctrl.p, 8, cudaMemcpyDeviceToHost));
    if (rows) *rows = u[0];
    if (capacity) *capacity = s->ucap;
    if (u[1]) return fail(GPK_ERR_STATE, "data-parallel union rows exceed the capacity (gpk_dp_reserve_union, recapture)");
    return ok();
}

int gpk_dp_reserve_union(gpk_session* s, uint64_t rows) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(dp_union_alloc(s));
    s->ucap = std::min<uint64_t>(s->cap, std::max<uint64_t>(rows, 1));
    ++s->alloc_epoch;  // captured graphs bake the exchange count
    return ok();
}

int gpk_allreduce_grads(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    NcclApi* api = nccl();
    void* comm = session_comm(s);
    if (!api || !comm) return fail(GPK_ERR_STATE, "allreduce: communicator not initialized");
    TRY(set_device(s));
    TRY(materialize_dense_grads(s));
    // 11 planes are contiguous with stride cap: reduce the whole [0, 11*cap) range.
    const int r = api->all_reduce(s->grads.p, s->grads.p, s->cap * 11, /*ncclFloat32*/ 7,
                                  /*ncclSum*/ 0, comm, s->stream);
    if (r != 0) return fail(GPK_ERR_NCCL, "ncclAllReduce failed");
    TRY(mark_grads_dense(s));  // non-zero wherever any rank had survivors
    return ok();
}


// ---- voxelizer ------------------------------------------------------------------

int gpk_voxelize(gpk_session* s, const gpk_voxelizer_config* cfg, float* volume_out) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(vox_prep_settled(s, cfg));
    {
        StageScope scope(s, GPK_STAGE_VOXEL_EVAL);
        launch_vox_eval(vox_eval_args(s), s->stream);
        CK(cudaGetLastError());
    }
    if (volume_out) {
        CK(cudaMemcpyAsync(volume_out, s->volume.p, s->vox.voxels * 4, cudaMemcpyDeviceToHost, s->stream));
        TRY(sync_and_check(s, "voxelize"));
    }
    return ok();
}

int gpk_voxel_tile_count(gpk_session* s, uint64_t* tiles, uint64_t* instances) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->vox.valid) return fail(GPK_ERR_STATE, "no voxelized volume");
    TRY(set_device(s));
    TRY(sync_and_check(s, "voxelize"));
    Control c;
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    if (tiles) *tiles = s->vox.tiles;
    if (instances) *instances = s->n ? c.pairs : 0;
    return ok();
}

int gpk_get_voxel_tile_lists(gpk_session* s, uint32_t* offsets, uint32_t* entries) {
    uint64_t T = 0, P = 0;
    TRY(gpk_voxel_tile_count(s, &T, &P));
    std::vector<uint32_t> keys(P);
    if (P) CK(cudaMemcpy(keys.data(), s->keys[s->vox.final_buf].p, P * 4, cudaMemcpyDeviceToHost));
    if (offsets) {
        uint64_t k = 0;
        for (uint64_t t = 0; t <= T; ++t) {
            while (k < P && keys[k] < (uint32_t)t) ++k;
            offsets[t] = (uint32_t)k;
        }
    }
    // values are set indices already (ascending within a tile, as the
    // reference's survivor order, voxelize.hpp:93-103)
    if (entries && P) CK(cudaMemcpy(entries, s->vals[s->vox.final_buf].p, P * 4, cudaMemcpyDeviceToHost));
    return ok();
}

int gpk_voxelize_backward(gpk_session* s, const gpk_voxelizer_config* cfg, const float* dl_dv,
                          float* grads_out) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    TRY(vox_prep_settled(s, cfg));
    Control c;
    CK(cudaMemcpy(&c, s->ctrl(), sizeof c, cudaMemcpyDeviceToHost));
    CK(s->vox_partials.ensure(std::max<uint64_t>(c.pairs, 1) * 40));
    if (dl_dv)
        CK(cudaMemcpyAsync(s->dl_dv_vol.p, dl_dv, s->vox.voxels * 4, cudaMemcpyHostToDevice, s->stream));
    CK(cudaMemsetAsync(s->grads.p, 0, s->cap * 11 * 4, s->stream));
    s->grads_in_slots = false;
    s->grads_in_union = false;
    TRY(mark_grads_dense(s));
    if (s->n) {
        StageScope scope(s, GPK_STAGE_VOXEL);
        launch_vox_bwd(vox_eval_args(s), s->stream);
        CK(cudaGetLastError());
        VoxChainLaunch ch;
        ch.params = s->params.as<float>();
        ch.cap = s->cap;
        ch.records = s->vox_records.as<VoxRecord>();
        ch.survivor_list = s->survivors.as<uint32_t>();
        ch.partials = s->vox_partials.as<float>();
        ch.ctrl = s->ctrl();
        ch.grads = s->grads.as<float>();
        ch.err = s->err();
        ch.v = s->vox.v;
        launch_vox_chain(ch, (int)std::min<uint64_t>((s->n + 127) / 128, (uint64_t)s->num_sms * 8), s->stream);
        CK(cudaGetLastError());
    }
    TRY(sync_and_check(s, "voxelize_backward"));
    if (grads_out && s->n) TRY(copy_planes_out(s, s->grads.as<float>(), grads_out));
    return ok();
}


/* ---- adaptive density control (optimize.hpp:228-344) --------------------- */

int gpk_densify_accum_enable(gpk_session* s, int on) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    const bool want = on != 0;
    if (want && !s->accum_on) {
        s->accum_on = true;
        TRY(accum_alloc_zero(s));
    }
    if (want != s->accum_on) s->accum_on = want;
    ++s->alloc_epoch;  // captured graphs hold the chain's accumulator pointers
    return ok();
}

int gpk_densify_accum_reset(gpk_session* s) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->accum_on) return fail(GPK_ERR_STATE, "densify accumulator not enabled");
    TRY(set_device(s));
    TRY(accum_alloc_zero(s));
    return ok();
}

int gpk_get_densify_accum(gpk_session* s, double* grad_norm_sum, int32_t* observations,
                          double* world_grad_sum) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->accum_on) return fail(GPK_ERR_STATE, "densify accumulator not enabled");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    if (grad_norm_sum && s->n) CK(cudaMemcpy(grad_norm_sum, s->acc_norm.p, s->n * 8, cudaMemcpyDeviceToHost));
    if (observations && s->n) CK(cudaMemcpy(observations, s->acc_obs.p, s->n * 4, cudaMemcpyDeviceToHost));
    if (world_grad_sum && s->n) CK(cudaMemcpy(world_grad_sum, s->acc_world.p, s->n * 24, cudaMemcpyDeviceToHost));
    return ok();
}

int gpk_set_densify_accum(gpk_session* s, const double* grad_norm_sum, const int32_t* observations,
                          const double* world_grad_sum) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (!s->accum_on) return fail(GPK_ERR_STATE, "densify accumulator not enabled");
    if (s->n && (!grad_norm_sum || !observations || !world_grad_sum))
        return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    TRY(set_device(s));
    CK(cudaStreamSynchronize(s->stream));
    if (s->n) {
        CK(cudaMemcpy(s->acc_norm.p, grad_norm_sum, s->n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(s->acc_obs.p, observations, s->n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(s->acc_world.p, world_grad_sum, s->n * 24, cudaMemcpyHostToDevice));
    }
    return ok();
}

// densify_and_prune (optimize.hpp:255-344) on the resident set: classify +
// block scan on the device, the split children's normals from the caller's
// generator (drawn in parent order, as the reference draws them), emit into
// fresh planes, then the new set (moments carried over, the step counter
// kept) replaces the old one. The accumulator is reset (fit, optimize.hpp:400).
static double draw_from_gpk_rng(void* user) {
    double v = 0.0;
    gpk_rng_normal(static_cast<gpk_rng*>(user), &v);
    return v;
}

int gpk_densify_and_prune(gpk_session* s, const gpk_densify_config* cfg, gpk_rng* rng,
                          gpk_densify_report* report) {
    if (!rng) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    return gpk_densify_and_prune_draw(s, cfg, draw_from_gpk_rng, rng, report);
}

int gpk_densify_and_prune_draw(gpk_session* s, const gpk_densify_config* cfg, gpk_normal_fn normal,
                               void* user, gpk_densify_report* report) {
    if (!s || !cfg || !normal) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (!s->accum_on) return fail(GPK_ERR_STATE, "densify accumulator not enabled");
    if (!(cfg->split_scale_divisor > 0.0)) return fail(GPK_ERR_INVALID_ARGUMENT, "split_scale_divisor must be > 0");
    TRY(set_device(s));
    TRY(lazy_kill(s));
    TRY(clear_gmap(s));  // the slot map of the last step is set-indexed
    const uint64_t n = s->n;
    DensifyLaunch a{};
    a.params = s->params.as<float>();
    a.m = s->adam_m.as<float>();
    a.v = s->adam_v.as<float>();
    a.cap = s->cap;
    a.n = n;
    a.acc_norm = s->acc_norm.as<double>();
    a.acc_obs = s->acc_obs.as<int>();
    a.acc_world = s->acc_world.as<double>();
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) {
        a.bmin[d] = s->bbox.min[d];
        a.bmax[d] = s->bbox.max[d];
    }
    {   // scene_extent = max extent (:257-259), as the reference evaluates it
        const double ex = s->bbox.max[0] - s->bbox.min[0], ey = s->bbox.max[1] - s->bbox.min[1],
                     ez = s->bbox.max[2] - s->bbox.min[2];
        ext = std::fmax(ex, std::fmax(ey, ez));
    }
    a.tau = cfg->tau;
    a.grad_threshold = cfg->grad_threshold;
    a.split_threshold = cfg->split_scale_fraction * ext;
    a.shrink = std::log(cfg->split_scale_divisor);
    a.mod = cfg->scale_modifier;
    const unsigned nb = densify_blocks(n);
    DevBuf cls, sums, normals, outp, outm, outv;
    CK(cls.ensure(std::max<uint64_t>(n, 1)));
    CK(sums.ensure((uint64_t)nb * 12 + 16));
    a.cls = cls.as<uint8_t>();
    a.block_sums = sums.as<unsigned>();
    a.totals = sums.as<unsigned>() + 3ull * nb;
    launch_densify_classify(a, s->stream);
    CK(cudaGetLastError());
    unsigned tot[3];
    CK(cudaMemcpyAsync(tot, a.totals, 12, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    const uint64_t kept = tot[0], born = tot[1], split = tot[2];
    const uint64_t n_new = kept + born;
    if (n_new >= (1ull << 31)) return fail(GPK_ERR_INVALID_ARGUMENT, "densify: set size must stay < 2^31");
    std::vector<double> xi(6 * split);
    for (uint64_t k = 0; k < xi.size(); ++k) xi[k] = normal(user);  // in parent order (:310)
    CK(normals.ensure(std::max<uint64_t>(xi.size(), 1) * 8));
    if (!xi.empty()) CK(cudaMemcpyAsync(normals.p, xi.data(), xi.size() * 8, cudaMemcpyHostToDevice, s->stream));
    const uint64_t need = (std::max<uint64_t>(n_new, 1) + kParamAlign - 1) / kParamAlign * kParamAlign;
    const uint64_t cap_out = std::max(need, s->cap);  // the plane stride after alloc_for_n
    for (DevBuf* b : {&outp, &outm, &outv}) {
        CK(b->ensure(cap_out * 44));
        CK(cudaMemsetAsync(b->p, 0, cap_out * 44, s->stream));
    }
    a.normals = normals.as<double>();
    a.out_params = outp.as<float>();
    a.out_m = outm.as<float>();
    a.out_v = outv.as<float>();
    a.cap_out = cap_out;
    launch_densify_emit(a, s->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));
    TRY(alloc_for_n(s, n_new));  // may reallocate the planes (contents not kept)
    if (s->cap != cap_out) return fail(GPK_ERR_CUDA, "densify: unexpected plane stride");
    CK(cudaMemcpyAsync(s->params.p, outp.p, cap_out * 44, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->adam_m.p, outm.p, cap_out * 44, cudaMemcpyDeviceToDevice, s->stream));
    CK(cudaMemcpyAsync(s->adam_v.p, outv.p, cap_out * 44, cudaMemcpyDeviceToDevice, s->stream));
    // gradients and prepared state refer to the old indices: clear them
    CK(cudaMemsetAsync(s->grads.p, 0, s->cap * 44, s->stream));
    s->grads_in_slots = false;
    s->grads_in_union = false;
    s->gmap_dirty = false;
    TRY(mark_grads_dense(s));
    s->prep.valid = false;
    s->prefilter.valid = false;
    TRY(accum_alloc_zero(s));
    CK(cudaStreamSynchronize(s->stream));
    for (DevBuf* b : {&cls, &sums, &normals, &outp, &outm, &outv}) b->release();
    if (report) {
        report->pruned = n - (kept + split);  // `kept` holds keeps and clone originals
        report->cloned = born - 2 * split;
        report->split = split;
    }
    return ok();
}

}  // extern "C"
