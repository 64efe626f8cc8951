// fit.cu — the fit driver on the device (fit, optimize.hpp:360-424): a host
// loop over the session's C-ABI, with the volume resident in HBM.
//
// Per iteration, as the reference (optimize.hpp:385-402):
//   k = rng.below(Z) (sample_slice :144-150); pose = slice_pose_for_index(k);
//   the target is slice k of the resident volume (z-major, so a contiguous
//   W*H run: one device-to-device copy into the session's target buffer);
//   gpk_train_step = prepare + rasterize + photometric_loss + backward (whose
//   chain adds the DensifyAccum statistics while the densify window is open)
//   + Adam with lr_at(lr0, it, iterations) from the device step counter;
//   densify_and_prune every densify_interval inside [densify_start,
//   densify_end] with the same generator (split normals drawn in order);
//   every progress_interval the monitor slice Z/2 is rendered, its loss taken
//   and the PSNR of the clamped render computed on the device (k_psnr_mse).
// The session is synchronized once per iteration: errors surface at their
// iteration (NumericFailure prefixed "fit: iteration N: ", optimize.hpp:419-421),
// and a slice whose (tile, Gaussian) pairs overflowed the buffers (the step
// then leaves parameters, moments and accumulators untouched) is replayed
// after the buffers grow.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/gpile_b200.h"
#include "common.cuh"

namespace {

constexpr int kPsnrThreads = 1024;

// Sum of squared differences of clamp(rendered, 0, 1) and the target (psnr,
// metrics.hpp:17-28, on the clamped monitor render, optimize.hpp:414-416), in
// fp64 with a fixed reduction order (deterministic).
__global__ void __launch_bounds__(kPsnrThreads) k_psnr_mse(const float* img, const float* tgt, uint64_t n,
                                                           double* out) {
    __shared__ double red[kPsnrThreads / 32];
    double acc = 0.0;
    for (uint64_t i = threadIdx.x; i < n; i += kPsnrThreads) {
        const double v = fmin(1.0, fmax(0.0, (double)img[i]));
        const double d = v - (double)tgt[i];
        acc += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) *out = v;
    }
}

struct DevMem {
    void* p = nullptr;
    ~DevMem() {
        if (p) cudaFree(p);
    }
};

int fail_fit(int code, const std::string& msg) { return gpk::set_last_error(code, msg); }

}  // namespace

extern "C" {

int gpk_default_init_count(uint64_t voxel_count, uint64_t* out) {
    if (!out) return GPK_ERR_INVALID_ARGUMENT;
    // default_init_count (optimize.hpp:64-66)
    *out = std::max<uint64_t>(1, std::min<uint64_t>(100000, 4 * voxel_count / 1000));
    return GPK_OK;
}

int gpk_fit(gpk_session* s, const float* volume, const int32_t dims[3], const double spacing[3],
            const double origin[3], const gpk_psf* psf, const gpk_fit_config* cfg,
            gpk_fit_progress_fn progress, void* user) {
#define FIT_TRY(expr)                                                                  \
    do {                                                                               \
        const int _st = (expr);                                                        \
        if (_st != GPK_OK) return _st; /* message already set */             \
    } while (0)
#define FIT_CK(expr)                                                                   \
    do {                                                                               \
        const cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) return fail_fit(GPK_ERR_CUDA, cudaGetErrorString(_e));  \
    } while (0)
    if (!dims || !spacing || !origin || !psf || !cfg)
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "fit: null argument");
    // VolumeGrid::validate (core.hpp:147-155), PsfSpec::validate (:111-116),
    // FitConfig::validate (optimize.hpp:45-58)
    for (int d = 0; d < 3; ++d) {
        if (dims[d] < 1) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "VolumeGrid: dims must be >= 1");
        if (!(spacing[d] > 0.0)) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "VolumeGrid: spacing must be > 0");
    }
    if (!(psf->sigma_x > 0.0) || !(psf->sigma_y > 0.0) || !(psf->sigma_z > 0.0))
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "PsfSpec: sigmas must be > 0");
    if (cfg->iterations < 1) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: iterations must be >= 1");
    if (!(cfg->lr_position > 0.0) || !(cfg->lr_opacity > 0.0) || !(cfg->lr_scale > 0.0) ||
        !(cfg->lr_rotation > 0.0))
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: learning rates must be > 0");
    if (!(cfg->densify_start < cfg->densify_end))
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: densify_start must be < densify_end");
    if (cfg->densify_interval < 1)
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: densify_interval must be >= 1");
    if (cfg->lambda < 0.0) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: lambda must be >= 0");
    if (!(cfg->tau >= 0.0 && cfg->tau < 1.0)) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: tau in [0,1)");
    if (cfg->init_mode != 0 && cfg->init_mode != 1)
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: init_mode must be random or grid");
    if (cfg->progress_interval < 1)
        return fail_fit(GPK_ERR_INVALID_ARGUMENT, "FitConfig: progress_interval must be >= 1");

    if (!s || !volume) return fail_fit(GPK_ERR_INVALID_ARGUMENT, "fit: null session or volume");

    const uint64_t W = (uint64_t)dims[0], H = (uint64_t)dims[1], Z = (uint64_t)dims[2];
    const uint64_t px = W * H, voxels = px * Z;
    // world_bounds (core.hpp:141-145)
    gpk_bounds bbox;
    for (int d = 0; d < 3; ++d) {
        bbox.min[d] = origin[d] - spacing[d] * 0.5;
        bbox.max[d] = origin[d] + (dims[d] - 0.5) * spacing[d];
    }
    const double scale_base = 1.5 * (spacing[0] + spacing[1] + spacing[2]) / 3.0;
    uint64_t m = cfg->init_count;
    if (m == 0) FIT_TRY(gpk_default_init_count(voxels, &m));
    std::vector<double> rec(m * 11);
    if (cfg->init_mode == 1)
        FIT_TRY(gpk_init_grid(m, &bbox, scale_base, cfg->rng_seed, rec.data()));
    else
        FIT_TRY(gpk_init_random(m, &bbox, scale_base, cfg->rng_seed, rec.data()));
    FIT_TRY(gpk_set_gaussians_f64(s, m, rec.data(), &bbox));  // also resets Adam
    rec.clear();
    rec.shrink_to_fit();
    FIT_TRY(gpk_densify_accum_enable(s, 1));

    void* stream_v = nullptr;
    FIT_TRY(gpk_session_get_stream(s, &stream_v));
    cudaStream_t st = static_cast<cudaStream_t>(stream_v);
    DevMem vol, mse;
    FIT_CK(cudaMalloc(&vol.p, voxels * 4));
    FIT_CK(cudaMalloc(&mse.p, 8));
    FIT_CK(cudaMemcpyAsync(vol.p, volume, voxels * 4, cudaMemcpyHostToDevice, st));
    const float* vol_f = static_cast<const float*>(vol.p);
    // size the image-shaped buffers (target) once from the host
    FIT_TRY(gpk_upload(s, GPK_BUF_TARGET, volume, px * 4));
    FIT_TRY(gpk_session_synchronize(s));

    gpk_rng* rng = nullptr;
    FIT_TRY(gpk_rng_create(cfg->rng_seed + 0x9e3779b97f4a7c15ull, &rng));
    struct RngGuard {
        gpk_rng* r;
        ~RngGuard() { gpk_rng_destroy(r); }
    } rng_guard{rng};

    const gpk_raster_config rcfg{cfg->tau, cfg->tile_size, cfg->footprint_sigmas, cfg->scale_modifier};
    const gpk_learning_rates lr0{cfg->lr_position, cfg->lr_opacity, cfg->lr_scale, cfg->lr_rotation};
    const gpk_densify_config dcfg{cfg->tau, cfg->grad_threshold, cfg->split_scale_fraction,
                                  cfg->split_scale_divisor, cfg->scale_modifier};
    const int monitor_slice = (int)(Z / 2);
    gpk_slice_pose mon_pose;
    FIT_TRY(gpk_slice_pose_for_index(dims, spacing, origin, monitor_slice, &mon_pose));

    auto load_target = [&](int k) -> int {
        void* tp = nullptr;
        uint64_t tb = 0;
        int stt = gpk_device_buffer(s, GPK_BUF_TARGET, &tp, &tb);
        if (stt != GPK_OK) return stt;
        const cudaError_t e = cudaMemcpyAsync(tp, vol_f + (uint64_t)k * px, px * 4, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? GPK_OK : GPK_ERR_CUDA;
    };
    auto iter_fail = [&](int it, int code) {
        return fail_fit(code, "fit: iteration " + std::to_string(it) + ": " + gpk_last_error_message());
    };

    // After the densify window the set size is fixed: each slice's step is a
    // CUDA graph captured once (GPK_FIT_NO_GRAPHS=1: direct launches).
    const bool graphs = std::getenv("GPK_FIT_NO_GRAPHS") == nullptr;
    std::vector<int32_t> graph_of(Z, -1);
    std::vector<int> visits(Z, 0);
    auto drop_graphs = [&] {
        gpk_graph_destroy_all(s);
        std::fill(graph_of.begin(), graph_of.end(), -1);
    };
    struct GraphGuard {
        gpk_session* s;
        ~GraphGuard() { gpk_graph_destroy_all(s); }
    } graph_guard{s};
    double prof[4] = {0, 0, 0, 0};
    const bool profile = std::getenv("GPK_FIT_PROFILE") != nullptr;
    const auto tfit = std::chrono::steady_clock::now();
    for (int it = 1; it <= cfg->iterations; ++it) {
        uint64_t k64 = 0;
        FIT_TRY(gpk_rng_below(rng, Z, &k64));
        const int k = (int)k64;
        gpk_slice_pose pose;
        FIT_TRY(gpk_slice_pose_for_index(dims, spacing, origin, k, &pose));
        // the DensifyAccum only feeds densify events (fit adds every
        // iteration's statistics; none are read after the window closes)
        if (it == cfg->densify_end + 1) FIT_TRY(gpk_densify_accum_enable(s, 0));
        for (int attempt = 0;; ++attempt) {
            const auto t0 = std::chrono::steady_clock::now();
            int stt = load_target(k);
            if (stt != GPK_OK) return iter_fail(it, stt);
            const auto t1 = std::chrono::steady_clock::now();
            // a slice's graph is captured on its second visit after the window
            // (a capture costs about ten direct steps' host time)
            if (graphs && it > cfg->densify_end && (graph_of[k] >= 0 || (attempt == 0 && ++visits[k] >= 2) ||
                                                    (attempt > 0 && visits[k] >= 2))) {
                // the set is frozen: replay the step's CUDA graph for this slice
                // (captured on first use; bitwise the direct step)
                for (int g = 0; g < 2; ++g) {
                    stt = GPK_OK;
                    if (graph_of[k] < 0) {
                        int32_t gid = -1;
                        stt = gpk_graph_capture_train(s, &pose, psf, &rcfg, cfg->lambda, cfg->dssim_scale, &lr0,
                                                      cfg->iterations, &gid);
                        if (stt == GPK_OK) graph_of[k] = gid;
                    }
                    if (stt == GPK_OK) stt = gpk_graph_launch(s, graph_of[k]);
                    if (stt != GPK_ERR_STATE) break;
                    drop_graphs();  // buffers were reallocated since capture
                }
            } else {
                stt = gpk_train_step(s, &pose, psf, &rcfg, cfg->lambda, cfg->dssim_scale, &lr0, cfg->iterations);
            }
            const auto t2 = std::chrono::steady_clock::now();
            if (stt == GPK_OK) stt = gpk_session_synchronize(s);
            const auto t3 = std::chrono::steady_clock::now();
            prof[0] += std::chrono::duration<double>(t1 - t0).count();
            prof[1] += std::chrono::duration<double>(t2 - t1).count();
            prof[2] += std::chrono::duration<double>(t3 - t2).count();
            if (stt == GPK_OK) break;
            uint64_t surv = 0, pairs = 0;
            if (stt == GPK_ERR_STATE && attempt == 0 && gpk_prepared_count(s, &surv, &pairs) == GPK_OK) {
                // pair overflow: nothing was updated; grow the buffers and replay
                if (gpk_session_reserve_pairs(s, pairs + pairs / 4 + 1024) == GPK_OK) {
                    drop_graphs();
                    continue;
                }
            }
            return iter_fail(it, stt);
        }
        if (it >= cfg->densify_start && it <= cfg->densify_end && it % cfg->densify_interval == 0) {
            gpk_densify_report rep;
            const int stt = gpk_densify_and_prune(s, &dcfg, rng, &rep);  // resets the accumulator
            if (stt != GPK_OK) return iter_fail(it, stt);
        }
        if (progress && (it % cfg->progress_interval == 0 || it == cfg->iterations)) {
            gpk_fit_progress p{};
            p.iteration = it;
            FIT_TRY(gpk_download(s, GPK_BUF_LOSS, &p.loss, 8));  // this iteration's loss
            FIT_TRY(gpk_session_synchronize(s));
            FIT_TRY(gpk_gaussian_count(s, &p.count));
            FIT_TRY(gpk_prepare(s, &mon_pose, psf, &rcfg));
            FIT_TRY(gpk_rasterize(s, nullptr));
            int stt = load_target(monitor_slice);
            if (stt != GPK_OK) return iter_fail(it, stt);
            FIT_TRY(gpk_photometric_loss(s, nullptr, cfg->lambda, cfg->dssim_scale, &p.monitor_loss, nullptr));
            void *ip = nullptr, *tp = nullptr;
            FIT_TRY(gpk_device_buffer(s, GPK_BUF_IMAGE, &ip, nullptr));
            FIT_TRY(gpk_device_buffer(s, GPK_BUF_TARGET, &tp, nullptr));
            k_psnr_mse<<<1, kPsnrThreads, 0, st>>>(static_cast<const float*>(ip), static_cast<const float*>(tp),
                                                   px, static_cast<double*>(mse.p));
            FIT_CK(cudaGetLastError());
            double sse = 0.0;
            FIT_CK(cudaMemcpyAsync(&sse, mse.p, 8, cudaMemcpyDeviceToHost, st));
            FIT_CK(cudaStreamSynchronize(st));
            const double msev = sse / (double)px;
            p.psnr2d = msev == 0.0 ? GPK_PSNR_INF : 10.0 * std::log10(1.0 / msev);
            progress(&p, user);
        }
    }
    FIT_TRY(gpk_session_synchronize(s));
    if (profile)
        std::fprintf(stderr, "gpk_fit profile: total %.3f s; target %.3f, train_step %.3f, sync %.3f s\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - tfit).count(), prof[0],
                     prof[1], prof[2]);
    return GPK_OK;
#undef FIT_TRY
#undef FIT_CK
}

}  // extern "C"
