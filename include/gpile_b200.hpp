// gpile_b200.hpp — C++ drop-in for the reference's slice-renderer hot path
// (GaussianPile, proj/include/gpile) on the B200 C-ABI
// (gpile_b200.h). The types are the reference's own — include this header
// where the reference headers are on the include path — and every function
// keeps the reference signature, argument meaning and exception types:
//
//   reference (namespace gpile)                 drop-in (namespace gpile::b200)
//   prepare_gaussians     render.hpp:83         prepare_gaussians
//   rasterize_prepared    render.hpp:166        rasterize_prepared
//   rasterize_slice       render.hpp:194        rasterize_slice
//   backward_prepared     backward.hpp:97       backward_prepared
//   backward_slice        backward.hpp:189      backward_slice
//   photometric_loss      loss.hpp:13           photometric_loss
//   lr_at                 optimize.hpp:71       lr_at
//   adam_step             optimize.hpp:195      adam_step
//   voxelize              voxelize.hpp:113      voxelize
//   voxelize_backward     voxelize.hpp:152      voxelize_backward
//   densify_and_prune     optimize.hpp:255      densify_and_prune
//   fit                   optimize.hpp:360      fit
//   save_checkpoint       checkpoint.hpp:38     save_checkpoint
//   load_checkpoint       checkpoint.hpp:60     load_checkpoint
//   morton_sort           morton.hpp:33         morton_sort
//   quantize              quant.hpp:67          quantize
//
// Errors: GPK_ERR_INVALID_ARGUMENT -> std::invalid_argument,
// GPK_ERR_DEGENERATE_COVARIANCE -> gpile::DegenerateCovariance,
// GPK_ERR_NUMERIC_FAILURE -> gpile::NumericFailure (message names the first
// failing primitive, as backward.hpp:182-184), anything else ->
// std::runtime_error. Calls are blocking, like the reference's.
//
// The free functions marshal the GaussianSet (AoS f64 -> f32 records) per
// call, as the reference's value semantics require. For throughput keep the
// parameters resident: use gpile::b200::Session (set_gaussians once, then
// fwd_bwd / train_step, parameters never leave HBM).
//
// PreparedGaussian: prepare_gaussians fills every field the reference fills
// (render.hpp:68-79; gpk_get_prepared_fields, the reference's fp64 operation
// order). The device keeps the most recent prepared slice; the drop-in also
// remembers the last few prepared vectors it returned on this thread (their
// pose, PSF, config and the set they came from), so rasterize_prepared /
// backward_prepared accept any of them — a vector other than the latest is
// prepared again on the device from the remembered inputs. A vector the
// drop-in did not return (or forgot: more than kPreparedMemory prepares ago)
// raises std::logic_error.
#pragma once

#include <gpile/backward.hpp>
#include <gpile/checkpoint.hpp>
#include <gpile/core.hpp>
#include <gpile/errors.hpp>
#include <gpile/image.hpp>
#include <gpile/loss.hpp>
#include <gpile/morton.hpp>
#include <gpile/optimize.hpp>
#include <gpile/quant.hpp>
#include <gpile/render.hpp>
#include <gpile/voxelize.hpp>

#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gpile_b200.h"

namespace gpile {
namespace b200 {

inline void check(int status) {
    if (status == GPK_OK) return;
    const char* m = gpk_last_error_message();
    const std::string msg = m ? m : "gpile_b200 error";
    switch (status) {
        case GPK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case GPK_ERR_DEGENERATE_COVARIANCE: throw DegenerateCovariance(msg);
        case GPK_ERR_NUMERIC_FAILURE: throw NumericFailure(msg);
        case GPK_ERR_CORRUPT_CONTAINER: throw CorruptContainer(msg);
        case GPK_ERR_LOAD: throw LoadError(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace detail {

inline std::vector<float> records_of(const GaussianSet& set) {
    std::vector<float> r(set.size() * 11);
    for (std::size_t i = 0; i < set.size(); ++i) {
        const GaussianPrimitive& g = set.primitives[i];
        const double v[11] = {g.mu.x, g.mu.y, g.mu.z, g.log_scale.x, g.log_scale.y, g.log_scale.z,
                              g.quat.w, g.quat.x, g.quat.y, g.quat.z, g.alpha_raw};
        for (int k = 0; k < 11; ++k) r[11 * i + k] = static_cast<float>(v[k]);
    }
    return r;
}

inline void store_records(const std::vector<float>& r, GaussianSet& set) {
    for (std::size_t i = 0; i < set.size(); ++i) {
        GaussianPrimitive& g = set.primitives[i];
        const float* v = &r[11 * i];
        g.mu = {v[0], v[1], v[2]};
        g.log_scale = {v[3], v[4], v[5]};
        g.quat = {v[6], v[7], v[8], v[9]};
        g.alpha_raw = v[10];
    }
}

inline GaussianGradients grads_of(const std::vector<float>& r, std::size_t n) {
    GaussianGradients g(n);
    for (std::size_t i = 0; i < n; ++i) {
        const float* v = &r[11 * i];
        g.d_mu[i] = {v[0], v[1], v[2]};
        g.d_log_scale[i] = {v[3], v[4], v[5]};
        g.d_quat[i] = {v[6], v[7], v[8], v[9]};
        g.d_alpha_raw[i] = v[10];
    }
    return g;
}

inline std::vector<float> records_of(const GaussianGradients& g) {
    std::vector<float> r(g.size() * 11);
    for (std::size_t i = 0; i < g.size(); ++i) {
        const double v[11] = {g.d_mu[i].x, g.d_mu[i].y, g.d_mu[i].z, g.d_log_scale[i].x, g.d_log_scale[i].y,
                              g.d_log_scale[i].z, g.d_quat[i].w, g.d_quat[i].x, g.d_quat[i].y, g.d_quat[i].z,
                              g.d_alpha_raw[i]};
        for (int k = 0; k < 11; ++k) r[11 * i + k] = static_cast<float>(v[k]);
    }
    return r;
}

inline gpk_bounds bounds_of(const Bounds& b) {
    return {{b.min.x, b.min.y, b.min.z}, {b.max.x, b.max.y, b.max.z}};
}

inline gpk_slice_pose pose_of(const SlicePose& p) {
    gpk_slice_pose c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.rotation[3 * i + j] = p.rotation.m[i][j];
    c.translation[0] = p.translation.x;
    c.translation[1] = p.translation.y;
    c.translation[2] = p.translation.z;
    c.width = p.width;
    c.height = p.height;
    c.pixel_spacing[0] = p.pixel_spacing.x;
    c.pixel_spacing[1] = p.pixel_spacing.y;
    c.principal_point[0] = p.principal_point.x;
    c.principal_point[1] = p.principal_point.y;
    return c;
}

inline gpk_psf psf_of(const PsfSpec& f) { return {f.sigma_x, f.sigma_y, f.sigma_z}; }

inline gpk_raster_config cfg_of(const RasterConfig& c) {
    return {c.tau, c.tile_size, c.footprint_sigmas, c.scale_modifier};
}

inline gpk_voxelizer_config vcfg_of(const VoxelizerConfig& v) {
    gpk_voxelizer_config c;
    for (int d = 0; d < 3; ++d) {
        c.dims[d] = v.dims[d];
        c.tile_dims[d] = v.tile_dims[d];
    }
    c.spacing[0] = v.spacing.x;
    c.spacing[1] = v.spacing.y;
    c.spacing[2] = v.spacing.z;
    c.origin[0] = v.origin.x;
    c.origin[1] = v.origin.y;
    c.origin[2] = v.origin.z;
    c.support_sigmas = v.support_sigmas;
    c.scale_modifier = v.scale_modifier;
    return c;
}

inline std::vector<float> pixels_of(const SliceImage& img) {
    return std::vector<float>(img.pixels.begin(), img.pixels.end());
}

}  // namespace detail

// One session per GPU: parameters, gradients and Adam moments stay in HBM.
class Session {
  public:
    explicit Session(int device = 0, void* cuda_stream = nullptr) { check(gpk_session_create(device, cuda_stream, &s_)); }
    ~Session() {
        if (s_) gpk_session_destroy(s_);
    }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;
    Session(Session&& o) noexcept : s_(std::exchange(o.s_, nullptr)) {}

    gpk_session* handle() const { return s_; }

    void set_gaussians(const GaussianSet& set) {
        const std::vector<float> r = detail::records_of(set);
        const gpk_bounds b = detail::bounds_of(set.bbox);
        check(gpk_set_gaussians(s_, set.size(), r.data(), &b));
    }
    // Parameters back into `set` (same size as uploaded).
    void get_gaussians(GaussianSet& set) const {
        std::vector<float> r(set.size() * 11);
        check(gpk_get_gaussians(s_, r.data()));
        detail::store_records(r, set);
    }

    std::vector<PreparedGaussian> prepare(const SlicePose& pose, const PsfSpec& psf, const RasterConfig& cfg) {
        const gpk_slice_pose p = detail::pose_of(pose);
        const gpk_psf f = detail::psf_of(psf);
        const gpk_raster_config c = detail::cfg_of(cfg);
        check(gpk_prepare(s_, &p, &f, &c));
        uint64_t S = 0, T = 0;
        check(gpk_prepared_count(s_, &S, &T));
        std::vector<uint32_t> idx(S);
        std::vector<int32_t> bnd(4 * S);
        std::vector<double> fld(GPK_PREPARED_FIELDS * S);
        if (S) {
            check(gpk_get_prepared(s_, idx.data(), bnd.data(), nullptr));
            check(gpk_get_prepared_fields(s_, fld.data()));
        }
        std::vector<PreparedGaussian> out(S);
        auto mat3 = [](const double* f) {
            Mat3 m;
            for (int i = 0; i < 9; ++i) m.m[i / 3][i % 3] = f[i];
            return m;
        };
        for (uint64_t k = 0; k < S; ++k) {
            PreparedGaussian& g = out[k];
            const double* f = &fld[GPK_PREPARED_FIELDS * k];
            g.index = idx[k];
            g.lo_x = bnd[4 * k];
            g.hi_x = bnd[4 * k + 1];
            g.lo_y = bnd[4 * k + 2];
            g.hi_y = bnd[4 * k + 3];
            g.alpha = f[0];
            g.opacity_r = f[1];
            g.alpha_tilde = f[2];
            g.mu_c = {f[3], f[4], f[5]};
            g.mu_e = {f[6], f[7], f[8]};
            g.sigma_c = mat3(f + 9);
            g.sigma_c_inv = mat3(f + 18);
            g.sigma_e = mat3(f + 27);
            g.mu_2d = {f[36], f[37]};
            g.cov2d = {f[38], f[39], f[40], f[41]};
            g.conic = {f[42], f[43], f[44], f[45]};
            g.det2 = f[46];
        }
        pose_ = pose;
        return out;
    }

    SliceImage rasterize() { return rasterize(pose_); }
    SliceImage rasterize(const SlicePose& pose) {
        SliceImage img(pose.width, pose.height);
        std::vector<float> px(img.size());
        check(gpk_rasterize(s_, px.data()));
        std::copy(px.begin(), px.end(), img.pixels.begin());
        return img;
    }

    GaussianGradients backward(const SliceImage& dl_di, ScreenGradStats* stats = nullptr) {
        return backward(dl_di, stats, pose_);
    }
    GaussianGradients backward(const SliceImage& dl_di, ScreenGradStats* stats, const SlicePose& pose) {
        if (dl_di.width != pose.width || dl_di.height != pose.height)
            throw std::invalid_argument("backward_prepared: dl_di shape mismatch");  // backward.hpp:102-103
        uint64_t n = 0;
        check(gpk_gaussian_count(s_, &n));
        const std::vector<float> dl = detail::pixels_of(dl_di);
        std::vector<float> g(n * 11);
        std::vector<double> nrm, wld;
        std::vector<uint8_t> obs;
        gpk_screen_stats st{};
        if (stats) {
            nrm.resize(n);
            obs.resize(n);
            wld.resize(3 * n);
            st = {nrm.data(), obs.data(), wld.data()};
        }
        check(gpk_backward(s_, dl.data(), g.data(), stats ? &st : nullptr));
        if (stats) {
            *stats = ScreenGradStats(n);
            for (uint64_t i = 0; i < n; ++i) {
                stats->mu2d_grad_norm[i] = nrm[i];
                stats->observed[i] = obs[i];
                stats->world_pos_grad[i] = {wld[3 * i], wld[3 * i + 1], wld[3 * i + 2]};
            }
        }
        return detail::grads_of(g, n);
    }

    // U1 / U2 on resident parameters; dL/dI resp. the target come from the
    // session buffers (gpk_upload GPK_BUF_DL_DI / GPK_BUF_TARGET).
    void fwd_bwd(const SlicePose& pose, const PsfSpec& psf, const RasterConfig& cfg) {
        const gpk_slice_pose p = detail::pose_of(pose);
        const gpk_psf f = detail::psf_of(psf);
        const gpk_raster_config c = detail::cfg_of(cfg);
        check(gpk_fwd_bwd_slice(s_, &p, &f, &c));
        pose_ = pose;
    }
    void train_step(const SlicePose& pose, const PsfSpec& psf, const RasterConfig& cfg, double lambda,
                    double dssim_scale, const LearningRates& lr0, int total_iterations) {
        const gpk_slice_pose p = detail::pose_of(pose);
        const gpk_psf f = detail::psf_of(psf);
        const gpk_raster_config c = detail::cfg_of(cfg);
        const gpk_learning_rates l{lr0.position, lr0.opacity, lr0.scale, lr0.rotation};
        check(gpk_train_step(s_, &p, &f, &c, lambda, dssim_scale, &l, total_iterations));
        pose_ = pose;
    }

    // Target slot 0 or 1 for later target uploads and losses (gpk_set_target_slot):
    // a loop alternating slots overlaps each upload with the previous step.
    void set_target_slot(int slot) { check(gpk_set_target_slot(s_, slot)); }

  private:
    gpk_session* s_ = nullptr;
    SlicePose pose_{};
};

namespace detail {

constexpr std::size_t kPreparedMemory = 8;  // prepared vectors remembered per thread

// One prepared vector the drop-in returned: its identity (storage, size and a
// fingerprint of its integer content) and the inputs that produced it.
struct PreparedEntry {
    const void* data = nullptr;
    std::size_t size = 0;
    uint64_t fingerprint = 0;
    uint64_t serial = 0;               // 1 + position in this thread's prepare sequence
    SlicePose pose{};
    PsfSpec psf{};
    RasterConfig cfg{};
    std::shared_ptr<const std::vector<float>> records;  // the set it was prepared from
    gpk_bounds bbox{};
};

inline uint64_t fingerprint_of(const std::vector<PreparedGaussian>& v) {
    uint64_t h = 1469598103934665603ull ^ v.size();
    for (const PreparedGaussian& g : v) {
        const uint64_t w[3] = {g.index, (uint64_t)(uint32_t)g.lo_x | ((uint64_t)(uint32_t)g.hi_x << 32),
                               (uint64_t)(uint32_t)g.lo_y | ((uint64_t)(uint32_t)g.hi_y << 32)};
        for (uint64_t x : w) h = (h ^ x) * 1099511628211ull;
    }
    return h;
}

// This thread's session on device 0, the prepared vectors it returned, and
// which of them the device holds now.
struct ThreadState {
    std::unique_ptr<Session> session;
    std::vector<PreparedEntry> prepared;   // most recent last, at most kPreparedMemory
    uint64_t serial = 0;
    uint64_t device_serial = 0;            // the entry whose slice the device holds (0: none)
    const std::vector<float>* device_records = nullptr;
};

inline ThreadState& state() {
    thread_local ThreadState st;
    if (!st.session) st.session = std::make_unique<Session>(0);
    return st;
}

// Make the device hold `prepared`'s slice: the latest prepare as is, an older
// remembered one prepared again from its own set, pose, PSF and config.
inline const PreparedEntry& bind_prepared(const std::vector<PreparedGaussian>& prepared) {
    ThreadState& st = state();
    const uint64_t fp = fingerprint_of(prepared);
    for (auto it = st.prepared.rbegin(); it != st.prepared.rend(); ++it) {
        if (it->data != prepared.data() || it->size != prepared.size() || it->fingerprint != fp) continue;
        if (st.device_serial != it->serial) {
            gpk_session* h = st.session->handle();
            if (st.device_records != it->records.get()) {
                check(gpk_set_gaussians(h, it->records->size() / 11, it->records->data(), &it->bbox));
                st.device_records = it->records.get();
            }
            const gpk_slice_pose p = pose_of(it->pose);
            const gpk_psf f = psf_of(it->psf);
            const gpk_raster_config c = cfg_of(it->cfg);
            check(gpk_prepare(h, &p, &f, &c));
            st.device_serial = it->serial;
        }
        return *it;
    }
    throw std::logic_error(
        "gpile::b200: prepared vector was not returned by one of this thread's recent prepare_gaussians calls");
}

}  // namespace detail

// The thread's session for direct use; whoever takes it may change the
// resident set or prepared slice, so the next rasterize_prepared /
// backward_prepared binds its vector again.
inline Session& default_session() {
    detail::ThreadState& st = detail::state();
    st.device_serial = 0;
    st.device_records = nullptr;
    return *st.session;
}

// ---- render.hpp ------------------------------------------------------------------
inline std::vector<PreparedGaussian> prepare_gaussians(const GaussianSet& set, const SlicePose& pose,
                                                       const PsfSpec& psf, const RasterConfig& cfg) {
    detail::ThreadState& st = detail::state();
    auto recs = std::make_shared<const std::vector<float>>(detail::records_of(set));
    const gpk_bounds b = detail::bounds_of(set.bbox);
    check(gpk_set_gaussians(st.session->handle(), set.size(), recs->data(), &b));
    st.device_records = recs.get();
    std::vector<PreparedGaussian> out = st.session->prepare(pose, psf, cfg);
    detail::PreparedEntry e;
    e.data = out.data();
    e.size = out.size();
    e.fingerprint = detail::fingerprint_of(out);
    e.serial = ++st.serial;
    e.pose = pose;
    e.psf = psf;
    e.cfg = cfg;
    e.records = std::move(recs);
    e.bbox = b;
    // vectors are returned by value: a moved-from result keeps its heap
    // storage, so data() identifies it (with the size and the fingerprint)
    if (st.prepared.size() == detail::kPreparedMemory) st.prepared.erase(st.prepared.begin());
    st.prepared.push_back(std::move(e));
    st.device_serial = st.serial;
    return out;
}

// The remembered slice of `prepared` rendered (render.hpp:166-192); pose and
// cfg are the caller's and must describe the same slice.
inline SliceImage rasterize_prepared(const std::vector<PreparedGaussian>& prepared, const SlicePose& pose,
                                     const RasterConfig& cfg) {
    const detail::PreparedEntry& e = detail::bind_prepared(prepared);
    if (pose.width != e.pose.width || pose.height != e.pose.height || cfg.tile_size != e.cfg.tile_size)
        throw std::invalid_argument("rasterize_prepared: pose / config differ from the prepared slice");
    return detail::state().session->rasterize(pose);
}

inline SliceImage rasterize_slice(const GaussianSet& set, const SlicePose& pose, const PsfSpec& psf,
                                  const RasterConfig& cfg = {}) {
    const auto prep = b200::prepare_gaussians(set, pose, psf, cfg);  // qualified: ADL also finds gpile::
    return b200::rasterize_prepared(prep, pose, cfg);
}

// ---- backward.hpp ----------------------------------------------------------------
inline GaussianGradients backward_prepared(const GaussianSet& set, const std::vector<PreparedGaussian>& prepared,
                                           const SlicePose& pose, const SliceImage& dl_di,
                                           const RasterConfig& cfg, ScreenGradStats* stats = nullptr) {
    (void)cfg;
    const detail::PreparedEntry& e = detail::bind_prepared(prepared);
    if (set.size() * 11 != e.records->size())
        throw std::invalid_argument("backward_prepared: set does not match the prepared slice");
    if (pose.width != e.pose.width || pose.height != e.pose.height)
        throw std::invalid_argument("backward_prepared: pose differs from the prepared slice");
    return detail::state().session->backward(dl_di, stats, pose);
}

inline GaussianGradients backward_slice(const GaussianSet& set, const SlicePose& pose, const PsfSpec& psf,
                                        const SliceImage& dl_di, const RasterConfig& cfg = {},
                                        ScreenGradStats* stats = nullptr) {
    const auto prep = b200::prepare_gaussians(set, pose, psf, cfg);
    return b200::backward_prepared(set, prep, pose, dl_di, cfg, stats);
}

// ---- loss.hpp --------------------------------------------------------------------
inline double photometric_loss(const SliceImage& rendered, const SliceImage& target, double lambda,
                               SliceImage& dl_di, double dssim_scale = 0.5) {
    if (rendered.width != target.width || rendered.height != target.height)
        throw std::invalid_argument("photometric_loss: image shape mismatch");  // loss.hpp:15-16
    const std::vector<float> r = detail::pixels_of(rendered), t = detail::pixels_of(target);
    std::vector<float> dl(r.size());
    double loss = 0.0;
    check(gpk_photometric_loss_images(default_session().handle(), rendered.width, rendered.height, r.data(),
                                      t.data(), lambda, dssim_scale, &loss, dl.data()));
    dl_di = SliceImage(rendered.width, rendered.height);
    std::copy(dl.begin(), dl.end(), dl_di.pixels.begin());
    return loss;
}

// ---- optimize.hpp ----------------------------------------------------------------
inline double lr_at(double lr0, int iteration, int total) { return gpk_lr_at(lr0, iteration, total); }

inline void adam_step(GaussianSet& set, const GaussianGradients& grads, AdamState& state,
                      const LearningRates& lrs) {
    const std::size_t n = set.size();
    if (grads.size() != n || state.m_a.size() != n)
        throw std::invalid_argument("adam_step: size mismatch");  // optimize.hpp:197-198
    Session& s = default_session();
    s.set_gaussians(set);
    std::vector<float> m(n * 11), v(n * 11);
    for (std::size_t i = 0; i < n; ++i) {
        const double mm[11] = {state.m_mu[i].x, state.m_mu[i].y, state.m_mu[i].z, state.m_ls[i].x, state.m_ls[i].y,
                               state.m_ls[i].z, state.m_q[i].w, state.m_q[i].x, state.m_q[i].y, state.m_q[i].z,
                               state.m_a[i]};
        const double vv[11] = {state.v_mu[i].x, state.v_mu[i].y, state.v_mu[i].z, state.v_ls[i].x, state.v_ls[i].y,
                               state.v_ls[i].z, state.v_q[i].w, state.v_q[i].x, state.v_q[i].y, state.v_q[i].z,
                               state.v_a[i]};
        for (int k = 0; k < 11; ++k) {
            m[11 * i + k] = static_cast<float>(mm[k]);
            v[11 * i + k] = static_cast<float>(vv[k]);
        }
    }
    check(gpk_set_adam_state(s.handle(), m.data(), v.data(), state.step));
    const std::vector<float> g = detail::records_of(grads);
    check(gpk_set_gradients(s.handle(), g.data()));
    const gpk_learning_rates l{lrs.position, lrs.opacity, lrs.scale, lrs.rotation};
    const gpk_adam_hparams hp{state.beta1, state.beta2, state.eps};
    check(gpk_adam_step(s.handle(), &l, &hp));
    int64_t step = 0;
    check(gpk_get_adam_state(s.handle(), m.data(), v.data(), &step));
    s.get_gaussians(set);
    state.step = static_cast<long>(step);
    for (std::size_t i = 0; i < n; ++i) {
        const float* a = &m[11 * i];
        const float* b = &v[11 * i];
        state.m_mu[i] = {a[0], a[1], a[2]};
        state.m_ls[i] = {a[3], a[4], a[5]};
        state.m_q[i] = {a[6], a[7], a[8], a[9]};
        state.m_a[i] = a[10];
        state.v_mu[i] = {b[0], b[1], b[2]};
        state.v_ls[i] = {b[3], b[4], b[5]};
        state.v_q[i] = {b[6], b[7], b[8], b[9]};
        state.v_a[i] = b[10];
    }
}

// ---- voxelize.hpp ----------------------------------------------------------------
inline VolumeGrid voxelize(const GaussianSet& set, const VoxelizerConfig& cfg) {
    Session& s = default_session();
    s.set_gaussians(set);
    const gpk_voxelizer_config c = detail::vcfg_of(cfg);
    VolumeGrid vol;
    for (int d = 0; d < 3; ++d) vol.dims[d] = cfg.dims[d];
    vol.spacing = cfg.spacing;
    vol.origin = cfg.origin;
    // validation (voxelize.hpp:24-37, incl. the 2^31 refusal) happens in the
    // library before anything is allocated
    check(gpk_voxelize(s.handle(), &c, nullptr));
    const std::size_t voxels = vol.voxel_count();
    std::vector<float> out(voxels);
    check(gpk_download(s.handle(), GPK_BUF_VOLUME, out.data(), voxels * sizeof(float)));
    check(gpk_session_synchronize(s.handle()));
    vol.data.assign(out.begin(), out.end());
    return vol;
}

inline GaussianGradients voxelize_backward(const GaussianSet& set, const VoxelizerConfig& cfg,
                                           const VolumeGrid& dl_dv) {
    for (int d = 0; d < 3; ++d)
        if (dl_dv.dims[d] != cfg.dims[d])
            throw std::invalid_argument("voxelize_backward: gradient volume shape mismatch");  // voxelize.hpp:155-157
    Session& s = default_session();
    s.set_gaussians(set);
    const gpk_voxelizer_config c = detail::vcfg_of(cfg);
    const std::vector<float> dl(dl_dv.data.begin(), dl_dv.data.end());
    std::vector<float> g(set.size() * 11);
    check(gpk_voxelize_backward(s.handle(), &c, dl.data(), g.data()));
    return detail::grads_of(g, set.size());
}

// ---- optimize.hpp: adaptive density control, fit -------------------------------
namespace detail {

inline void adam_records(const AdamState& st, std::vector<float>& m, std::vector<float>& v) {
    const std::size_t n = st.size();
    m.assign(n * 11, 0.0f);
    v.assign(n * 11, 0.0f);
    for (std::size_t i = 0; i < n; ++i) {
        const double mm[11] = {st.m_mu[i].x, st.m_mu[i].y, st.m_mu[i].z, st.m_ls[i].x, st.m_ls[i].y, st.m_ls[i].z,
                               st.m_q[i].w, st.m_q[i].x, st.m_q[i].y, st.m_q[i].z, st.m_a[i]};
        const double vv[11] = {st.v_mu[i].x, st.v_mu[i].y, st.v_mu[i].z, st.v_ls[i].x, st.v_ls[i].y, st.v_ls[i].z,
                               st.v_q[i].w, st.v_q[i].x, st.v_q[i].y, st.v_q[i].z, st.v_a[i]};
        for (int k = 0; k < 11; ++k) {
            m[11 * i + k] = static_cast<float>(mm[k]);
            v[11 * i + k] = static_cast<float>(vv[k]);
        }
    }
}

inline void store_adam(const std::vector<float>& m, const std::vector<float>& v, AdamState& st) {
    const std::size_t n = m.size() / 11;
    st.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        const float* a = &m[11 * i];
        const float* b = &v[11 * i];
        st.m_mu[i] = {a[0], a[1], a[2]};
        st.m_ls[i] = {a[3], a[4], a[5]};
        st.m_q[i] = {a[6], a[7], a[8], a[9]};
        st.m_a[i] = a[10];
        st.v_mu[i] = {b[0], b[1], b[2]};
        st.v_ls[i] = {b[3], b[4], b[5]};
        st.v_q[i] = {b[6], b[7], b[8], b[9]};
        st.v_a[i] = b[10];
    }
}

// The resident set of `s` (any size) into `set`.
inline void fetch_set(gpk_session* s, GaussianSet& set) {
    uint64_t n = 0;
    check(gpk_gaussian_count(s, &n));
    std::vector<float> r(n * 11);
    if (n) check(gpk_get_gaussians(s, r.data()));
    set.primitives.resize(n);
    store_records(r, set);
}

}  // namespace detail

// densify_and_prune(set, adam, accum, cfg, rng) (optimize.hpp:255-344): the
// split normals come from the caller's own generator, in the reference's order.
inline DensifyReport densify_and_prune(GaussianSet& set, AdamState& adam, const DensifyAccum& accum,
                                       const FitConfig& cfg, Rng& rng) {
    const std::size_t n = set.size();
    if (adam.size() != n || accum.observations.size() != n)
        throw std::invalid_argument("densify_and_prune: size mismatch");
    Session& s = default_session();
    s.set_gaussians(set);
    std::vector<float> m, v;
    detail::adam_records(adam, m, v);
    check(gpk_set_adam_state(s.handle(), m.data(), v.data(), adam.step));
    check(gpk_densify_accum_enable(s.handle(), 1));
    std::vector<double> wsum(3 * n);
    for (std::size_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) wsum[3 * i + d] = accum.world_grad_sum[i][d];
    std::vector<int32_t> obs(accum.observations.begin(), accum.observations.end());
    check(gpk_set_densify_accum(s.handle(), accum.grad_norm_sum.data(), obs.data(), wsum.data()));
    const gpk_densify_config c{cfg.tau, cfg.grad_threshold, cfg.split_scale_fraction, cfg.split_scale_divisor,
                               cfg.scale_modifier};
    gpk_densify_report rep{};
    const int st = gpk_densify_and_prune_draw(
        s.handle(), &c, [](void* u) { return static_cast<Rng*>(u)->normal(); }, &rng, &rep);
    gpk_densify_accum_enable(s.handle(), 0);
    check(st);
    detail::fetch_set(s.handle(), set);
    int64_t step = 0;
    m.assign(set.size() * 11, 0.0f);
    v.assign(set.size() * 11, 0.0f);
    check(gpk_get_adam_state(s.handle(), m.data(), v.data(), &step));
    detail::store_adam(m, v, adam);
    adam.step = static_cast<long>(step);
    DensifyReport out;
    out.pruned = rep.pruned;
    out.cloned = rep.cloned;
    out.split = rep.split;
    return out;
}

// fit(volume, psf, cfg, progress) (optimize.hpp:360-424) on the device: the
// volume stays resident, the loop runs in the library (gpk_fit).
inline GaussianSet fit(const VolumeGrid& volume, const PsfSpec& psf, const FitConfig& cfg,
                       const ProgressSink& progress = nullptr) {
    volume.validate();
    psf.validate();
    cfg.validate();
    const std::vector<float> vol(volume.data.begin(), volume.data.end());
    gpk_fit_config c{};
    c.iterations = cfg.iterations;
    c.lr_position = cfg.lr_position;
    c.lr_opacity = cfg.lr_opacity;
    c.lr_scale = cfg.lr_scale;
    c.lr_rotation = cfg.lr_rotation;
    c.init_count = cfg.init_count;
    c.tau = cfg.tau;
    c.densify_start = cfg.densify_start;
    c.densify_end = cfg.densify_end;
    c.grad_threshold = cfg.grad_threshold;
    c.lambda = cfg.lambda;
    c.densify_interval = cfg.densify_interval;
    c.rng_seed = cfg.rng_seed;
    c.init_mode = cfg.init_mode == "grid" ? 1 : 0;
    c.scale_modifier = cfg.scale_modifier;
    c.split_scale_fraction = cfg.split_scale_fraction;
    c.split_scale_divisor = cfg.split_scale_divisor;
    c.dssim_scale = cfg.dssim_scale;
    c.progress_interval = cfg.progress_interval;
    c.tile_size = cfg.tile_size;
    c.footprint_sigmas = cfg.footprint_sigmas;
    struct Sink {
        const ProgressSink* fn;
        std::exception_ptr err;
    } sink{&progress, nullptr};
    auto tramp = [](const gpk_fit_progress* p, void* u) {
        Sink* k = static_cast<Sink*>(u);
        if (k->err) return;
        try {
            FitProgress fp;
            fp.iteration = p->iteration;
            fp.loss = p->loss;
            fp.count = p->count;
            fp.psnr2d = p->psnr2d;
            fp.monitor_loss = p->monitor_loss;
            (*k->fn)(fp);
        } catch (...) {
            k->err = std::current_exception();
        }
    };
    Session& s = default_session();
    const double spacing[3] = {volume.spacing.x, volume.spacing.y, volume.spacing.z};
    const double origin[3] = {volume.origin.x, volume.origin.y, volume.origin.z};
    const gpk_psf f = detail::psf_of(psf);
    const int st = gpk_fit(s.handle(), vol.data(), volume.dims, spacing, origin, &f, &c,
                           progress ? +tramp : nullptr, &sink);
    if (sink.err) std::rethrow_exception(sink.err);
    check(st);
    GaussianSet set;
    set.bbox = volume.world_bounds();
    detail::fetch_set(s.handle(), set);
    return set;
}

// ---- morton.hpp / quant.hpp (the codec's front half) -------------------------------
inline std::vector<std::size_t> morton_sort(const GaussianSet& set, int bits = 14) {
    Session& s = default_session();
    s.set_gaussians(set);
    std::vector<uint64_t> p(set.size());
    check(gpk_morton_sort(s.handle(), bits, p.data()));
    return std::vector<std::size_t>(p.begin(), p.end());
}

inline QuantizedSet quantize(const GaussianSet& set, const QuantSpec& spec) {
    spec.validate();
    Session& s = default_session();
    s.set_gaussians(set);
    const gpk_quant_spec c{spec.pos_bits, spec.opacity_bits, spec.scale_bits, spec.quat_bits, spec.morton_bits};
    QuantizedSet q;
    q.spec = spec;
    q.bbox = set.bbox;
    const std::size_t n = set.size();
    q.positions.resize(3 * n);
    q.opacities.resize(n);
    q.log_scales.resize(3 * n);
    q.quats.resize(4 * n);
    double lo[3], hi[3];
    check(gpk_quantize(s.handle(), &c, 0, q.positions.data(), q.opacities.data(), q.log_scales.data(),
                       q.quats.data(), lo, hi));
    q.scale_min = {lo[0], lo[1], lo[2]};
    q.scale_max = {hi[0], hi[1], hi[2]};
    return q;
}

// ---- checkpoint.hpp ----------------------------------------------------------------
inline void save_checkpoint(const GaussianSet& set, const std::string& path) {
    Session& s = default_session();
    s.set_gaussians(set);
    check(gpk_save_checkpoint(s.handle(), path.c_str()));
}

inline GaussianSet load_checkpoint(const std::string& path) {
    Session& s = default_session();
    check(gpk_load_checkpoint(s.handle(), path.c_str()));
    GaussianSet set;
    gpk_bounds b;
    check(gpk_get_bounds(s.handle(), &b));
    set.bbox = {{b.min[0], b.min[1], b.min[2]}, {b.max[0], b.max[1], b.max[2]}};
    detail::fetch_set(s.handle(), set);
    return set;
}

}  // namespace b200
}  // namespace gpile
