// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A flat extern "C" surface over the UNMODIFIED reference headers
// (/root/reference/proj/include/gpile), compiled by oracle/Makefile into
// oracle/_ref/libgpile_ref.so. It is the ground truth the C restatement
// (oracle/gpile_oracle.c) is pinned against, the generator of the golden
// fixtures under tests/golden/, and the CPU arm of bench.py (--impl reference
// and the cpu_baseline leg). Nothing in the product path
// (paper_2603_20611_b200/) may load it.
//
// Only the hot-path headers are included (render, backward, loss, metrics,
// optimize, voxelize); gpile.hpp / container.hpp are not, because they need
// <lzma.h> which this image lacks.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpile/backward.hpp"
#include "gpile/checkpoint.hpp"
#include "gpile/container.hpp"  // pack_deltas only (oracle/stub/lzma.h)
#include "gpile/morton.hpp"
#include "gpile/quant.hpp"
#include "gpile/core.hpp"
#include "gpile/errors.hpp"
#include "gpile/loss.hpp"
#include "gpile/metrics.hpp"
#include "gpile/optimize.hpp"
#include "gpile/parallel.hpp"
#include "gpile/render.hpp"
#include "gpile/rng.hpp"
#include "gpile/voxelize.hpp"

#include "../include/gpile_b200.h"  // flat struct layouts only

using namespace gpile;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_err.clear();
        return GPK_OK;
    } catch (const DegenerateCovariance& e) {
        g_err = e.what();
        return GPK_ERR_DEGENERATE_COVARIANCE;
    } catch (const NumericFailure& e) {
        g_err = e.what();
        return GPK_ERR_NUMERIC_FAILURE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return GPK_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

GaussianPrimitive prim_from(const double* r) {
    GaussianPrimitive g;
    g.mu = {r[0], r[1], r[2]};
    g.log_scale = {r[3], r[4], r[5]};
    g.quat = {r[6], r[7], r[8], r[9]};
    g.alpha_raw = r[10];
    return g;
}

void prim_to(const GaussianPrimitive& g, double* r) {
    r[0] = g.mu.x; r[1] = g.mu.y; r[2] = g.mu.z;
    r[3] = g.log_scale.x; r[4] = g.log_scale.y; r[5] = g.log_scale.z;
    r[6] = g.quat.w; r[7] = g.quat.x; r[8] = g.quat.y; r[9] = g.quat.z;
    r[10] = g.alpha_raw;
}

Bounds bounds_from(const gpk_bounds* b) {
    Bounds o;
    o.min = {b->min[0], b->min[1], b->min[2]};
    o.max = {b->max[0], b->max[1], b->max[2]};
    return o;
}

SlicePose pose_from(const gpk_slice_pose* p) {
    SlicePose o;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.rotation.m[i][j] = p->rotation[3 * i + j];
    o.translation = {p->translation[0], p->translation[1], p->translation[2]};
    o.width = p->width;
    o.height = p->height;
    o.pixel_spacing = {p->pixel_spacing[0], p->pixel_spacing[1]};
    o.principal_point = {p->principal_point[0], p->principal_point[1]};
    return o;
}

void pose_to(const SlicePose& p, gpk_slice_pose* o) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o->rotation[3 * i + j] = p.rotation.m[i][j];
    o->translation[0] = p.translation.x;
    o->translation[1] = p.translation.y;
    o->translation[2] = p.translation.z;
    o->width = p.width;
    o->height = p.height;
    o->pixel_spacing[0] = p.pixel_spacing.x;
    o->pixel_spacing[1] = p.pixel_spacing.y;
    o->principal_point[0] = p.principal_point.x;
    o->principal_point[1] = p.principal_point.y;
}

PsfSpec psf_from(const gpk_psf* p) {
    PsfSpec o;
    o.sigma_x = p->sigma_x;
    o.sigma_y = p->sigma_y;
    o.sigma_z = p->sigma_z;
    return o;
}

RasterConfig cfg_from(const gpk_raster_config* c) {
    RasterConfig o;
    o.tau = c->tau;
    o.tile_size = c->tile_size;
    o.footprint_sigmas = c->footprint_sigmas;
    o.scale_modifier = c->scale_modifier;
    return o;
}

VoxelizerConfig vcfg_from(const gpk_voxelizer_config* c) {
    VoxelizerConfig o;
    for (int d = 0; d < 3; ++d) {
        o.dims[d] = c->dims[d];
        o.tile_dims[d] = c->tile_dims[d];
    }
    o.spacing = {c->spacing[0], c->spacing[1], c->spacing[2]};
    o.origin = {c->origin[0], c->origin[1], c->origin[2]};
    o.support_sigmas = c->support_sigmas;
    o.scale_modifier = c->scale_modifier;
    return o;
}

void grads_to(const GaussianGradients& g, double* out) {
    for (std::size_t i = 0; i < g.size(); ++i) {
        double* r = out + 11 * i;
        r[0] = g.d_mu[i].x; r[1] = g.d_mu[i].y; r[2] = g.d_mu[i].z;
        r[3] = g.d_log_scale[i].x; r[4] = g.d_log_scale[i].y; r[5] = g.d_log_scale[i].z;
        r[6] = g.d_quat[i].w; r[7] = g.d_quat[i].x; r[8] = g.d_quat[i].y; r[9] = g.d_quat[i].z;
        r[10] = g.d_alpha_raw[i];
    }
}

GaussianGradients grads_from(std::size_t n, const double* in) {
    GaussianGradients g(n);
    for (std::size_t i = 0; i < n; ++i) {
        const double* r = in + 11 * i;
        g.d_mu[i] = {r[0], r[1], r[2]};
        g.d_log_scale[i] = {r[3], r[4], r[5]};
        g.d_quat[i] = {r[6], r[7], r[8], r[9]};
        g.d_alpha_raw[i] = r[10];
    }
    return g;
}

SliceImage image_from(int w, int h, const double* px) {
    SliceImage img(w, h);
    std::memcpy(img.pixels.data(), px, sizeof(double) * img.pixels.size());
    return img;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* gref_last_error(void) { return g_err.c_str(); }
void gref_set_threads(int n) { worker_cap() = n; }
int gref_effective_workers(void) { return effective_workers(); }

// ---- RNG (rng.hpp) --------------------------------------------------------
void* gref_rng_new(uint64_t seed) { return new Rng(seed); }
void gref_rng_free(void* r) { delete static_cast<Rng*>(r); }
double gref_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
double gref_rng_uniform_range(void* r, double lo, double hi) {
    return static_cast<Rng*>(r)->uniform(lo, hi);
}
double gref_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
uint64_t gref_rng_below(void* r, uint64_t n) { return static_cast<Rng*>(r)->below(n); }
void gref_rng_unit_quaternion(void* r, double* out4) {
    const Vec4 q = static_cast<Rng*>(r)->unit_quaternion();
    out4[0] = q.w; out4[1] = q.x; out4[2] = q.y; out4[3] = q.z;
}

// test_util.hpp:10-18 (random_primitive), restated on the reference Rng so
// fixtures draw the identical stream.
void gref_random_primitive(void* r, const gpk_bounds* b, double lo, double hi, double* out11) {
    Rng& rng = *static_cast<Rng*>(r);
    GaussianPrimitive g;
    g.mu = rng.uniform_in_box({b->min[0], b->min[1], b->min[2]}, {b->max[0], b->max[1], b->max[2]});
    for (int d = 0; d < 3; ++d) g.log_scale[d] = std::log(rng.uniform(lo, hi));
    g.quat = rng.unit_quaternion();
    g.alpha_raw = alpha_activation_inverse(rng.uniform(0.2, 0.9));
    prim_to(g, out11);
}

// test_util.hpp:27-36 (random_pose)
void gref_random_pose(void* r, int w, int h, gpk_slice_pose* out) {
    Rng& rng = *static_cast<Rng*>(r);
    SlicePose pose;
    pose.rotation = quat_to_rotation(rng.unit_quaternion());
    pose.translation = {rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0)};
    pose.width = w;
    pose.height = h;
    pose.pixel_spacing = {1.0, 1.0};
    pose.principal_point = {w / 2.0, h / 2.0};
    pose_to(pose, out);
}

double gref_alpha_activation_inverse(double a) { return alpha_activation_inverse(a); }

int gref_init_random(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                     double* out) {
    return guarded([&] {
        const GaussianSet set = init_random(n, bounds_from(bbox), scale_base, seed);
        for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out + 11 * i);
    });
}

int gref_init_grid(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                   double* out) {
    return guarded([&] {
        const GaussianSet set = init_grid(n, bounds_from(bbox), scale_base, seed);
        for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out + 11 * i);
    });
}

uint64_t gref_default_init_count(uint64_t voxels) { return default_init_count(voxels); }

int gref_slice_pose_for_index(const int32_t dims[3], const double spacing[3],
                              const double origin[3], int k, gpk_slice_pose* out) {
    return guarded([&] {
        VolumeGrid vol;
        for (int d = 0; d < 3; ++d) vol.dims[d] = dims[d];
        vol.spacing = {spacing[0], spacing[1], spacing[2]};
        vol.origin = {origin[0], origin[1], origin[2]};
        pose_to(slice_pose_for_index(vol, k), out);
    });
}

// ---- GaussianSet handle ------------------------------------------------------
void* gref_set_new(uint64_t n, const double* records, const gpk_bounds* bbox) {
    auto* set = new GaussianSet;
    set->bbox = bounds_from(bbox);
    set->primitives.resize(n);
    for (std::size_t i = 0; i < n; ++i) set->primitives[i] = prim_from(records + 11 * i);
    return set;
}
void gref_set_free(void* s) { delete static_cast<GaussianSet*>(s); }
void gref_set_get(void* s, double* out) {
    const auto& set = *static_cast<GaussianSet*>(s);
    for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out + 11 * i);
}

// prepare_gaussians (render.hpp:83). fields: 19 doubles per survivor =
// alpha, opacity_r, alpha_tilde, mu_c(3), mu_e(3), mu_2d(2), cov2d(a,b,d),
// conic(a,b,d), det2, sigma_e_zz.
int gref_prepare(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                 const gpk_raster_config* cfg, uint64_t* count, uint32_t* index,
                 int32_t* bounds, double* fields) {
    return guarded([&] {
        psf_from(psf).validate();
        const auto prep = prepare_gaussians(*static_cast<GaussianSet*>(s), pose_from(pose),
                                            psf_from(psf), cfg_from(cfg));
        *count = prep.size();
        for (std::size_t k = 0; k < prep.size(); ++k) {
            const PreparedGaussian& p = prep[k];
            if (index) index[k] = p.index;
            if (bounds) {
                bounds[4 * k + 0] = p.lo_x;
                bounds[4 * k + 1] = p.hi_x;
                bounds[4 * k + 2] = p.lo_y;
                bounds[4 * k + 3] = p.hi_y;
            }
            if (fields) {
                double* f = fields + 19 * k;
                f[0] = p.alpha; f[1] = p.opacity_r; f[2] = p.alpha_tilde;
                f[3] = p.mu_c.x; f[4] = p.mu_c.y; f[5] = p.mu_c.z;
                f[6] = p.mu_e.x; f[7] = p.mu_e.y; f[8] = p.mu_e.z;
                f[9] = p.mu_2d.x; f[10] = p.mu_2d.y;
                f[11] = p.cov2d.a; f[12] = p.cov2d.b; f[13] = p.cov2d.d;
                f[14] = p.conic.a; f[15] = p.conic.b; f[16] = p.conic.d;
                f[17] = p.det2; f[18] = p.sigma_e.m[2][2];
            }
        }
    });
}

// prepare_gaussians (render.hpp:83), every PreparedGaussian field (:68-79):
// 47 doubles per survivor in gpk_get_prepared_fields' layout (alpha,
// opacity_r, alpha_tilde, mu_c, mu_e, sigma_c, sigma_c_inv, sigma_e, mu_2d,
// cov2d a b c d, conic a b c d, det2).
int gref_prepare_full(void* s, const gpk_slice_pose* pose, const gpk_psf* psf, const gpk_raster_config* cfg,
                      uint64_t* count, double* fields, uint64_t capacity) {
    return guarded([&] {
        psf_from(psf).validate();
        const auto prep = prepare_gaussians(*static_cast<GaussianSet*>(s), pose_from(pose), psf_from(psf),
                                            cfg_from(cfg));
        *count = prep.size();
        for (std::size_t k = 0; k < prep.size() && k < capacity; ++k) {
            const PreparedGaussian& p = prep[k];
            double* f = fields + 47 * k;
            f[0] = p.alpha; f[1] = p.opacity_r; f[2] = p.alpha_tilde;
            f[3] = p.mu_c.x; f[4] = p.mu_c.y; f[5] = p.mu_c.z;
            f[6] = p.mu_e.x; f[7] = p.mu_e.y; f[8] = p.mu_e.z;
            for (int i = 0; i < 9; ++i) {
                f[9 + i] = p.sigma_c.m[i / 3][i % 3];
                f[18 + i] = p.sigma_c_inv.m[i / 3][i % 3];
                f[27 + i] = p.sigma_e.m[i / 3][i % 3];
            }
            f[36] = p.mu_2d.x; f[37] = p.mu_2d.y;
            f[38] = p.cov2d.a; f[39] = p.cov2d.b; f[40] = p.cov2d.c; f[41] = p.cov2d.d;
            f[42] = p.conic.a; f[43] = p.conic.b; f[44] = p.conic.c; f[45] = p.conic.d;
            f[46] = p.det2;
        }
    });
}

// detail::TileGrid (render.hpp:142-160), entries translated to set indices.
int gref_tile_lists(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                    const gpk_raster_config* cfg, uint32_t* offsets, uint32_t* entries,
                    uint64_t capacity, uint64_t* total, uint64_t* tiles) {
    return guarded([&] {
        const SlicePose sp = pose_from(pose);
        const auto prep =
            prepare_gaussians(*static_cast<GaussianSet*>(s), sp, psf_from(psf), cfg_from(cfg));
        const detail::TileGrid grid(sp, prep, cfg->tile_size);
        *tiles = grid.lists.size();
        std::size_t pos = 0;
        for (std::size_t t = 0; t < grid.lists.size(); ++t) {
            if (offsets) offsets[t] = static_cast<uint32_t>(pos);
            for (uint32_t pi : grid.lists[t]) {
                if (entries && pos < capacity) entries[pos] = prep[pi].index;
                ++pos;
            }
        }
        if (offsets) offsets[grid.lists.size()] = static_cast<uint32_t>(pos);
        *total = pos;
    });
}

int gref_rasterize(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                   const gpk_raster_config* cfg, double* image) {
    return guarded([&] {
        const SliceImage img =
            rasterize_slice(*static_cast<GaussianSet*>(s), pose_from(pose), psf_from(psf),
                            cfg_from(cfg));
        std::memcpy(image, img.pixels.data(), sizeof(double) * img.pixels.size());
    });
}

int gref_rasterize_naive(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                         const gpk_raster_config* cfg, double* image) {
    return guarded([&] {
        const SliceImage img =
            rasterize_naive(*static_cast<GaussianSet*>(s), pose_from(pose), psf_from(psf),
                            cfg_from(cfg));
        std::memcpy(image, img.pixels.data(), sizeof(double) * img.pixels.size());
    });
}

// backward_slice (backward.hpp:189). grads: n*11 record order. Stats optional.
int gref_backward(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                  const gpk_raster_config* cfg, const double* dl_di, double* grads,
                  double* stat_norm, uint8_t* stat_observed, double* stat_world) {
    return guarded([&] {
        const SlicePose sp = pose_from(pose);
        const SliceImage g = image_from(sp.width, sp.height, dl_di);
        ScreenGradStats stats;
        const GaussianGradients out = backward_slice(*static_cast<GaussianSet*>(s), sp,
                                                     psf_from(psf), g, cfg_from(cfg), &stats);
        grads_to(out, grads);
        for (std::size_t i = 0; i < out.size(); ++i) {
            if (stat_norm) stat_norm[i] = stats.mu2d_grad_norm[i];
            if (stat_observed) stat_observed[i] = stats.observed[i];
            if (stat_world) {
                stat_world[3 * i + 0] = stats.world_pos_grad[i].x;
                stat_world[3 * i + 1] = stats.world_pos_grad[i].y;
                stat_world[3 * i + 2] = stats.world_pos_grad[i].z;
            }
        }
    });
}

// Backward with a mismatched dL/dI shape (error-path pin, backward.hpp:102-103).
int gref_backward_shape(void* s, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, int w, int h, const double* dl_di,
                        double* grads) {
    return guarded([&] {
        const SliceImage g = image_from(w, h, dl_di);
        const GaussianGradients out = backward_slice(*static_cast<GaussianSet*>(s),
                                                     pose_from(pose), psf_from(psf), g,
                                                     cfg_from(cfg));
        grads_to(out, grads);
    });
}

// photometric_loss (loss.hpp:13).
int gref_loss(int w, int h, const double* rendered, const double* target, double lambda,
              double dssim_scale, double* dl_di, double* loss) {
    return guarded([&] {
        SliceImage d;
        *loss = photometric_loss(image_from(w, h, rendered), image_from(w, h, target), lambda,
                                 d, dssim_scale);
        std::memcpy(dl_di, d.pixels.data(), sizeof(double) * d.pixels.size());
    });
}

// ssim_with_gradient (metrics.hpp:187), 2-D.
int gref_ssim_grad(int w, int h, const double* x, const double* y, double* grad, double* ssim) {
    return guarded([&] {
        const int dims[3] = {w, h, 1};
        std::vector<double> vx(x, x + static_cast<std::size_t>(w) * h);
        std::vector<double> vy(y, y + static_cast<std::size_t>(w) * h);
        std::vector<double> g;
        *ssim = ssim_with_gradient(vx, vy, dims, 2, g);
        std::memcpy(grad, g.data(), sizeof(double) * g.size());
    });
}

double gref_lr_at(double lr0, int it, int total) { return lr_at(lr0, it, total); }

// adam_step (optimize.hpp:195). m, v: n*11 record order; updated in place with
// the set; *step in/out.
int gref_adam_step(void* s, const double* grads, double* m, double* v, int64_t* step,
                   const gpk_learning_rates* lrs, const gpk_adam_hparams* hp) {
    return guarded([&] {
        GaussianSet& set = *static_cast<GaussianSet*>(s);
        const std::size_t n = set.size();
        AdamState st(n);
        if (hp) {
            st.beta1 = hp->beta1;
            st.beta2 = hp->beta2;
            st.eps = hp->eps;
        }
        st.step = static_cast<long>(*step);
        for (std::size_t i = 0; i < n; ++i) {
            const double* mi = m + 11 * i;
            const double* vi = v + 11 * i;
            st.m_mu[i] = {mi[0], mi[1], mi[2]};
            st.v_mu[i] = {vi[0], vi[1], vi[2]};
            st.m_ls[i] = {mi[3], mi[4], mi[5]};
            st.v_ls[i] = {vi[3], vi[4], vi[5]};
            st.m_q[i] = {mi[6], mi[7], mi[8], mi[9]};
            st.v_q[i] = {vi[6], vi[7], vi[8], vi[9]};
            st.m_a[i] = mi[10];
            st.v_a[i] = vi[10];
        }
        adam_step(set, grads_from(n, grads), st,
                  LearningRates{lrs->position, lrs->opacity, lrs->scale, lrs->rotation});
        *step = st.step;
        for (std::size_t i = 0; i < n; ++i) {
            double* mi = m + 11 * i;
            double* vi = v + 11 * i;
            for (int d = 0; d < 3; ++d) {
                mi[d] = st.m_mu[i][d];
                vi[d] = st.v_mu[i][d];
                mi[3 + d] = st.m_ls[i][d];
                vi[3 + d] = st.v_ls[i][d];
            }
            for (int d = 0; d < 4; ++d) {
                mi[6 + d] = st.m_q[i][d];
                vi[6 + d] = st.v_q[i][d];
            }
            mi[10] = st.m_a[i];
            vi[10] = st.v_a[i];
        }
    });
}

// voxelize (voxelize.hpp:113).
int gref_voxelize(void* s, const gpk_voxelizer_config* cfg, double* out) {
    return guarded([&] {
        const VolumeGrid vol = voxelize(*static_cast<GaussianSet*>(s), vcfg_from(cfg));
        std::memcpy(out, vol.data.data(), sizeof(double) * vol.data.size());
    });
}

// detail::VoxelTiles (voxelize.hpp:86-105), entries translated to set indices.
int gref_voxel_tiles(void* s, const gpk_voxelizer_config* cfg, uint32_t* offsets,
                     uint32_t* entries, uint64_t capacity, uint64_t* total, uint64_t* tiles) {
    return guarded([&] {
        const VoxelizerConfig vc = vcfg_from(cfg);
        vc.validate();
        const auto prims = detail::prepare_voxel_prims(*static_cast<GaussianSet*>(s), vc);
        const detail::VoxelTiles vt(vc, prims);
        *tiles = vt.lists.size();
        std::size_t pos = 0;
        for (std::size_t t = 0; t < vt.lists.size(); ++t) {
            if (offsets) offsets[t] = static_cast<uint32_t>(pos);
            for (uint32_t pi : vt.lists[t]) {
                if (entries && pos < capacity) entries[pos] = prims[pi].index;
                ++pos;
            }
        }
        if (offsets) offsets[vt.lists.size()] = static_cast<uint32_t>(pos);
        *total = pos;
    });
}

// voxelize_backward (voxelize.hpp:152).
int gref_voxelize_backward(void* s, const gpk_voxelizer_config* cfg, const double* dl_dv,
                           double* grads) {
    return guarded([&] {
        VolumeGrid g;
        for (int d = 0; d < 3; ++d) g.dims[d] = cfg->dims[d];
        g.data.assign(dl_dv, dl_dv + g.voxel_count());
        const GaussianGradients out =
            voxelize_backward(*static_cast<GaussianSet*>(s), vcfg_from(cfg), g);
        grads_to(out, grads);
    });
}

// render_oracle (render.hpp:251): quadrature ground truth for one primitive.
double gref_render_oracle(void* s, uint64_t i, const gpk_slice_pose* pose, const gpk_psf* psf,
                          double px, double py, double mod) {
    double v = 0.0;
    const int st = guarded([&] {
        v = render_oracle(static_cast<GaussianSet*>(s)->primitives[i], pose_from(pose),
                          psf_from(psf), Vec2{px, py}, mod);
    });
    return st == GPK_OK ? v : std::nan("");
}

// ---- CPU timing of the reference units ----------------------
// U1 = prepare_gaussians + rasterize_prepared + backward_prepared, exactly as
// fit() calls them (optimize.hpp:386-395). seconds[3] = per-stage sums over
// `reps` slices (poses cycle through `npose` entries).
int gref_time_u1(void* s, const gpk_slice_pose* poses, int npose, const gpk_psf* psf,
                 const gpk_raster_config* cfg, const double* dl_di, int reps,
                 double* seconds) {
    return guarded([&] {
        GaussianSet& set = *static_cast<GaussianSet*>(s);
        const RasterConfig rc = cfg_from(cfg);
        const PsfSpec ps = psf_from(psf);
        seconds[0] = seconds[1] = seconds[2] = 0.0;
        for (int r = 0; r < reps; ++r) {
            const SlicePose sp = pose_from(&poses[r % npose]);
            const SliceImage g = image_from(sp.width, sp.height, dl_di);
            auto t0 = std::chrono::steady_clock::now();
            const auto prep = prepare_gaussians(set, sp, ps, rc);
            seconds[0] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            const SliceImage img = rasterize_prepared(prep, sp, rc);
            seconds[1] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            ScreenGradStats stats;
            const GaussianGradients grads = backward_prepared(set, prep, sp, g, rc, &stats);
            seconds[2] += seconds_since(t0);
            if (img.pixels.empty() || grads.size() != set.size())
                throw std::runtime_error("gref_time_u1: empty result");
        }
    });
}

// U2 = U1 + photometric_loss + adam_step (optimize.hpp:385-402). seconds[5]:
// prepare, raster, loss, backward, adam.
int gref_time_u2(void* s, const gpk_slice_pose* poses, int npose, const gpk_psf* psf,
                 const gpk_raster_config* cfg, const double* target, double lambda,
                 int reps, double* seconds) {
    return guarded([&] {
        GaussianSet& set = *static_cast<GaussianSet*>(s);
        const RasterConfig rc = cfg_from(cfg);
        const PsfSpec ps = psf_from(psf);
        AdamState adam(set.size());
        for (int k = 0; k < 5; ++k) seconds[k] = 0.0;
        for (int r = 0; r < reps; ++r) {
            const SlicePose sp = pose_from(&poses[r % npose]);
            const SliceImage tgt = image_from(sp.width, sp.height, target);
            auto t0 = std::chrono::steady_clock::now();
            const auto prep = prepare_gaussians(set, sp, ps, rc);
            seconds[0] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            const SliceImage img = rasterize_prepared(prep, sp, rc);
            seconds[1] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            SliceImage dl_di;
            photometric_loss(img, tgt, lambda, dl_di, 0.5);
            seconds[2] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            ScreenGradStats stats;
            const GaussianGradients grads = backward_prepared(set, prep, sp, dl_di, rc, &stats);
            seconds[3] += seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            adam_step(set, grads, adam, LearningRates{6e-4, 0.02, 2e-3, 1e-3});
            seconds[4] += seconds_since(t0);
        }
    });
}

// Voxelizer wall time (C4).
int gref_time_voxelize(void* s, const gpk_voxelizer_config* cfg, int reps, double* seconds) {
    return guarded([&] {
        *seconds = 0.0;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const VolumeGrid vol = voxelize(*static_cast<GaussianSet*>(s), vcfg_from(cfg));
            *seconds += seconds_since(t0);
            if (vol.data.empty()) throw std::runtime_error("empty volume");
        }
    });
}


// ---- adaptive density control + fit (optimize.hpp:228-424) -------------------
// densify_and_prune on (set, Adam moments n x 11, accum) with the caller's
// generator; the new set (capacity 2n suffices: a primitive yields at most
// two) replaces records/m/v (out_n).
int gref_densify_and_prune(void* s, double* m, double* v, int64_t step, const double* grad_norm_sum,
                           const int32_t* observations, const double* world_grad_sum,
                           const gpk_densify_config* cfg, void* rng, double* out_rec, double* out_m,
                           double* out_v, uint64_t* out_n, uint64_t* report3) {
    return guarded([&] {
        GaussianSet& set = *static_cast<GaussianSet*>(s);
        const std::size_t n = set.size();
        AdamState st(n);
        st.step = static_cast<long>(step);
        for (std::size_t i = 0; i < n; ++i) {
            const double* mi = m + 11 * i;
            const double* vi = v + 11 * i;
            st.m_mu[i] = {mi[0], mi[1], mi[2]};
            st.v_mu[i] = {vi[0], vi[1], vi[2]};
            st.m_ls[i] = {mi[3], mi[4], mi[5]};
            st.v_ls[i] = {vi[3], vi[4], vi[5]};
            st.m_q[i] = {mi[6], mi[7], mi[8], mi[9]};
            st.v_q[i] = {vi[6], vi[7], vi[8], vi[9]};
            st.m_a[i] = mi[10];
            st.v_a[i] = vi[10];
        }
        DensifyAccum acc(n);
        for (std::size_t i = 0; i < n; ++i) {
            acc.grad_norm_sum[i] = grad_norm_sum[i];
            acc.observations[i] = observations[i];
            acc.world_grad_sum[i] = {world_grad_sum[3 * i], world_grad_sum[3 * i + 1], world_grad_sum[3 * i + 2]};
        }
        FitConfig fc;
        fc.tau = cfg->tau;
        fc.grad_threshold = cfg->grad_threshold;
        fc.split_scale_fraction = cfg->split_scale_fraction;
        fc.split_scale_divisor = cfg->split_scale_divisor;
        fc.scale_modifier = cfg->scale_modifier;
        const DensifyReport rep = densify_and_prune(set, st, acc, fc, *static_cast<Rng*>(rng));
        *out_n = set.size();
        for (std::size_t i = 0; i < set.size(); ++i) {
            prim_to(set.primitives[i], out_rec + 11 * i);
            double* mi = out_m + 11 * i;
            double* vi = out_v + 11 * i;
            for (int d = 0; d < 3; ++d) {
                mi[d] = st.m_mu[i][d];
                vi[d] = st.v_mu[i][d];
                mi[3 + d] = st.m_ls[i][d];
                vi[3 + d] = st.v_ls[i][d];
            }
            for (int d = 0; d < 4; ++d) {
                mi[6 + d] = st.m_q[i][d];
                vi[6 + d] = st.v_q[i][d];
            }
            mi[10] = st.m_a[i];
            vi[10] = st.v_a[i];
        }
        report3[0] = rep.pruned;
        report3[1] = rep.cloned;
        report3[2] = rep.split;
    });
}

// fit (optimize.hpp:360-424) on a z-major f64 volume; the fitted set goes to
// out_rec (capacity records) and each FitProgress to progress (5 doubles:
// iteration, loss, count, psnr2d, monitor_loss; up to max_progress).
int gref_fit(const double* volume, const int32_t dims[3], const double spacing[3], const double origin[3],
             const gpk_psf* psf, const gpk_fit_config* c, double* out_rec, uint64_t capacity, uint64_t* out_n,
             double* progress, uint64_t max_progress, uint64_t* n_progress) {
    return guarded([&] {
        VolumeGrid vol;
        for (int d = 0; d < 3; ++d) vol.dims[d] = dims[d];
        vol.spacing = {spacing[0], spacing[1], spacing[2]};
        vol.origin = {origin[0], origin[1], origin[2]};
        vol.data.assign(volume, volume + (std::size_t)dims[0] * dims[1] * dims[2]);
        FitConfig fc;
        fc.iterations = c->iterations;
        fc.lr_position = c->lr_position;
        fc.lr_opacity = c->lr_opacity;
        fc.lr_scale = c->lr_scale;
        fc.lr_rotation = c->lr_rotation;
        fc.init_count = c->init_count;
        fc.tau = c->tau;
        fc.densify_start = c->densify_start;
        fc.densify_end = c->densify_end;
        fc.grad_threshold = c->grad_threshold;
        fc.lambda = c->lambda;
        fc.densify_interval = c->densify_interval;
        fc.rng_seed = c->rng_seed;
        fc.init_mode = c->init_mode == 1 ? "grid" : "random";
        fc.scale_modifier = c->scale_modifier;
        fc.split_scale_fraction = c->split_scale_fraction;
        fc.split_scale_divisor = c->split_scale_divisor;
        fc.dssim_scale = c->dssim_scale;
        fc.progress_interval = c->progress_interval;
        fc.tile_size = c->tile_size;
        fc.footprint_sigmas = c->footprint_sigmas;
        *n_progress = 0;
        const GaussianSet set = fit(vol, psf_from(psf), fc, [&](const FitProgress& p) {
            if (*n_progress < max_progress) {
                double* o = progress + 5 * (*n_progress);
                o[0] = p.iteration;
                o[1] = p.loss;
                o[2] = (double)p.count;
                o[3] = p.psnr2d;
                o[4] = p.monitor_loss;
            }
            ++*n_progress;
        });
        *out_n = set.size();
        if (set.size() > capacity) throw std::invalid_argument("gref_fit: output capacity");
        for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out_rec + 11 * i);
    });
}


// ---- checkpoints (checkpoint.hpp:38-97) --------------------------------------
int gref_save_checkpoint(void* s, const char* path) {
    return guarded([&] { save_checkpoint(*static_cast<GaussianSet*>(s), path); });
}
// load_checkpoint -> records (capacity) + bbox; status 8 CorruptContainer, 9 LoadError
int gref_load_checkpoint(const char* path, double* out, uint64_t capacity, uint64_t* n, gpk_bounds* bbox) {
    try {
        const GaussianSet set = load_checkpoint(path);
        *n = set.size();
        if (set.size() > capacity) throw std::invalid_argument("capacity");
        for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out + 11 * i);
        for (int d = 0; d < 3; ++d) {
            bbox->min[d] = set.bbox.min[d];
            bbox->max[d] = set.bbox.max[d];
        }
        g_err.clear();
        return GPK_OK;
    } catch (const CorruptContainer& e) {
        g_err = e.what();
        return GPK_ERR_CORRUPT_CONTAINER;
    } catch (const LoadError& e) {
        g_err = e.what();
        return GPK_ERR_LOAD;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GPK_ERR_INVALID_ARGUMENT;
    }
}
uint64_t gref_checkpoint_bytes(uint64_t count) { return checkpoint_bytes(count); }


// ---- codec front half (morton.hpp:33-48, quant.hpp:67-132, container.hpp:136-156)
int gref_morton_sort(void* s, int bits, uint64_t* perm) {
    return guarded([&] {
        const auto p = morton_sort(*static_cast<GaussianSet*>(s), bits);
        for (std::size_t k = 0; k < p.size(); ++k) perm[k] = p[k];
    });
}

// quantize of the set (in morton order when morton_order: encode's order)
int gref_quantize(void* s, const gpk_quant_spec* spec, int morton_order, uint32_t* pos, uint32_t* opa,
                  uint32_t* ls, uint32_t* quat, double* smin, double* smax) {
    return guarded([&] {
        QuantSpec q;
        q.pos_bits = spec->pos_bits;
        q.opacity_bits = spec->opacity_bits;
        q.scale_bits = spec->scale_bits;
        q.quat_bits = spec->quat_bits;
        q.morton_bits = spec->morton_bits;
        const GaussianSet& set = *static_cast<GaussianSet*>(s);
        const QuantizedSet qs = morton_order ? quantize(apply_permutation(set, morton_sort(set, q.morton_bits)), q)
                                             : quantize(set, q);
        std::copy(qs.positions.begin(), qs.positions.end(), pos);
        std::copy(qs.opacities.begin(), qs.opacities.end(), opa);
        std::copy(qs.log_scales.begin(), qs.log_scales.end(), ls);
        std::copy(qs.quats.begin(), qs.quats.end(), quat);
        for (int d = 0; d < 3; ++d) {
            smin[d] = qs.scale_min[d];
            smax[d] = qs.scale_max[d];
        }
    });
}

int gref_pack_deltas(const uint32_t* values, uint64_t total, int components, int bits, uint8_t* out) {
    return guarded([&] {
        const std::vector<std::uint32_t> v(values, values + total);
        const auto b = detail::pack_deltas(v, components, bits);
        std::copy(b.begin(), b.end(), out);
    });
}

int gref_unpack_deltas(const uint8_t* bytes, uint64_t nbytes, uint64_t count, int components, int bits,
                       uint32_t* out) {
    return guarded([&] {
        const std::vector<std::uint8_t> b(bytes, bytes + nbytes);
        const auto v = detail::unpack_deltas(b, count, components, bits, "test");
        std::copy(v.begin(), v.end(), out);
    });
}


// dequantize (quant.hpp:134-176) of u32 streams -> n x 11 f64 records
int gref_dequantize(const gpk_quant_spec* spec, uint64_t n, const gpk_bounds* bbox, const double* smin,
                    const double* smax, const uint32_t* pos, const uint32_t* opa, const uint32_t* ls,
                    const uint32_t* quat, double* out) {
    return guarded([&] {
        QuantizedSet q;
        q.spec.pos_bits = spec->pos_bits;
        q.spec.opacity_bits = spec->opacity_bits;
        q.spec.scale_bits = spec->scale_bits;
        q.spec.quat_bits = spec->quat_bits;
        q.spec.morton_bits = spec->morton_bits;
        q.bbox = bounds_from(bbox);
        q.scale_min = {smin[0], smin[1], smin[2]};
        q.scale_max = {smax[0], smax[1], smax[2]};
        q.positions.assign(pos, pos + 3 * n);
        q.opacities.assign(opa, opa + n);
        q.log_scales.assign(ls, ls + 3 * n);
        q.quats.assign(quat, quat + 4 * n);
        const GaussianSet set = dequantize(q);
        for (std::size_t i = 0; i < set.size(); ++i) prim_to(set.primitives[i], out + 11 * i);
    });
}

}  // extern "C"
