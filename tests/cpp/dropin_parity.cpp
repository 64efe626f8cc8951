// dropin_parity.cpp — TEST ONLY. The reference's own call sequence, run twice
// on the same inputs: once through the reference (namespace gpile, header-only
// CPU implementation compiled into this binary as the oracle) and once through
// the drop-in (namespace gpile::b200, include/gpile_b200.hpp over the C-ABI).
// Mirrors the fit loop (optimize.hpp:385-402) and proj/tests/test_render.cpp /
// test_grad.cpp / test_voxelize.cpp pins. Exit status 0 iff every comparison
// is within the north-star tolerances (images 1e-4 rel, gradients 1e-3 rel,
// tile-derived survivor sets bit-exact).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <stdexcept>

#include "../../include/gpile_b200.hpp"

using namespace gpile;

static int failures = 0;

static void expect(bool ok, const char* what) {
    std::printf("%-58s %s\n", what, ok ? "ok" : "FAIL");
    if (!ok) ++failures;
}

static bool images_close(const SliceImage& a, const SliceImage& b) {
    if (a.width != b.width || a.height != b.height) return false;
    double peak = 0.0;
    for (double v : b.pixels) peak = std::fmax(peak, std::fabs(v));
    for (std::size_t i = 0; i < a.pixels.size(); ++i)
        if (std::fabs(a.pixels[i] - b.pixels[i]) > 1e-4 * std::fabs(b.pixels[i]) + 1e-6 * peak) return false;
    return true;
}

static bool grads_close(const GaussianGradients& a, const GaussianGradients& b) {
    if (a.size() != b.size()) return false;
    const std::size_t n = a.size();
    auto plane = [&](auto get) {
        double mx = 0.0;
        for (std::size_t i = 0; i < n; ++i) mx = std::fmax(mx, std::fabs(get(b, i)));
        for (std::size_t i = 0; i < n; ++i) {
            const double r = get(b, i), x = get(a, i);
            if (std::fabs(x - r) > 1e-3 * std::fabs(r) + 1e-3 * mx) return false;
        }
        return true;
    };
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
        ok &= plane([k](const GaussianGradients& g, std::size_t i) { return g.d_mu[i][k]; });
        ok &= plane([k](const GaussianGradients& g, std::size_t i) { return g.d_log_scale[i][k]; });
    }
    ok &= plane([](const GaussianGradients& g, std::size_t i) { return g.d_quat[i].w; });
    ok &= plane([](const GaussianGradients& g, std::size_t i) { return g.d_quat[i].x; });
    ok &= plane([](const GaussianGradients& g, std::size_t i) { return g.d_quat[i].y; });
    ok &= plane([](const GaussianGradients& g, std::size_t i) { return g.d_quat[i].z; });
    ok &= plane([](const GaussianGradients& g, std::size_t i) { return g.d_alpha_raw[i]; });
    return ok;
}

static GaussianSet f32_set(GaussianSet s) {  // the device stores f32: give both sides identical inputs
    auto r = [](double v) { return (double)(float)v; };
    for (auto& g : s.primitives) {
        g.mu = {r(g.mu.x), r(g.mu.y), r(g.mu.z)};
        g.log_scale = {r(g.log_scale.x), r(g.log_scale.y), r(g.log_scale.z)};
        g.quat = {r(g.quat.w), r(g.quat.x), r(g.quat.y), r(g.quat.z)};
        g.alpha_raw = r(g.alpha_raw);
    }
    return s;
}

int main() {
    VolumeGrid vol;
    vol.dims[0] = 96;
    vol.dims[1] = 80;
    vol.dims[2] = 24;
    const Bounds bbox = vol.world_bounds();
    const GaussianSet set = f32_set(init_random(8000, bbox, 1.5, 1));
    const PsfSpec psf{};
    const RasterConfig cfg{};

    // fit-loop sequence: prepare -> rasterize -> loss -> backward -> adam
    const SlicePose pose = slice_pose_for_index(vol, 11);
    const auto prep_ref = prepare_gaussians(set, pose, psf, cfg);
    const auto prep_gpu = b200::prepare_gaussians(set, pose, psf, cfg);
    bool same = prep_ref.size() == prep_gpu.size();
    for (std::size_t k = 0; same && k < prep_ref.size(); ++k)
        same = prep_ref[k].index == prep_gpu[k].index && prep_ref[k].lo_x == prep_gpu[k].lo_x &&
               prep_ref[k].hi_x == prep_gpu[k].hi_x && prep_ref[k].lo_y == prep_gpu[k].lo_y &&
               prep_ref[k].hi_y == prep_gpu[k].hi_y;
    expect(same, "prepare_gaussians: survivors + pixel bounds bit-exact");

    const SliceImage img_ref = rasterize_prepared(prep_ref, pose, cfg);
    const SliceImage img_gpu = b200::rasterize_prepared(prep_gpu, pose, cfg);
    expect(images_close(img_gpu, img_ref), "rasterize_prepared within 1e-4 rel");

    SliceImage target(vol.dims[0], vol.dims[1]);
    for (std::size_t i = 0; i < target.size(); ++i) target.pixels[i] = (double)(float)(0.05 + 0.04 * std::sin(0.37 * i));
    SliceImage dl_ref, dl_gpu;
    SliceImage img32 = img_gpu;  // both losses on the same (f32-exact) rendered image
    const double L_ref = photometric_loss(img32, target, 0.2, dl_ref);
    const double L_gpu = b200::photometric_loss(img32, target, 0.2, dl_gpu);
    expect(std::fabs(L_gpu - L_ref) <= 1e-5 * std::fabs(L_ref), "photometric_loss value within 1e-5 rel");

    ScreenGradStats st_ref, st_gpu;
    SliceImage dl32 = dl_ref;
    for (double& v : dl32.pixels) v = (double)(float)v;
    const GaussianGradients g_ref = backward_prepared(set, prep_ref, pose, dl32, cfg, &st_ref);
    const GaussianGradients g_gpu = b200::backward_prepared(set, prep_gpu, pose, dl32, cfg, &st_gpu);
    expect(grads_close(g_gpu, g_ref), "backward_prepared within 1e-3 rel (+plane floor)");
    expect(st_gpu.observed == st_ref.observed, "ScreenGradStats.observed identical");

    GaussianSet s_ref = set, s_gpu = set;
    AdamState a_ref(set.size()), a_gpu(set.size());
    const LearningRates lrs{6e-4, 0.02, 2e-3, 1e-3};
    adam_step(s_ref, g_gpu, a_ref, lrs);
    b200::adam_step(s_gpu, g_gpu, a_gpu, lrs);
    bool adam_ok = a_ref.step == a_gpu.step;
    for (std::size_t i = 0; adam_ok && i < set.size(); ++i)
        for (int k = 0; k < 3; ++k)
            adam_ok = std::fabs(s_ref.primitives[i].mu[k] - s_gpu.primitives[i].mu[k]) <=
                      2e-6 * std::fabs(s_ref.primitives[i].mu[k]) + 1e-6;
    expect(adam_ok, "adam_step parameters within fp32 tolerance");
    expect(b200::lr_at(6e-4, 7, 30) == lr_at(6e-4, 7, 30), "lr_at identical");

    // every PreparedGaussian field (render.hpp:68-79), reference fp64 order
    {
        auto close = [](double a, double b) { return std::fabs(a - b) <= 1e-9 * std::fabs(b) + 1e-12; };
        bool ok = prep_ref.size() == prep_gpu.size();
        for (std::size_t k = 0; ok && k < prep_ref.size(); ++k) {
            const PreparedGaussian &r = prep_ref[k], &g = prep_gpu[k];
            ok = close(g.alpha, r.alpha) && close(g.opacity_r, r.opacity_r) && close(g.alpha_tilde, r.alpha_tilde) &&
                 close(g.det2, r.det2);
            for (int i = 0; i < 3 && ok; ++i) ok = close(g.mu_c[i], r.mu_c[i]) && close(g.mu_e[i], r.mu_e[i]);
            for (int i = 0; i < 9 && ok; ++i)
                ok = close(g.sigma_c.m[i / 3][i % 3], r.sigma_c.m[i / 3][i % 3]) &&
                     close(g.sigma_c_inv.m[i / 3][i % 3], r.sigma_c_inv.m[i / 3][i % 3]) &&
                     close(g.sigma_e.m[i / 3][i % 3], r.sigma_e.m[i / 3][i % 3]);
            ok = ok && close(g.mu_2d.x, r.mu_2d.x) && close(g.mu_2d.y, r.mu_2d.y) && close(g.cov2d.a, r.cov2d.a) &&
                 close(g.cov2d.b, r.cov2d.b) && close(g.cov2d.c, r.cov2d.c) && close(g.cov2d.d, r.cov2d.d) &&
                 close(g.conic.a, r.conic.a) && close(g.conic.b, r.conic.b) && close(g.conic.c, r.conic.c) &&
                 close(g.conic.d, r.conic.d);
        }
        expect(ok, "PreparedGaussian: every field within 1e-9 rel");
    }

    // two prepared slices held at once, used in any order (the drop-in
    // re-binds an older vector on the device)
    {
        const SlicePose pa = slice_pose_for_index(vol, 6), pb = slice_pose_for_index(vol, 17);
        const auto ra = prepare_gaussians(set, pa, psf, cfg);
        const auto rb = prepare_gaussians(set, pb, psf, cfg);
        const auto ga = b200::prepare_gaussians(set, pa, psf, cfg);
        const auto gb = b200::prepare_gaussians(set, pb, psf, cfg);
        bool ok = images_close(b200::rasterize_prepared(ga, pa, cfg), rasterize_prepared(ra, pa, cfg));
        ok = ok && images_close(b200::rasterize_prepared(gb, pb, cfg), rasterize_prepared(rb, pb, cfg));
        SliceImage dla(pa.width, pa.height);
        for (std::size_t i = 0; i < dla.size(); ++i) dla.pixels[i] = (double)(float)(std::cos(0.11 * i) / dla.size());
        ok = ok && grads_close(b200::backward_prepared(set, ga, pa, dla, cfg), backward_prepared(set, ra, pa, dla, cfg));
        ok = ok && images_close(b200::rasterize_prepared(gb, pb, cfg), rasterize_prepared(rb, pb, cfg));
        expect(ok, "rasterize/backward_prepared on an older prepared vector");
        bool threw = false;
        try {
            std::vector<PreparedGaussian> foreign = ra;  // not returned by the drop-in
            (void)b200::rasterize_prepared(foreign, pa, cfg);
        } catch (const std::logic_error&) {
            threw = true;
        }
        expect(threw, "a vector the drop-in did not return -> std::logic_error");
    }

    // rasterize_slice / backward_slice, random pose, tau = 0 (test_grad.cpp:128-177)
    Rng rng(5);
    GaussianSet small;
    small.bbox = {{-3, -3, -3}, {3, 3, 3}};
    for (int i = 0; i < 30; ++i) {
        GaussianPrimitive g;
        g.mu = rng.uniform_in_box(small.bbox.min, small.bbox.max);
        g.log_scale = {std::log(rng.uniform(0.5, 2.0)), std::log(rng.uniform(0.5, 2.0)), std::log(rng.uniform(0.5, 2.0))};
        g.quat = rng.unit_quaternion();
        g.alpha_raw = alpha_activation_inverse(rng.uniform(0.2, 0.9));
        small.primitives.push_back(g);
    }
    small = f32_set(small);
    SlicePose rp;
    rp.rotation = quat_to_rotation(rng.unit_quaternion());
    rp.translation = {rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0)};
    rp.width = 24;
    rp.height = 20;
    rp.pixel_spacing = {0.5, 0.5};
    rp.principal_point = {12.0, 10.0};
    const RasterConfig cfg0{0.0, 16, 8.0, 1.0};
    const PsfSpec psf08{1.0, 1.0, 0.8};
    expect(images_close(b200::rasterize_slice(small, rp, psf08, cfg0), rasterize_slice(small, rp, psf08, cfg0)),
           "rasterize_slice (random pose) within 1e-4 rel");
    SliceImage dl(24, 20);
    for (std::size_t i = 0; i < dl.size(); ++i) dl.pixels[i] = (double)(float)std::cos(0.91 * i);
    expect(grads_close(b200::backward_slice(small, rp, psf08, dl, cfg0), backward_slice(small, rp, psf08, dl, cfg0)),
           "backward_slice (random pose) within 1e-3 rel");

    // voxelizer (voxelize.hpp:113-240)
    VoxelizerConfig vc;
    vc.dims[0] = 40;
    vc.dims[1] = 36;
    vc.dims[2] = 28;
    GaussianSet vs = f32_set(init_random(1500, {{2, 2, 2}, {38, 34, 26}}, 1.2, 9));
    const VolumeGrid v_ref = voxelize(vs, vc), v_gpu = b200::voxelize(vs, vc);
    double vpeak = 0.0;
    for (double x : v_ref.data) vpeak = std::fmax(vpeak, x);
    bool vok = v_gpu.data.size() == v_ref.data.size();
    for (std::size_t i = 0; vok && i < v_ref.data.size(); ++i)
        vok = std::fabs(v_gpu.data[i] - v_ref.data[i]) <= 1e-4 * std::fabs(v_ref.data[i]) + 1e-6 * vpeak;
    expect(vok, "voxelize within 1e-4 rel");
    VolumeGrid dlv = v_ref;
    for (std::size_t i = 0; i < dlv.data.size(); ++i) dlv.data[i] = (double)(float)std::sin(0.013 * i);
    expect(grads_close(b200::voxelize_backward(vs, vc, dlv), voxelize_backward(vs, vc, dlv)),
           "voxelize_backward within 1e-3 rel");

    // error semantics
    bool threw = false;
    try {
        VoxelizerConfig big;
        big.dims[0] = big.dims[1] = 2048;
        big.dims[2] = 1024;
        b200::voxelize(vs, big);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "voxelize > 2^31 voxels -> std::invalid_argument");
    threw = false;
    try {
        b200::rasterize_slice(set, pose, PsfSpec{1.0, 1.0, 0.0}, cfg);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "bad PsfSpec -> std::invalid_argument");
    threw = false;
    try {
        GaussianSet bad = small;
        bad.primitives[3].quat = {0, 0, 0, 0};
        b200::rasterize_slice(bad, rp, psf08, cfg0);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "zero quaternion -> std::invalid_argument");

    // densify_and_prune (optimize.hpp:255-344): same inputs, same Rng seed
    {
        GaussianSet ds = f32_set(init_random(2000, {{0, 0, 0}, {40, 40, 40}}, 0.4, 12));
        Rng r0(77);
        AdamState ad(ds.size());
        DensifyAccum acc(ds.size());
        for (std::size_t i = 0; i < ds.size(); ++i) {
            acc.observations[i] = (int)(i % 4);
            acc.grad_norm_sum[i] = acc.observations[i] * r0.uniform(0.0, 1e-4);
            acc.world_grad_sum[i] = {r0.normal(), r0.normal(), r0.normal()};
            ad.m_a[i] = (double)(float)r0.normal();
        }
        ad.step = 9;
        FitConfig fc;
        GaussianSet d_ref = ds, d_gpu = ds;
        AdamState a1 = ad, a2 = ad;
        Rng g1(31), g2(31);
        const DensifyReport r_ref = densify_and_prune(d_ref, a1, acc, fc, g1);
        const DensifyReport r_gpu = b200::densify_and_prune(d_gpu, a2, acc, fc, g2);
        bool dok = r_ref.pruned == r_gpu.pruned && r_ref.cloned == r_gpu.cloned && r_ref.split == r_gpu.split &&
                   d_ref.size() == d_gpu.size() && a2.size() == d_gpu.size() && a2.step == 9 &&
                   r_ref.cloned > 0 && r_ref.split > 0 && r_ref.pruned > 0;
        for (std::size_t i = 0; dok && i < d_ref.size(); ++i) {
            for (int k = 0; k < 3; ++k)
                dok = dok && std::fabs(d_ref.primitives[i].mu[k] - d_gpu.primitives[i].mu[k]) <=
                                 2e-7 * std::fabs(d_ref.primitives[i].mu[k]) + 1e-6;
            dok = dok && (float)a1.m_a[i] == (float)a2.m_a[i];
        }
        dok = dok && g1.normal() == g2.normal();  // the caller's generator advanced identically
        expect(dok, "densify_and_prune: report, order, moments, generator state");
    }

    // fit (optimize.hpp:360-424) on a blob volume, progress every 25
    {
        VolumeGrid fv;
        fv.dims[0] = 24;
        fv.dims[1] = 24;
        fv.dims[2] = 8;
        fv.data.assign(fv.voxel_count(), 0.0);
        for (int k = 0; k < 8; ++k)
            for (int j = 0; j < 24; ++j)
                for (int i = 0; i < 24; ++i) {
                    const double dx = (i - 12.0) / 3.0, dy = (j - 12.0) / 3.0, dz = (k - 3.0) / 1.5;
                    fv.at(i, j, k) = (double)(float)(0.9 * std::exp(-0.5 * (dx * dx + dy * dy + dz * dz)));
                }
        FitConfig fc;
        fc.iterations = 200;
        fc.init_count = 16;
        fc.densify_start = 100;
        fc.densify_end = 200;
        fc.densify_interval = 100;
        fc.rng_seed = 11;
        fc.progress_interval = 50;
        std::vector<FitProgress> pr, pg;
        const GaussianSet f_ref = fit(fv, PsfSpec{}, fc, [&](const FitProgress& p) { pr.push_back(p); });
        const GaussianSet f_gpu = b200::fit(fv, PsfSpec{}, fc, [&](const FitProgress& p) { pg.push_back(p); });
        bool fok = pr.size() == pg.size() && f_ref.size() == f_gpu.size() && f_gpu.size() > 16;
        for (std::size_t i = 0; fok && i < pr.size(); ++i)
            fok = pr[i].iteration == pg[i].iteration && pr[i].count == pg[i].count &&
                  std::fabs(pr[i].loss - pg[i].loss) <= 2e-3 * std::fabs(pr[i].loss) &&
                  std::fabs(pr[i].psnr2d - pg[i].psnr2d) <= 0.05;
        expect(fok, "fit: progress (count, loss, PSNR) tracks the reference");
        bool threw_cfg = false;
        try {
            FitConfig bad = fc;
            bad.densify_start = 300;
            bad.densify_end = 200;
            b200::fit(fv, PsfSpec{}, bad);
        } catch (const std::invalid_argument&) {
            threw_cfg = true;
        }
        expect(threw_cfg, "fit: FitConfig validation -> std::invalid_argument");
    }

    // checkpoints (checkpoint.hpp:38-92): byte-identical files, round trip
    {
        const std::string a = "/tmp/gpk_dropin_a.gpile", b = "/tmp/gpk_dropin_b.gpile";
        save_checkpoint(set, a);
        b200::save_checkpoint(set, b);
        std::ifstream fa(a, std::ios::binary), fb(b, std::ios::binary);
        const std::string ba((std::istreambuf_iterator<char>(fa)), {}), bb((std::istreambuf_iterator<char>(fb)), {});
        const GaussianSet back = b200::load_checkpoint(a);
        bool cok = ba == bb && back.size() == set.size() && back.bbox.max.x == set.bbox.max.x;
        for (std::size_t i = 0; cok && i < set.size(); ++i)
            cok = back.primitives[i].mu.y == set.primitives[i].mu.y &&
                  back.primitives[i].alpha_raw == set.primitives[i].alpha_raw;
        expect(cok, "save/load_checkpoint: byte-identical file, bitwise round trip");
        bool threw_c = false;
        try {
            b200::load_checkpoint("/tmp/gpk_dropin_missing.gpile");
        } catch (const LoadError&) {
            threw_c = true;
        }
        expect(threw_c, "load_checkpoint: missing file -> gpile::LoadError");
        std::remove(a.c_str());
        std::remove(b.c_str());
    }

    // codec front half (morton.hpp:33-48, quant.hpp:67-132)
    {
        const auto p_ref = morton_sort(set, 14), p_gpu = b200::morton_sort(set, 14);
        expect(p_ref == p_gpu, "morton_sort: identical stable permutation");
        QuantSpec qs;
        const QuantizedSet q_ref = quantize(set, qs), q_gpu = b200::quantize(set, qs);
        expect(q_ref.positions == q_gpu.positions && q_ref.opacities == q_gpu.opacities &&
                   q_ref.log_scales == q_gpu.log_scales && q_ref.quats == q_gpu.quats &&
                   q_ref.scale_min.x == q_gpu.scale_min.x && q_ref.scale_max.z == q_gpu.scale_max.z,
               "quantize: identical integer streams and scale ranges");
    }

    std::printf("%s\n", failures ? "DROPIN PARITY FAILED" : "DROPIN PARITY OK");
    return failures ? 1 : 0;
}
