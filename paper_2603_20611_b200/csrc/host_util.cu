// host_util.cu — host-side helpers of the fit driver that the benchmark and
// callers need to build inputs identical to the reference's:
//   gpk_init_random        init_random (optimize.hpp:94-108) on the reference's
//                          seeded generator: std::mt19937_64 with the
//                          self-contained distributions of rng.hpp:14-70.
//   gpk_slice_pose_for_index  slice_pose_for_index (core.hpp:202-211).
//   gpk_lr_at              lr_at (optimize.hpp:71-73).
// Pure host code (no kernels); the sequences are bit-identical to the
// reference because the engine is the standard one and the distribution
// arithmetic is the same.
#include <cmath>
#include <cstdint>
#include <random>

#include "../../include/gpile_b200.h"

namespace {

class SeededRng {
public:
    explicit SeededRng(uint64_t seed) : eng_(seed) {}
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    // Rng::below (rng.hpp:24-31): rejection keeps the draw unbiased
    uint64_t below(uint64_t n) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t v;
        do {
            v = eng_();
        } while (v >= limit);
        return v % n;
    }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1, u2;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare_ = r * std::sin(2.0 * M_PI * u2);
        have_spare_ = true;
        return r * std::cos(2.0 * M_PI * u2);
    }

private:
    std::mt19937_64 eng_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

double logit(double a) {
    const double eps = 1e-12;
    a = std::fmin(1.0 - eps, std::fmax(eps, a));
    return std::log(a / (1.0 - a));
}

// detail::sample_shape (optimize.hpp:81-88): log-scales, unit quaternion
// (Rng::unit_quaternion, rng.hpp:56-64), raw alpha
void sample_shape(SeededRng& rng, double scale_base, double* r) {
    for (int d = 0; d < 3; ++d) r[3 + d] = std::log(scale_base * (1.0 + rng.uniform(-0.2, 0.2)));
    double q[4], nrm;
    do {
        for (int k = 0; k < 4; ++k) q[k] = rng.normal();
        nrm = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    } while (nrm < 1e-12);
    for (int k = 0; k < 4; ++k) r[6 + k] = q[k] * (1.0 / nrm);
    r[10] = logit(0.1 * (1.0 + rng.uniform(-0.5, 0.5)));
}

}  // namespace

struct gpk_rng {
    SeededRng r;
    explicit gpk_rng(uint64_t seed) : r(seed) {}
};

extern "C" {

int gpk_rng_create(uint64_t seed, gpk_rng** out) {
    if (!out) return GPK_ERR_INVALID_ARGUMENT;
    *out = new gpk_rng(seed);
    return GPK_OK;
}

int gpk_rng_destroy(gpk_rng* g) {
    delete g;
    return GPK_OK;
}

int gpk_rng_uniform(gpk_rng* g, double* out) {
    if (!g || !out) return GPK_ERR_INVALID_ARGUMENT;
    *out = g->r.uniform();
    return GPK_OK;
}

int gpk_rng_below(gpk_rng* g, uint64_t n, uint64_t* out) {
    if (!g || !out || n == 0) return GPK_ERR_INVALID_ARGUMENT;
    *out = g->r.below(n);
    return GPK_OK;
}

int gpk_rng_normal(gpk_rng* g, double* out) {
    if (!g || !out) return GPK_ERR_INVALID_ARGUMENT;
    *out = g->r.normal();
    return GPK_OK;
}

// records: n x 11 doubles (record order). Draw order per primitive follows
// sample_shape (optimize.hpp:81-88) then the position (optimize.hpp:104).
int gpk_init_random(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                    double* records) {
    if (n < 1 || !bbox || !records) return GPK_ERR_INVALID_ARGUMENT;
    for (int d = 0; d < 3; ++d)
        if (!(bbox->max[d] > bbox->min[d])) return GPK_ERR_INVALID_ARGUMENT;
    SeededRng rng(seed);
    for (uint64_t i = 0; i < n; ++i) {
        double* r = records + 11 * i;
        sample_shape(rng, scale_base, r);
        for (int d = 0; d < 3; ++d) r[d] = rng.uniform(bbox->min[d], bbox->max[d]);
    }
    return GPK_OK;
}

// Lattice positions in k, j, i order (z slowest); the shape is drawn before
// the position is set, as the reference draws it (optimize.hpp:123-131).
int gpk_init_grid(uint64_t n, const gpk_bounds* bbox, double scale_base, uint64_t seed,
                  double* records) {
    if (n < 1 || !bbox || !records) return GPK_ERR_INVALID_ARGUMENT;
    for (int d = 0; d < 3; ++d)
        if (!(bbox->max[d] > bbox->min[d])) return GPK_ERR_INVALID_ARGUMENT;
    SeededRng rng(seed);
    uint64_t side = static_cast<uint64_t>(std::ceil(std::cbrt(static_cast<double>(n)) - 1e-9));
    while (side * side * side < n) ++side;
    const double ext[3] = {bbox->max[0] - bbox->min[0], bbox->max[1] - bbox->min[1],
                           bbox->max[2] - bbox->min[2]};
    uint64_t c = 0;
    for (uint64_t k = 0; k < side && c < n; ++k)
        for (uint64_t j = 0; j < side && c < n; ++j)
            for (uint64_t i = 0; i < side && c < n; ++i, ++c) {
                double* r = records + 11 * c;
                sample_shape(rng, scale_base, r);
                const uint64_t ijk[3] = {i, j, k};
                for (int d = 0; d < 3; ++d)
                    r[d] = bbox->min[d] + (ijk[d] + 0.5) / side * ext[d];
            }
    return GPK_OK;
}

int gpk_slice_pose_for_index(const int32_t dims[3], const double spacing[3], const double origin[3],
                             int k, gpk_slice_pose* out) {
    if (!dims || !spacing || !origin || !out) return GPK_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < 9; ++i) out->rotation[i] = (i % 4 == 0) ? 1.0 : 0.0;
    out->translation[0] = (origin[0] + 0.0) * -1.0;
    out->translation[1] = (origin[1] + 0.0) * -1.0;
    out->translation[2] = (origin[2] + k * spacing[2]) * -1.0;
    out->width = dims[0];
    out->height = dims[1];
    out->pixel_spacing[0] = spacing[0];
    out->pixel_spacing[1] = spacing[1];
    out->principal_point[0] = 0.0;
    out->principal_point[1] = 0.0;
    return GPK_OK;
}

double gpk_lr_at(double lr0, int iteration, int total) {
    return lr0 * std::pow(0.1, static_cast<double>(iteration - 1) / total);
}

}  // extern "C"
