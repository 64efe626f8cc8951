/* gpile_oracle.c — TEST INFRASTRUCTURE ONLY: fp64 C restatement of the
 * GaussianPile hot path (see gpile_oracle.h). Single-threaded; every loop runs
 * in the reference's index order, so results equal the reference's
 * bit-for-bit when compiled like it (gcc -O2, x86-64, no FMA contraction).
 * Citations are to /root/reference/proj/include/gpile/<file>:<line>.
 */
#define _GNU_SOURCE
#include "gpile_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
static int64_t g_err_index = -1;

const char* gor_last_error(void) { return g_err; }
int64_t gor_last_error_index(void) { return g_err_index; }

static int fail(int code, int64_t idx, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    g_err_index = idx;
    return code;
}

static int ok(void) {
    g_err[0] = 0;
    g_err_index = -1;
    return GPK_OK;
}

/* ---- vec.hpp: fixed-size fp64 algebra, same evaluation order ------------- */
typedef struct { double x, y, z; } v3;
typedef struct { double m[3][3]; } m3;

static m3 m3_zero(void) { m3 r; memset(&r, 0, sizeof r); return r; }
static m3 m3_eye(void) { m3 r = m3_zero(); r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0; return r; }

static double v3_get(v3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }
static double v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }  /* vec.hpp:26 */

static m3 m3_mul(m3 a, m3 b) {  /* vec.hpp:107-113 */
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
    return r;
}
static v3 m3_mulv(m3 a, v3 v) {  /* vec.hpp:114-118 */
    v3 r = {a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
            a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
            a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z};
    return r;
}
static m3 m3_t(m3 a) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
static m3 m3_add(m3 a, m3 b) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
    return r;
}
static m3 m3_sub(m3 a, m3 b) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] - b.m[i][j];
    return r;
}
static m3 m3_scale(m3 a, double s) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] * s;
    return r;
}
static m3 m3_outer(v3 u, v3 v) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = v3_get(u, i) * v3_get(v, j);
    return r;
}
static double m3_det(m3 a) {  /* vec.hpp:131-135 */
    return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
           a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
           a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
static m3 m3_inv(m3 a) {  /* vec.hpp:137-150 */
    const double dt = m3_det(a);
    double (*m)[3] = a.m;
    m3 r;
    r.m[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / dt;
    r.m[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / dt;
    r.m[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / dt;
    r.m[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / dt;
    r.m[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / dt;
    r.m[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / dt;
    r.m[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / dt;
    r.m[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / dt;
    r.m[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / dt;
    return r;
}
static void m3_eig(m3 a, double out[3]) {  /* vec.hpp:154-179 */
    double (*m)[3] = a.m;
    const double p1 = m[0][1] * m[0][1] + m[0][2] * m[0][2] + m[1][2] * m[1][2];
    if (p1 == 0.0) {
        double d[3] = {m[0][0], m[1][1], m[2][2]}, t;
        if (d[0] > d[1]) { t = d[0]; d[0] = d[1]; d[1] = t; }
        if (d[1] > d[2]) { t = d[1]; d[1] = d[2]; d[2] = t; }
        if (d[0] > d[1]) { t = d[0]; d[0] = d[1]; d[1] = t; }
        out[0] = d[0]; out[1] = d[1]; out[2] = d[2];
        return;
    }
    const double q = (m[0][0] + m[1][1] + m[2][2]) / 3.0;
    const double p2 = (m[0][0] - q) * (m[0][0] - q) + (m[1][1] - q) * (m[1][1] - q) +
                      (m[2][2] - q) * (m[2][2] - q) + 2.0 * p1;
    const double p = sqrt(p2 / 6.0);
    m3 B = m3_scale(m3_sub(a, m3_scale(m3_eye(), q)), 1.0 / p);
    double r = m3_det(B) / 2.0;
    r = fmax(-1.0, fmin(1.0, r));
    const double phi = acos(r) / 3.0;
    const double e_hi = q + 2.0 * p * cos(phi);
    const double e_lo = q + 2.0 * p * cos(phi + 2.0 * M_PI / 3.0);
    out[0] = e_lo;
    out[2] = e_hi;
    out[1] = 3.0 * q - e_lo - e_hi;
}

/* x86-64 static_cast<int>(double): NaN / out of range -> INT_MIN. */
static int trunc_int(double v) {
    if (!(v >= -2147483648.0 && v < 2147483648.0)) return (int)0x80000000u;
    return (int)v;
}

/* ---- core.hpp ------------------------------------------------------------ */
static double alpha_act(double raw) { return 1.0 / (1.0 + exp(-raw)); } /* core.hpp:21 */

static int quat_rot(const double q[4], m3* r) { /* vec.hpp:183-199 */
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(n > 0.0) || !isfinite(n)) return GPK_ERR_INVALID_ARGUMENT;
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    r->m[0][0] = 1.0 - 2.0 * (y * y + z * z);
    r->m[0][1] = 2.0 * (x * y - w * z);
    r->m[0][2] = 2.0 * (x * z + w * y);
    r->m[1][0] = 2.0 * (x * y + w * z);
    r->m[1][1] = 1.0 - 2.0 * (x * x + z * z);
    r->m[1][2] = 2.0 * (y * z - w * x);
    r->m[2][0] = 2.0 * (x * z - w * y);
    r->m[2][1] = 2.0 * (y * z + w * x);
    r->m[2][2] = 1.0 - 2.0 * (x * x + y * y);
    return GPK_OK;
}

static int cov_from_scale_rot(const double* rec, double mod, m3* sigma) { /* core.hpp:165-173 */
    const double s[3] = {exp(rec[3]), exp(rec[4]), exp(rec[5])};
    if (!(s[0] > 0.0) || !(s[1] > 0.0) || !(s[2] > 0.0) || !(mod > 0.0))
        return GPK_ERR_INVALID_ARGUMENT;
    m3 r;
    if (quat_rot(rec + 6, &r)) return GPK_ERR_INVALID_ARGUMENT;
    const double sx = mod * s[0], sy = mod * s[1], sz = mod * s[2];
    m3 s2 = m3_zero();
    s2.m[0][0] = sx * sx;
    s2.m[1][1] = sy * sy;
    s2.m[2][2] = sz * sz;
    *sigma = m3_mul(m3_mul(r, s2), m3_t(r));
    return GPK_OK;
}

static int invert_cov(m3 sigma, m3* out) { /* core.hpp:184-198 */
    double ev[3];
    m3_eig(sigma, ev);
    m3 s = sigma;
    if (!(ev[0] > 0.0) || ev[2] / ev[0] > 1e12) {
        const double eps = 1e-9 * (sigma.m[0][0] + sigma.m[1][1] + sigma.m[2][2]) / 3.0;
        if (!(eps > 0.0)) return GPK_ERR_DEGENERATE_COVARIANCE;
        for (int i = 0; i < 3; ++i) s.m[i][i] += eps;
        m3_eig(s, ev);
        if (!(ev[0] > 0.0)) return GPK_ERR_DEGENERATE_COVARIANCE;
    }
    *out = m3_inv(s);
    return GPK_OK;
}

static m3 pose_rot(const gpk_slice_pose* p) {
    m3 r;
    for (int i = 0; i < 9; ++i) r.m[i / 3][i % 3] = p->rotation[i];
    return r;
}

/* ---- render.hpp: prepare_gaussians --------------------------------------- */
typedef struct {
    uint32_t index;
    double alpha, op, at;
    v3 mu_c, mu_e;
    m3 sc, sci, se;
    double mux, muy;
    double ca, cb, cc, cd;      /* cov2d */
    double ka, kb, kc, kd;      /* conic */
    double det2;
    int lo_x, hi_x, lo_y, hi_y;
} prep_t;

static int validate_psf(const gpk_psf* p) { /* core.hpp:112-116 */
    if (!(p->sigma_x > 0.0) || !(p->sigma_y > 0.0) || !(p->sigma_z > 0.0) || !isfinite(p->sigma_x) ||
        !isfinite(p->sigma_y) || !isfinite(p->sigma_z))
        return fail(GPK_ERR_INVALID_ARGUMENT, -1, "PsfSpec: sigmas must be positive and finite");
    return GPK_OK;
}

/* render.hpp:83-138: survivors in ascending set order; *out malloc'ed. */
static int prepare_all(uint64_t n, const double* rec, const gpk_slice_pose* pose,
                       const gpk_psf* psf, const gpk_raster_config* cfg, prep_t** out,
                       uint64_t* count) {
    prep_t* all = (prep_t*)malloc(sizeof(prep_t) * (n ? n : 1));
    uint64_t k = 0;
    const m3 R = pose_rot(pose);
    const m3 Rt = m3_t(R);
    for (uint64_t i = 0; i < n; ++i) {
        const double* g = rec + 11 * i;
        prep_t p;
        memset(&p, 0, sizeof p);
        p.index = (uint32_t)i;
        p.alpha = alpha_act(g[10]);
        m3 sigma;
        if (cov_from_scale_rot(g, cfg->scale_modifier, &sigma)) {
            free(all);
            return fail(GPK_ERR_INVALID_ARGUMENT, (int64_t)i, "invalid primitive");
        }
        const v3 mu = {g[0], g[1], g[2]};
        const v3 rm = m3_mulv(R, mu); /* core.hpp:176-180 */
        p.mu_c.x = rm.x + pose->translation[0];
        p.mu_c.y = rm.y + pose->translation[1];
        p.mu_c.z = rm.z + pose->translation[2];
        p.sc = m3_mul(m3_mul(R, sigma), Rt);
        if (invert_cov(p.sc, &p.sci)) {
            free(all);
            return fail(GPK_ERR_DEGENERATE_COVARIANCE, (int64_t)i, "invert_covariance");
        }
        m3 b = p.sci;
        b.m[2][2] += 1.0 / (psf->sigma_z * psf->sigma_z);
        p.se = m3_inv(b);
        const v3 amu = m3_mulv(p.sci, p.mu_c);
        p.mu_e = m3_mulv(p.se, amu);
        const double q = v3_dot(p.mu_c, amu) - v3_dot(p.mu_e, m3_mulv(b, p.mu_e)); /* :105 */
        p.op = exp(-0.5 * q);
        if (p.alpha * p.op < cfg->tau) continue; /* :107 */
        p.mux = p.mu_e.x;
        p.muy = p.mu_e.y;
        p.ca = p.se.m[0][0];
        p.cb = p.se.m[0][1];
        p.cc = p.se.m[1][0];
        p.cd = p.se.m[1][1];
        p.det2 = p.ca * p.cd - p.cb * p.cc;
        if (!(p.det2 > 0.0)) {
            free(all);
            return fail(GPK_ERR_DEGENERATE_COVARIANCE, (int64_t)i,
                        "prepare_gaussians: non-positive det(Sigma_2d)");
        }
        const double dt = p.ca * p.cd - p.cb * p.cc; /* Mat2::inverse, vec.hpp:51-54 */
        p.ka = p.cd / dt;
        p.kb = -p.cb / dt;
        p.kc = -p.cc / dt;
        p.kd = p.ca / dt;
        p.at = p.alpha * p.op / sqrt(p.det2);
        const double m = 0.5 * (p.ca + p.cd); /* vec.hpp:63-68 */
        const double r = sqrt(0.25 * (p.ca - p.cd) * (p.ca - p.cd) + p.cb * p.cb);
        const double hi_ev = m + r;
        const double radius = cfg->footprint_sigmas * sqrt(fmax(hi_ev, 0.0));
        const double cx = p.mux / pose->pixel_spacing[0] + pose->principal_point[0];
        const double cy = p.muy / pose->pixel_spacing[1] + pose->principal_point[1];
        const double rx = radius / pose->pixel_spacing[0];
        const double ry = radius / pose->pixel_spacing[1];
        int v;
        v = trunc_int(ceil(cx - rx)); p.lo_x = v > 0 ? v : 0;
        v = trunc_int(floor(cx + rx)); p.hi_x = v < pose->width - 1 ? v : pose->width - 1;
        v = trunc_int(ceil(cy - ry)); p.lo_y = v > 0 ? v : 0;
        v = trunc_int(floor(cy + ry)); p.hi_y = v < pose->height - 1 ? v : pose->height - 1;
        if (p.lo_x > p.hi_x || p.lo_y > p.hi_y) continue; /* :127 */
        all[k++] = p;
    }
    *out = all;
    *count = k;
    return GPK_OK;
}

int gor_prepare(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                const gpk_raster_config* cfg, uint64_t* count, uint32_t* index, int32_t* bounds,
                double* fields) {
    if (validate_psf(psf)) return GPK_ERR_INVALID_ARGUMENT;
    prep_t* P;
    uint64_t S;
    int st = prepare_all(n, rec, pose, psf, cfg, &P, &S);
    if (st) return st;
    *count = S;
    for (uint64_t k = 0; k < S; ++k) {
        const prep_t* p = &P[k];
        if (index) index[k] = p->index;
        if (bounds) {
            bounds[4 * k] = p->lo_x;
            bounds[4 * k + 1] = p->hi_x;
            bounds[4 * k + 2] = p->lo_y;
            bounds[4 * k + 3] = p->hi_y;
        }
        if (fields) {
            double* f = fields + 19 * k;
            f[0] = p->alpha; f[1] = p->op; f[2] = p->at;
            f[3] = p->mu_c.x; f[4] = p->mu_c.y; f[5] = p->mu_c.z;
            f[6] = p->mu_e.x; f[7] = p->mu_e.y; f[8] = p->mu_e.z;
            f[9] = p->mux; f[10] = p->muy;
            f[11] = p->ca; f[12] = p->cb; f[13] = p->cd;
            f[14] = p->ka; f[15] = p->kb; f[16] = p->kd;
            f[17] = p->det2; f[18] = p->se.m[2][2];
        }
    }
    free(P);
    return ok();
}

/* ---- render.hpp:142-160: TileGrid as CSR (offsets, prepared indices) ------- */
typedef struct {
    int tiles_x, tiles_y, tile;
    uint32_t* off;   /* tiles + 1 */
    uint32_t* ent;   /* prepared indices */
} grid_t;

static void grid_build(grid_t* g, const gpk_slice_pose* pose, const prep_t* P, uint64_t S, int tile) {
    g->tile = tile;
    g->tiles_x = (pose->width + tile - 1) / tile;
    g->tiles_y = (pose->height + tile - 1) / tile;
    const int T = g->tiles_x * g->tiles_y;
    g->off = (uint32_t*)calloc((size_t)T + 1, sizeof(uint32_t));
    for (uint64_t pi = 0; pi < S; ++pi)
        for (int ty = P[pi].lo_y / tile; ty <= P[pi].hi_y / tile; ++ty)
            for (int tx = P[pi].lo_x / tile; tx <= P[pi].hi_x / tile; ++tx) g->off[ty * g->tiles_x + tx + 1]++;
    for (int t = 0; t < T; ++t) g->off[t + 1] += g->off[t];
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)T + 1));
    memcpy(cur, g->off, sizeof(uint32_t) * ((size_t)T + 1));
    g->ent = (uint32_t*)malloc(sizeof(uint32_t) * (g->off[T] ? g->off[T] : 1));
    for (uint64_t pi = 0; pi < S; ++pi) /* ascending pi -> ascending within each list */
        for (int ty = P[pi].lo_y / tile; ty <= P[pi].hi_y / tile; ++ty)
            for (int tx = P[pi].lo_x / tile; tx <= P[pi].hi_x / tile; ++tx)
                g->ent[cur[ty * g->tiles_x + tx]++] = (uint32_t)pi;
    free(cur);
}

static void grid_free(grid_t* g) {
    free(g->off);
    free(g->ent);
}

int gor_tile_lists(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                   const gpk_raster_config* cfg, uint32_t* offsets, uint32_t* entries,
                   uint64_t capacity, uint64_t* total, uint64_t* tiles) {
    prep_t* P;
    uint64_t S;
    int st = prepare_all(n, rec, pose, psf, cfg, &P, &S);
    if (st) return st;
    grid_t g;
    grid_build(&g, pose, P, S, cfg->tile_size);
    const int T = g.tiles_x * g.tiles_y;
    *tiles = (uint64_t)T;
    *total = g.off[T];
    if (offsets) memcpy(offsets, g.off, sizeof(uint32_t) * ((size_t)T + 1));
    if (entries)
        for (uint32_t k = 0; k < g.off[T] && k < capacity; ++k) entries[k] = P[g.ent[k]].index;
    grid_free(&g);
    free(P);
    return ok();
}

/* ---- render.hpp:166-199: tiled rasterization ------------------------------ */
int gor_rasterize(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                  const gpk_raster_config* cfg, double* image) {
    if (validate_psf(psf)) return GPK_ERR_INVALID_ARGUMENT;
    prep_t* P;
    uint64_t S;
    int st = prepare_all(n, rec, pose, psf, cfg, &P, &S);
    if (st) return st;
    const int W = pose->width, H = pose->height;
    memset(image, 0, sizeof(double) * (size_t)W * H);
    grid_t g;
    grid_build(&g, pose, P, S, cfg->tile_size);
    for (int t = 0; t < g.tiles_x * g.tiles_y; ++t) {
        const int tx = t % g.tiles_x, ty = t / g.tiles_x;
        const int x0 = tx * g.tile, x1 = (W < x0 + g.tile) ? W : x0 + g.tile;
        const int y0 = ty * g.tile, y1 = (H < y0 + g.tile) ? H : y0 + g.tile;
        for (uint32_t k = g.off[t]; k < g.off[t + 1]; ++k) {
            const prep_t* p = &P[g.ent[k]];
            const int ax0 = x0 > p->lo_x ? x0 : p->lo_x, ax1 = (x1 - 1) < p->hi_x ? x1 - 1 : p->hi_x;
            const int ay0 = y0 > p->lo_y ? y0 : p->lo_y, ay1 = (y1 - 1) < p->hi_y ? y1 - 1 : p->hi_y;
            for (int j = ay0; j <= ay1; ++j)
                for (int i = ax0; i <= ax1; ++i) {
                    const double dx = (i - pose->principal_point[0]) * pose->pixel_spacing[0] - p->mux;
                    const double dy = (j - pose->principal_point[1]) * pose->pixel_spacing[1] - p->muy;
                    const double e = p->ka * dx * dx + 2.0 * p->kb * dx * dy + p->kd * dy * dy;
                    image[(size_t)j * W + i] += p->at * exp(-0.5 * e);
                }
        }
    }
    grid_free(&g);
    free(P);
    return ok();
}

/* rasterize_naive (render.hpp:203-219): survivors in set order, each over its
 * whole pixel box — the all-pairs oracle the tiled path must equal bitwise. */
int gor_rasterize_naive(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                        const gpk_raster_config* cfg, double* image) {
    if (validate_psf(psf)) return GPK_ERR_INVALID_ARGUMENT;
    prep_t* P;
    uint64_t S;
    int st = prepare_all(n, rec, pose, psf, cfg, &P, &S);
    if (st) return st;
    const int W = pose->width, H = pose->height;
    memset(image, 0, sizeof(double) * (size_t)W * H);
    for (uint64_t k = 0; k < S; ++k) {
        const prep_t* p = &P[k];
        for (int j = p->lo_y; j <= p->hi_y; ++j)
            for (int i = p->lo_x; i <= p->hi_x; ++i) {
                const double dx = (i - pose->principal_point[0]) * pose->pixel_spacing[0] - p->mux;
                const double dy = (j - pose->principal_point[1]) * pose->pixel_spacing[1] - p->muy;
                const double e = p->ka * dx * dx + 2.0 * p->kb * dx * dy + p->kd * dy * dy;
                image[(size_t)j * W + i] += p->at * exp(-0.5 * e);
            }
    }
    free(P);
    return ok();
}

/* ---- backward.hpp + grad_chain.hpp ---------------------------------------- */
static void rotation_backward(const double q[4], m3 g, double out[4]) { /* grad_chain.hpp:27-40 */
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    double (*G)[3] = g.m;
    out[0] = 2.0 * (-z * G[0][1] + y * G[0][2] + z * G[1][0] - x * G[1][2] - y * G[2][0] + x * G[2][1]);
    out[1] = 2.0 * (y * G[0][1] + z * G[0][2] + y * G[1][0] - 2.0 * x * G[1][1] - w * G[1][2] +
                    z * G[2][0] + w * G[2][1] - 2.0 * x * G[2][2]);
    out[2] = 2.0 * (-2.0 * y * G[0][0] + x * G[0][1] + w * G[0][2] + x * G[1][0] + z * G[1][2] -
                    w * G[2][0] + z * G[2][1] - 2.0 * y * G[2][2]);
    out[3] = 2.0 * (-2.0 * z * G[0][0] - w * G[0][1] + x * G[0][2] + w * G[1][0] - 2.0 * z * G[1][1] +
                    y * G[1][2] + x * G[2][0] + y * G[2][1]);
}

/* grad_chain.hpp:48-77 */
static void chain_world(const double* g, m3 dl_dsigma, double mod, double d_ls[3], double d_q[4]) {
    const double qn = sqrt(g[6] * g[6] + g[7] * g[7] + g[8] * g[8] + g[9] * g[9]);
    const double inv = 1.0 / qn;
    const double q[4] = {g[6] * inv, g[7] * inv, g[8] * inv, g[9] * inv}; /* core.hpp:42-46 */
    m3 r;
    quat_rot(q, &r);
    const double s[3] = {exp(g[3]), exp(g[4]), exp(g[5])};
    const double ms[3] = {mod * s[0], mod * s[1], mod * s[2]};
    const m3 sym2 = m3_add(dl_dsigma, m3_t(dl_dsigma));
    m3 M;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) M.m[i][j] = r.m[i][j] * ms[j];
    const m3 dl_dm = m3_mul(sym2, M);
    for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int i = 0; i < 3; ++i) acc += r.m[i][j] * dl_dm.m[i][j];
        d_ls[j] = acc * mod * s[j];
    }
    m3 dl_dr;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dl_dr.m[i][j] = dl_dm.m[i][j] * ms[j];
    double dq[4];
    rotation_backward(q, dl_dr, dq);
    const double along = dq[0] * q[0] + dq[1] * q[1] + dq[2] * q[2] + dq[3] * q[3];
    for (int k = 0; k < 4; ++k) d_q[k] = (dq[k] - q[k] * along) * (1.0 / qn);
}

typedef struct { double at, mx, my, cxx, cxy, cyy; } accum_t; /* backward.hpp:32-44 */

int gor_backward(uint64_t n, const double* rec, const gpk_slice_pose* pose, const gpk_psf* psf,
                 const gpk_raster_config* cfg, const double* dl_di, double* grads,
                 double* stat_norm, uint8_t* stat_observed, double* stat_world) {
    if (validate_psf(psf)) return GPK_ERR_INVALID_ARGUMENT;
    prep_t* P;
    uint64_t S;
    int st = prepare_all(n, rec, pose, psf, cfg, &P, &S);
    if (st) return st;
    const int W = pose->width, H = pose->height;
    grid_t g;
    grid_build(&g, pose, P, S, cfg->tile_size);
    const int T = g.tiles_x * g.tiles_y;
    accum_t* part = (accum_t*)calloc(g.off[T] ? g.off[T] : 1, sizeof(accum_t));
    /* stage 1 (backward.hpp:108-139) */
    for (int t = 0; t < T; ++t) {
        const int tx = t % g.tiles_x, ty = t / g.tiles_x;
        const int x0 = tx * g.tile, x1 = (W < x0 + g.tile) ? W : x0 + g.tile;
        const int y0 = ty * g.tile, y1 = (H < y0 + g.tile) ? H : y0 + g.tile;
        for (uint32_t k = g.off[t]; k < g.off[t + 1]; ++k) {
            const prep_t* p = &P[g.ent[k]];
            accum_t a = {0, 0, 0, 0, 0, 0};
            const int ax0 = x0 > p->lo_x ? x0 : p->lo_x, ax1 = (x1 - 1) < p->hi_x ? x1 - 1 : p->hi_x;
            const int ay0 = y0 > p->lo_y ? y0 : p->lo_y, ay1 = (y1 - 1) < p->hi_y ? y1 - 1 : p->hi_y;
            for (int j = ay0; j <= ay1; ++j)
                for (int i = ax0; i <= ax1; ++i) {
                    const double gi = dl_di[(size_t)j * W + i];
                    if (gi == 0.0) continue;
                    const double dx = (i - pose->principal_point[0]) * pose->pixel_spacing[0] - p->mux;
                    const double dy = (j - pose->principal_point[1]) * pose->pixel_spacing[1] - p->muy;
                    const double cdx = p->ka * dx + p->kb * dy, cdy = p->kc * dx + p->kd * dy;
                    const double e = exp(-0.5 * (dx * cdx + dy * cdy));
                    a.at += gi * e;
                    const double w = p->at * e * gi;
                    a.mx = a.mx + cdx * w;
                    a.my = a.my + cdy * w;
                    a.cxx += w * (-0.5) * dx * dx;
                    a.cxy += w * (-0.5) * dx * dy;
                    a.cyy += w * (-0.5) * dy * dy;
                }
            part[k] = a;
        }
    }
    /* stage 2: merge in tile order (backward.hpp:141-145) */
    accum_t* tot = (accum_t*)calloc(S ? S : 1, sizeof(accum_t));
    for (uint32_t k = 0; k < g.off[T]; ++k) {
        accum_t* d = &tot[g.ent[k]];
        d->at += part[k].at;
        d->mx = d->mx + part[k].mx;
        d->my = d->my + part[k].my;
        d->cxx += part[k].cxx;
        d->cxy += part[k].cxy;
        d->cyy += part[k].cyy;
    }
    memset(grads, 0, sizeof(double) * 11 * n);
    if (stat_norm) memset(stat_norm, 0, sizeof(double) * n);
    if (stat_observed) memset(stat_observed, 0, n);
    if (stat_world) memset(stat_world, 0, sizeof(double) * 3 * n);
    const m3 R = pose_rot(pose), Rt = m3_t(R);
    /* stage 3 (backward.hpp:148-173): camera_space_backward (:55-89) + chain */
    for (uint64_t pi = 0; pi < S; ++pi) {
        const prep_t* p = &P[pi];
        const accum_t* a = &tot[pi];
        const double sqrt_det = sqrt(p->det2);
        const double d_alpha = a->at * p->op / sqrt_det;
        const double d_opacity = a->at * p->alpha / sqrt_det;
        const double d_det = a->at * p->alpha * p->op * (-0.5) / (p->det2 * sqrt_det);
        /* Mat2 products (vec.hpp:56-59) */
        const double xa = a->cxx, xb = a->cxy, xc = a->cxy, xd = a->cyy;
        const double ta = p->ka * xa + p->kb * xc, tb = p->ka * xb + p->kb * xd;
        const double tc = p->kc * xa + p->kd * xc, td = p->kc * xb + p->kd * xd;
        const double cma = ta * p->ka + tb * p->kc, cmb = ta * p->kb + tb * p->kd;
        const double cmc = tc * p->ka + td * p->kc, cmd = tc * p->kb + td * p->kd;
        const double kk = d_det * p->det2;
        m3 gse = m3_zero();
        gse.m[0][0] = cma * -1.0 + p->ka * kk;
        gse.m[0][1] = cmb * -1.0 + p->kb * kk;
        gse.m[1][0] = cmc * -1.0 + p->kc * kk;
        gse.m[1][1] = cmd * -1.0 + p->kd * kk;
        const v3 g_mu_e = {a->mx, a->my, 0.0};
        const double g_q = d_opacity * (-0.5) * p->op;
        const v3 delta = {p->mu_c.x - p->mu_e.x, p->mu_c.y - p->mu_e.y, p->mu_c.z - p->mu_e.z};
        const v3 seg = m3_mulv(p->se, g_mu_e);
        const v3 a1 = m3_mulv(p->sci, seg), a2 = m3_mulv(p->sci, delta);
        const v3 dmc = {a1.x + a2.x * (2.0 * g_q), a1.y + a2.y * (2.0 * g_q), a1.z + a2.z * (2.0 * g_q)};
        m3 dl_da = m3_sub(m3_add(m3_outer(seg, delta), m3_scale(m3_outer(delta, delta), g_q)),
                          m3_mul(m3_mul(p->se, gse), p->se));
        dl_da = m3_scale(m3_add(dl_da, m3_t(dl_da)), 0.5);
        const m3 dsc = m3_scale(m3_mul(m3_mul(p->sci, dl_da), p->sci), -1.0);
        const v3 dmu = m3_mulv(Rt, dmc);
        const m3 dsig = m3_mul(m3_mul(Rt, dsc), R);
        const double* gp = rec + 11 * p->index;
        double d_ls[3], d_q[4];
        chain_world(gp, dsig, cfg->scale_modifier, d_ls, d_q);
        double* o = grads + 11 * (size_t)p->index;
        o[0] = dmu.x; o[1] = dmu.y; o[2] = dmu.z;
        o[3] = d_ls[0]; o[4] = d_ls[1]; o[5] = d_ls[2];
        o[6] = d_q[0]; o[7] = d_q[1]; o[8] = d_q[2]; o[9] = d_q[3];
        o[10] = d_alpha * (p->alpha * (1.0 - p->alpha));
        if (stat_norm) stat_norm[p->index] = sqrt(a->mx * a->mx + a->my * a->my);
        if (stat_observed) stat_observed[p->index] = 1;
        if (stat_world) {
            stat_world[3 * (size_t)p->index] = dmu.x;
            stat_world[3 * (size_t)p->index + 1] = dmu.y;
            stat_world[3 * (size_t)p->index + 2] = dmu.z;
        }
    }
    free(tot);
    free(part);
    grid_free(&g);
    free(P);
    /* backward.hpp:175-185 */
    for (uint64_t i = 0; i < n; ++i) {
        const double* o = grads + 11 * i;
        if (!(isfinite(o[10]) && isfinite(o[0] + o[1] + o[2]) && isfinite(o[3] + o[4] + o[5]) &&
              isfinite(o[6] + o[7] + o[8] + o[9]))) {
            char m[96];
            snprintf(m, sizeof m, "backward_slice: non-finite gradient for primitive %llu",
                     (unsigned long long)i);
            return fail(GPK_ERR_NUMERIC_FAILURE, (int64_t)i, m);
        }
    }
    return ok();
}

/* ---- metrics.hpp + loss.hpp ------------------------------------------------ */
static int reflect_index(int p, int n) { /* metrics.hpp:77-83 */
    while (p < 0 || p >= n) {
        if (p < 0) p = -p - 1;
        if (p >= n) p = 2 * n - 1 - p;
    }
    return p;
}

/* metrics.hpp:88-108 (2-D), then conv_nd (:110-118): axis 0 then axis 1. */
static void conv2(const double* in, double* out, int nx, int ny, const double* w) {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)nx * ny);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double acc = 0.0;
            for (int t = -5; t <= 5; ++t) acc += w[t + 5] * in[(size_t)j * nx + reflect_index(i + t, nx)];
            tmp[(size_t)j * nx + i] = acc;
        }
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double acc = 0.0;
            for (int t = -5; t <= 5; ++t) acc += w[t + 5] * tmp[(size_t)reflect_index(j + t, ny) * nx + i];
            out[(size_t)j * nx + i] = acc;
        }
    free(tmp);
}

int gor_loss(int w, int h, const double* x, const double* y, double lambda, double dssim_scale,
             double* dl_di, double* loss) {
    if (w < 1 || h < 1) return fail(GPK_ERR_INVALID_ARGUMENT, -1, "photometric_loss: image shape mismatch");
    const size_t n = (size_t)w * h;
    const double inv_n = 1.0 / (double)n;
    double l1 = 0.0;
    for (size_t i = 0; i < n; ++i) { /* loss.hpp:22-27 */
        const double d = x[i] - y[i];
        l1 += fabs(d);
        dl_di[i] = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n;
    }
    l1 *= inv_n;
    if (lambda == 0.0) {
        *loss = l1;
        return ok();
    }
    double win[11], sum = 0.0; /* metrics.hpp:66-75 */
    for (int t = -5; t <= 5; ++t) {
        win[t + 5] = exp(-0.5 * t * t / (1.5 * 1.5));
        sum += win[t + 5];
    }
    for (int t = 0; t < 11; ++t) win[t] /= sum;
    double* buf = (double*)malloc(sizeof(double) * n * 12);
    double *xx = buf, *xy = buf + n, *yy = buf + 2 * n, *mx = buf + 3 * n, *my = buf + 4 * n;
    double *m2 = buf + 5 * n, *m12 = buf + 6 * n, *m2y = buf + 7 * n;
    double *g1 = buf + 8 * n, *g2 = buf + 9 * n, *g3 = buf + 10 * n, *tmp = buf + 11 * n;
    for (size_t i = 0; i < n; ++i) {
        xx[i] = x[i] * x[i];
        xy[i] = x[i] * y[i];
        yy[i] = y[i] * y[i];
    }
    conv2(x, mx, w, h, win);
    conv2(y, my, w, h, win);
    conv2(xx, m2, w, h, win);
    conv2(xy, m12, w, h, win);
    conv2(yy, m2y, w, h, win);
    const double c1 = 1e-4, c2 = 9e-4; /* metrics.hpp:155-156 */
    double mean = 0.0;
    for (size_t i = 0; i < n; ++i) { /* metrics.hpp:198-215 */
        const double ux = mx[i], uy = my[i];
        const double vx = m2[i] - ux * ux, vy = m2y[i] - uy * uy, vxy = m12[i] - ux * uy;
        const double a1 = 2.0 * ux * uy + c1, a2 = 2.0 * vxy + c2;
        const double b1 = ux * ux + uy * uy + c1, b2 = vx + vy + c2;
        const double s = (a1 * a2) / (b1 * b2);
        mean += s;
        const double inv_b1b2 = 1.0 / (b1 * b2);
        g1[i] = (2.0 * uy * a2 * inv_b1b2 - 2.0 * ux * s / b1 + 2.0 * ux * s / b2 -
                 2.0 * uy * a1 * inv_b1b2) * inv_n;
        g2[i] = (-s / b2) * inv_n;
        g3[i] = (2.0 * a1 * inv_b1b2) * inv_n;
    }
    mean *= inv_n;
    conv2(g1, mx, w, h, win); /* metrics.hpp:218-223 */
    conv2(g2, my, w, h, win);
    conv2(g3, tmp, w, h, win);
    for (size_t i = 0; i < n; ++i) {
        const double gs = mx[i] + 2.0 * x[i] * my[i] + y[i] * tmp[i];
        dl_di[i] += lambda * dssim_scale * (-gs);
    }
    *loss = l1 + lambda * dssim_scale * (1.0 - mean);
    free(buf);
    return ok();
}

/* ---- optimize.hpp:184-221: Adam -------------------------------------------- */
static double adam_update(double* m, double* v, double g, double lr, const gpk_adam_hparams* hp,
                          double bc1, double bc2) {
    *m = hp->beta1 * *m + (1.0 - hp->beta1) * g;
    *v = hp->beta2 * *v + (1.0 - hp->beta2) * g * g;
    return lr * (*m / bc1) / (sqrt(*v / bc2) + hp->eps);
}

int gor_adam_step(uint64_t n, double* rec, const gpk_bounds* bbox, const double* grads, double* m,
                  double* v, int64_t* step, const gpk_learning_rates* lrs,
                  const gpk_adam_hparams* hp_in) {
    const gpk_adam_hparams def = {0.9, 0.999, 1e-8};
    const gpk_adam_hparams* hp = hp_in ? hp_in : &def;
    *step += 1;
    const double bc1 = 1.0 - pow(hp->beta1, (double)*step);
    const double bc2 = 1.0 - pow(hp->beta2, (double)*step);
    for (uint64_t i = 0; i < n; ++i) {
        double* g = rec + 11 * i;
        const double* d = grads + 11 * i;
        double* mi = m + 11 * i;
        double* vi = v + 11 * i;
        double mu[3] = {g[0], g[1], g[2]};
        for (int k = 0; k < 3; ++k) {
            mu[k] -= adam_update(&mi[k], &vi[k], d[k], lrs->position, hp, bc1, bc2);
            g[3 + k] -= adam_update(&mi[3 + k], &vi[3 + k], d[3 + k], lrs->scale, hp, bc1, bc2);
        }
        for (int k = 0; k < 3; ++k) /* Bounds::clamp, core.hpp:58-62 */
            g[k] = fmin(bbox->max[k], fmax(bbox->min[k], mu[k]));
        for (int k = 0; k < 4; ++k)
            g[6 + k] -= adam_update(&mi[6 + k], &vi[6 + k], d[6 + k], lrs->rotation, hp, bc1, bc2);
        const double qn = sqrt(g[6] * g[6] + g[7] * g[7] + g[8] * g[8] + g[9] * g[9]);
        if (qn > 0.0)
            for (int k = 0; k < 4; ++k) g[6 + k] = g[6 + k] * (1.0 / qn);
        g[10] -= adam_update(&mi[10], &vi[10], d[10], lrs->opacity, hp, bc1, bc2);
    }
    return ok();
}

/* ---- voxelize.hpp ------------------------------------------------------------ */
typedef struct {
    uint32_t index;
    double alpha;
    v3 mu;
    m3 sinv;
    int lo[3], hi[3];
} vprim_t;

static int vcfg_validate(const gpk_voxelizer_config* c) { /* voxelize.hpp:24-37 */
    if (c->dims[0] < 1 || c->dims[1] < 1 || c->dims[2] < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, -1, "VoxelizerConfig: dims must be >= 1");
    if (c->tile_dims[0] < 1 || c->tile_dims[1] < 1 || c->tile_dims[2] < 1)
        return fail(GPK_ERR_INVALID_ARGUMENT, -1, "VoxelizerConfig: tile_dims must be >= 1");
    if (!(c->support_sigmas > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT, -1, "VoxelizerConfig: support_sigmas must be > 0");
    if (!(c->spacing[0] > 0.0) || !(c->spacing[1] > 0.0) || !(c->spacing[2] > 0.0))
        return fail(GPK_ERR_INVALID_ARGUMENT, -1, "VoxelizerConfig: spacing must be positive");
    const uint64_t vox = (uint64_t)c->dims[0] * (uint64_t)c->dims[1] * (uint64_t)c->dims[2];
    if (vox > (1ull << 31)) return fail(GPK_ERR_INVALID_ARGUMENT, -1, "VoxelizerConfig: refusing > 2^31 voxels");
    return GPK_OK;
}

/* voxelize.hpp:52-84 */
static int vprims(uint64_t n, const double* rec, const gpk_voxelizer_config* c, vprim_t** out,
                  uint64_t* count) {
    vprim_t* P = (vprim_t*)malloc(sizeof(vprim_t) * (n ? n : 1));
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double* g = rec + 11 * i;
        vprim_t p;
        p.index = (uint32_t)i;
        p.alpha = alpha_act(g[10]);
        p.mu.x = g[0];
        p.mu.y = g[1];
        p.mu.z = g[2];
        m3 sigma;
        if (cov_from_scale_rot(g, c->scale_modifier, &sigma)) {
            free(P);
            return fail(GPK_ERR_INVALID_ARGUMENT, (int64_t)i, "invalid primitive");
        }
        if (invert_cov(sigma, &p.sinv)) {
            free(P);
            return fail(GPK_ERR_DEGENERATE_COVARIANCE, (int64_t)i, "invert_covariance");
        }
        int inside = 1;
        for (int d = 0; d < 3; ++d) {
            const double half = c->support_sigmas * sqrt(sigma.m[d][d]);
            const double md = v3_get(p.mu, d);
            const double lo_w = md - half, hi_w = md + half;
            const double o = c->origin[d], s = c->spacing[d];
            int v = trunc_int(ceil((lo_w - o) / s));
            p.lo[d] = v > 0 ? v : 0;
            v = trunc_int(floor((hi_w - o) / s));
            p.hi[d] = v < c->dims[d] - 1 ? v : c->dims[d] - 1;
            if (p.lo[d] > p.hi[d]) inside = 0;
        }
        if (!inside) continue;
        P[k++] = p;
    }
    *out = P;
    *count = k;
    return GPK_OK;
}

/* voxelize.hpp:86-105 as CSR */
static uint64_t vtiles(const gpk_voxelizer_config* c, const vprim_t* P, uint64_t S, int nt[3],
                       uint32_t** off_out, uint32_t** ent_out) {
    for (int d = 0; d < 3; ++d) nt[d] = (c->dims[d] + c->tile_dims[d] - 1) / c->tile_dims[d];
    const uint64_t T = (uint64_t)nt[0] * nt[1] * nt[2];
    uint32_t* off = (uint32_t*)calloc(T + 1, sizeof(uint32_t));
    for (int pass = 0; pass < 2; ++pass) {
        uint32_t* cur = NULL;
        uint32_t* ent = NULL;
        if (pass == 1) {
            for (uint64_t t = 0; t < T; ++t) off[t + 1] += off[t];
            cur = (uint32_t*)malloc(sizeof(uint32_t) * (T + 1));
            memcpy(cur, off, sizeof(uint32_t) * (T + 1));
            ent = (uint32_t*)malloc(sizeof(uint32_t) * (off[T] ? off[T] : 1));
        }
        for (uint64_t pi = 0; pi < S; ++pi) {
            const vprim_t* p = &P[pi];
            for (int tz = p->lo[2] / c->tile_dims[2]; tz <= p->hi[2] / c->tile_dims[2]; ++tz)
                for (int ty = p->lo[1] / c->tile_dims[1]; ty <= p->hi[1] / c->tile_dims[1]; ++ty)
                    for (int tx = p->lo[0] / c->tile_dims[0]; tx <= p->hi[0] / c->tile_dims[0]; ++tx) {
                        const uint64_t t = ((uint64_t)tz * nt[1] + ty) * nt[0] + tx;
                        if (pass == 0) off[t + 1]++;
                        else ent[cur[t]++] = (uint32_t)pi;
                    }
        }
        if (pass == 1) {
            free(cur);
            *ent_out = ent;
        }
    }
    *off_out = off;
    return T;
}

int gor_voxel_tiles(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg,
                    uint32_t* offsets, uint32_t* entries, uint64_t capacity, uint64_t* total,
                    uint64_t* tiles) {
    if (vcfg_validate(cfg)) return GPK_ERR_INVALID_ARGUMENT;
    vprim_t* P;
    uint64_t S;
    int st = vprims(n, rec, cfg, &P, &S);
    if (st) return st;
    int nt[3];
    uint32_t *off, *ent;
    const uint64_t T = vtiles(cfg, P, S, nt, &off, &ent);
    *tiles = T;
    *total = off[T];
    if (offsets) memcpy(offsets, off, sizeof(uint32_t) * (T + 1));
    if (entries)
        for (uint32_t k = 0; k < off[T] && k < capacity; ++k) entries[k] = P[ent[k]].index;
    free(off);
    free(ent);
    free(P);
    return ok();
}

int gor_voxelize(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg, double* out) {
    if (vcfg_validate(cfg)) return GPK_ERR_INVALID_ARGUMENT;
    vprim_t* P;
    uint64_t S;
    int st = vprims(n, rec, cfg, &P, &S);
    if (st) return st;
    const int X = cfg->dims[0], Y = cfg->dims[1], Z = cfg->dims[2];
    memset(out, 0, sizeof(double) * (size_t)X * Y * Z);
    int nt[3];
    uint32_t *off, *ent;
    const uint64_t T = vtiles(cfg, P, S, nt, &off, &ent);
    for (uint64_t t = 0; t < T; ++t) { /* voxelize.hpp:126-145 */
        const int tx = (int)(t % nt[0]), ty = (int)((t / nt[0]) % nt[1]), tz = (int)(t / ((uint64_t)nt[0] * nt[1]));
        const int x0 = tx * cfg->tile_dims[0], x1 = X < x0 + cfg->tile_dims[0] ? X : x0 + cfg->tile_dims[0];
        const int y0 = ty * cfg->tile_dims[1], y1 = Y < y0 + cfg->tile_dims[1] ? Y : y0 + cfg->tile_dims[1];
        const int z0 = tz * cfg->tile_dims[2], z1 = Z < z0 + cfg->tile_dims[2] ? Z : z0 + cfg->tile_dims[2];
        for (uint32_t k = off[t]; k < off[t + 1]; ++k) {
            const vprim_t* p = &P[ent[k]];
            for (int kz = z0; kz < z1; ++kz)
                for (int j = y0; j < y1; ++j)
                    for (int i = x0; i < x1; ++i) {
                        const v3 d = {cfg->origin[0] + i * cfg->spacing[0] - p->mu.x,
                                      cfg->origin[1] + j * cfg->spacing[1] - p->mu.y,
                                      cfg->origin[2] + kz * cfg->spacing[2] - p->mu.z};
                        const double q = v3_dot(d, m3_mulv(p->sinv, d));
                        out[((size_t)kz * Y + j) * X + i] += p->alpha * exp(-0.5 * q);
                    }
        }
    }
    for (size_t i = 0; i < (size_t)X * Y * Z; ++i) out[i] = fmax(0.0, out[i]); /* :146 */
    free(off);
    free(ent);
    free(P);
    return ok();
}

int gor_voxelize_backward(uint64_t n, const double* rec, const gpk_voxelizer_config* cfg,
                          const double* dl_dv, double* grads) {
    if (vcfg_validate(cfg)) return GPK_ERR_INVALID_ARGUMENT;
    vprim_t* P;
    uint64_t S;
    int st = vprims(n, rec, cfg, &P, &S);
    if (st) return st;
    const int X = cfg->dims[0], Y = cfg->dims[1], Z = cfg->dims[2];
    int nt[3];
    uint32_t *off, *ent;
    const uint64_t T = vtiles(cfg, P, S, nt, &off, &ent);
    typedef struct { double da; v3 dmu; m3 dsi; } vacc_t;
    vacc_t* part = (vacc_t*)calloc(off[T] ? off[T] : 1, sizeof(vacc_t));
    for (uint64_t t = 0; t < T; ++t) { /* voxelize.hpp:175-205 */
        const int tx = (int)(t % nt[0]), ty = (int)((t / nt[0]) % nt[1]), tz = (int)(t / ((uint64_t)nt[0] * nt[1]));
        const int x0 = tx * cfg->tile_dims[0], x1 = X < x0 + cfg->tile_dims[0] ? X : x0 + cfg->tile_dims[0];
        const int y0 = ty * cfg->tile_dims[1], y1 = Y < y0 + cfg->tile_dims[1] ? Y : y0 + cfg->tile_dims[1];
        const int z0 = tz * cfg->tile_dims[2], z1 = Z < z0 + cfg->tile_dims[2] ? Z : z0 + cfg->tile_dims[2];
        for (uint32_t k = off[t]; k < off[t + 1]; ++k) {
            const vprim_t* p = &P[ent[k]];
            vacc_t a;
            memset(&a, 0, sizeof a);
            for (int kz = z0; kz < z1; ++kz)
                for (int j = y0; j < y1; ++j)
                    for (int i = x0; i < x1; ++i) {
                        const double g = dl_dv[((size_t)kz * Y + j) * X + i];
                        if (g == 0.0) continue;
                        const v3 d = {cfg->origin[0] + i * cfg->spacing[0] - p->mu.x,
                                      cfg->origin[1] + j * cfg->spacing[1] - p->mu.y,
                                      cfg->origin[2] + kz * cfg->spacing[2] - p->mu.z};
                        const v3 sd = m3_mulv(p->sinv, d);
                        const double e = exp(-0.5 * v3_dot(d, sd));
                        a.da += g * e;
                        const double w = g * p->alpha * e;
                        a.dmu.x += sd.x * w;
                        a.dmu.y += sd.y * w;
                        a.dmu.z += sd.z * w;
                        for (int r = 0; r < 3; ++r)
                            for (int c = 0; c < 3; ++c)
                                a.dsi.m[r][c] += w * (-0.5) * v3_get(d, r) * v3_get(d, c);
                    }
            part[k] = a;
        }
    }
    vacc_t* tot = (vacc_t*)calloc(S ? S : 1, sizeof(vacc_t));
    for (uint32_t k = 0; k < off[T]; ++k) { /* :207-215 */
        vacc_t* d = &tot[ent[k]];
        d->da += part[k].da;
        d->dmu.x += part[k].dmu.x;
        d->dmu.y += part[k].dmu.y;
        d->dmu.z += part[k].dmu.z;
        d->dsi = m3_add(d->dsi, part[k].dsi);
    }
    memset(grads, 0, sizeof(double) * 11 * n);
    for (uint64_t pi = 0; pi < S; ++pi) { /* :218-232 */
        const vprim_t* p = &P[pi];
        const vacc_t* a = &tot[pi];
        m3 dsig = m3_scale(m3_mul(m3_mul(p->sinv, a->dsi), p->sinv), -1.0);
        dsig = m3_scale(m3_add(dsig, m3_t(dsig)), 0.5);
        double d_ls[3], d_q[4];
        const double* gp = rec + 11 * p->index;
        chain_world(gp, dsig, cfg->scale_modifier, d_ls, d_q);
        double* o = grads + 11 * (size_t)p->index;
        o[0] = a->dmu.x; o[1] = a->dmu.y; o[2] = a->dmu.z;
        o[3] = d_ls[0]; o[4] = d_ls[1]; o[5] = d_ls[2];
        o[6] = d_q[0]; o[7] = d_q[1]; o[8] = d_q[2]; o[9] = d_q[3];
        o[10] = a->da * (p->alpha * (1.0 - p->alpha));
    }
    free(tot);
    free(part);
    free(off);
    free(ent);
    free(P);
    for (uint64_t i = 0; i < n; ++i) { /* :234-238 */
        const double* o = grads + 11 * i;
        if (!isfinite(o[10] + o[0] + o[3] + o[6])) {
            char m[96];
            snprintf(m, sizeof m, "voxelize_backward: non-finite gradient for primitive %llu",
                     (unsigned long long)i);
            return fail(GPK_ERR_NUMERIC_FAILURE, (int64_t)i, m);
        }
    }
    return ok();
}
