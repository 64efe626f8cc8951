// loss.cu — photometric_loss (loss.hpp:13-37) with ssim_with_gradient
// (metrics.hpp:187-225), the dL/dI producer of the training step.
//
// L = mean|I - T| + lambda * dssim_scale * (1 - mean SSIM), SSIM over an
// 11-tap separable Gaussian window (sigma 1.5, metrics.hpp:66-75) with
// symmetric reflection at the borders (metrics.hpp:77-83).
//
// Two tiled kernels, 32x32 outputs per CTA, inputs staged with a 5-pixel
// reflected halo in shared memory:
//   k_ssim_fwd : 5 windowed moments (separable: rows then columns) -> per-pixel
//                SSIM and its three partials g1 = dS/dmu_x, g2 = dS/dm2,
//                g3 = dS/dm12 (already / N); per-CTA sums of SSIM and |I - T|.
//   k_ssim_bwd : the window operator is self-adjoint, so dSSIM/dI =
//                W g1 + 2 I (W g2) + T (W g3) (metrics.hpp:218-223); fused with
//                the L1 sign term into dL/dI. The last CTA reduces the per-CTA
//                sums in a fixed order (deterministic loss).
// lambda == 0 takes the L1-only kernel (loss.hpp:29).
#include "common.cuh"

namespace gpk {

namespace {

constexpr int kT = 32, kR = 5, kH = kT + 2 * kR;  // tile, radius, haloed extent
constexpr double kC1 = 1e-4, kC2 = 9e-4;         // metrics.hpp:155-156
constexpr int kSsimThreads = 512;                // 2 output pixels per thread (column pairs)

__device__ __forceinline__ int reflect(int p, int n) {
    while (p < 0 || p >= n) {
        if (p < 0) p = -p - 1;
        if (p >= n) p = 2 * n - 1 - p;
    }
    return p;
}

// Last CTA: the loss from every CTA's partial sums (common.cuh loss_reduce).
__device__ __forceinline__ void finish_loss(const LossLaunch& a, bool with_ssim) {
    __shared__ unsigned s_last;
    __shared__ double s_red2[2 * 32];
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nblk = gridDim.x * gridDim.y;
        s_last = (ticket_acq_rel(a.done_ctr) == nblk - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!s_last) return;
    LossFinish f;
    f.partial = a.partial;
    f.nblk = gridDim.x * gridDim.y;
    f.with_ssim = with_ssim ? 1 : 0;
    f.inv_n = 1.0 / ((double)a.W * (double)a.H);
    f.lambda = a.lambda;
    f.dssim_scale = a.dssim_scale;
    f.loss = a.loss;
    f.loss_host = a.loss_host;
    loss_reduce(f, s_red2);
    if (threadIdx.x == 0) *a.done_ctr = 0;
}

__global__ void __launch_bounds__(256) k_l1_only(const LossLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ double s_red[16];
    const size_t n = (size_t)a.W * a.H;
    const float inv_n = (float)(1.0 / (double)n);
    double l1 = 0.0, dummy = 0.0;
    const unsigned nblk = gridDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)nblk * blockDim.x) {
        const float d = a.image[i] - a.target[i];
        l1 += fabs((double)d);
        a.dl_di[i] = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_n;
    }
    block_sum2(dummy, l1, s_red);
    if (threadIdx.x == 0) {
        a.partial[2 * blockIdx.x] = 0.0;
        a.partial[2 * blockIdx.x + 1] = l1;
    }
    finish_loss(a, false);
}

__global__ void __launch_bounds__(kSsimThreads) k_ssim_fwd(const LossLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    // (x, y) and the moment pairs interleaved, so the filters run on packed
    // fp32 pairs (FFMA2: two moments per instruction, each rounded as a scalar
    // FFMA)
    __shared__ float2 s_xy[kH][kH + 1];
    __shared__ float2 s_m1[kH][kT + 1];  // (W x, W y) along rows
    __shared__ float2 s_m2[kH][kT + 1];  // (W xx, W yy)
    __shared__ float s_m3[kH][kT + 1];   // W xy
    __shared__ double s_red[2 * 32];
    const int X0 = blockIdx.x * kT, Y0 = blockIdx.y * kT;
    const int W = a.W, H = a.H;
    {
        // every load of the haloed tile in flight at once (a load-store loop
        // would wait one global round trip per element); an interior tile's
        // halo needs no reflection: one uniform branch per CTA, each element's
        // row divided once and its shared offset (r * (kH + 1) + c = idx + r) kept
        constexpr int kPer = (kH * kH + kSsimThreads - 1) / kSsimThreads;
        float vx[kPer], vy[kPer];
        int soff[kPer];
        const bool inner = X0 >= kR && Y0 >= kR && X0 + kT + kR <= W && Y0 + kT + kR <= H;
        if (inner) {
            const size_t base = (size_t)(Y0 - kR) * W + (X0 - kR);
            const float* gx = a.image + base;
            const float* gy = a.target + base;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * kSsimThreads;
                const int r = idx / kH;
                soff[k] = idx + r;
                if (idx < kH * kH) {
                    const unsigned o = (unsigned)(r * W + (idx - r * kH));
                    vx[k] = gx[o];
                    vy[k] = gy[o];
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * kSsimThreads;
                const int r = idx / kH;
                soff[k] = idx + r;
                if (idx < kH * kH) {
                    const size_t o = (size_t)reflect(Y0 + r - kR, H) * W + reflect(X0 + (idx - r * kH) - kR, W);
                    vx[k] = a.image[o];
                    vy[k] = a.target[o];
                }
            }
        }
        float2* sxy = &s_xy[0][0];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (threadIdx.x + k * kSsimThreads < kH * kH) sxy[soff[k]] = make_float2(vx[k], vy[k]);
    }
    __syncthreads();
    // rows (axis 0 of conv_nd, metrics.hpp:112-116): a thread filters 4
    // consecutive outputs from 14 samples in registers (each output still sums
    // its 11 taps in order): per tap (W x, W y) by one FFMA2, the products
    // (w x, w y) by one FMUL2, (W xx, W yy) by one FFMA2 on them, W xy by FFMA
    for (int item = threadIdx.x; item < kH * (kT / 4); item += blockDim.x) {
        const int r = item / (kT / 4), c0 = (item % (kT / 4)) * 4;
        float2 xy[4 + 2 * kR];
#pragma unroll
        for (int t = 0; t < 4 + 2 * kR; ++t) xy[t] = s_xy[r][c0 + t];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            f32x2 h1 = f2(0.f, 0.f), h2 = h1;
            float h3 = 0.f;
#pragma unroll
            for (int t = 0; t < 2 * kR + 1; ++t) {
                const float w = a.w[t];
                const f32x2 v = f2(xy[o + t]);
                h1 = ffma2(f2(w, w), v, h1);
                const f32x2 wv = fmul2(f2(w, w), v);
                h2 = ffma2(wv, v, h2);
                h3 = fmaf(f2_unpack(wv).x, xy[o + t].y, h3);
            }
            s_m1[r][c0 + o] = f2_unpack(h1);
            s_m2[r][c0 + o] = f2_unpack(h2);
            s_m3[r][c0 + o] = h3;
        }
    }
    __syncthreads();
    const double inv_n = 1.0 / ((double)W * (double)H);
    double ssum = 0.0, l1 = 0.0;
    const size_t P = (size_t)W * H;
    // columns: a thread owns 2 vertically adjacent pixels (12 samples per moment)
    {
        const int c = threadIdx.x % kT, r0 = (threadIdx.x / kT) * 2;
        float m[2][5];
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            f32x2 a1 = f2(0.f, 0.f), a2 = a1;
            float a3 = 0.f;
#pragma unroll
            for (int t = 0; t < 2 * kR + 1; ++t) {
                const float w = a.w[t];
                a1 = ffma2(f2(w, w), f2(s_m1[r0 + o + t][c]), a1);
                a2 = ffma2(f2(w, w), f2(s_m2[r0 + o + t][c]), a2);
                a3 = fmaf(w, s_m3[r0 + o + t][c], a3);
            }
            const float2 u1 = f2_unpack(a1), u2 = f2_unpack(a2);
            m[o][0] = u1.x;
            m[o][1] = u1.y;
            m[o][2] = u2.x;
            m[o][3] = a3;
            m[o][4] = u2.y;
        }
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            const int r = r0 + o;
            const int i = X0 + c, j = Y0 + r;
            if (i >= W || j >= H) continue;
            // metrics.hpp:199-215, evaluated in double per pixel
            const double mx = m[o][0], my = m[o][1];
            const double vx = m[o][2] - mx * mx, vy = m[o][4] - my * my, vxy = m[o][3] - mx * my;
            const double a1 = 2.0 * mx * my + kC1, a2 = 2.0 * vxy + kC2;
            const double b1 = mx * mx + my * my + kC1, b2 = vx + vy + kC2;
            // one fp64 reciprocal instead of four divisions (metrics.hpp:205-215)
            const double inv_b1b2 = 1.0 / (b1 * b2);
            const double s = a1 * a2 * inv_b1b2;
            const double inv_b1 = b2 * inv_b1b2, inv_b2 = b1 * inv_b1b2;
            const double ds_dm2 = -s * inv_b2;
            const double ds_dm12 = 2.0 * a1 * inv_b1b2;
            const double ds_dm1 = 2.0 * my * a2 * inv_b1b2 - 2.0 * mx * s * inv_b1 + 2.0 * mx * s * inv_b2 -
                                  2.0 * my * a1 * inv_b1b2;
            const size_t off = (size_t)j * W + i;
            a.g[off] = (float)(ds_dm1 * inv_n);
            a.g[P + off] = (float)(ds_dm2 * inv_n);
            a.g[2 * P + off] = (float)(ds_dm12 * inv_n);
            ssum += s;
            const float2 px = s_xy[r + kR][c + kR];
            l1 += fabs((double)(px.x - px.y));
        }
    }
    block_sum2(ssum, l1, s_red);
    if (threadIdx.x == 0) {
        const unsigned b = blockIdx.y * gridDim.x + blockIdx.x;
        a.partial[2 * b] = ssum;
        a.partial[2 * b + 1] = l1;
    }
    if (a.finish_in_fwd) finish_loss(a, true);
}

__global__ void __launch_bounds__(256) k_ssim_bwd(const LossLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ float s_g[3][kH][kH + 1];
    __shared__ float s_h[3][kH][kT + 1];
    const int X0 = blockIdx.x * kT, Y0 = blockIdx.y * kT;
    const int W = a.W, H = a.H;
    const size_t P = (size_t)W * H;
    {
        // every load of the haloed tile in flight at once, then to shared (an
        // interior tile's halo needs no reflection: one uniform branch per CTA)
        constexpr int kPer = (kH * kH + 255) / 256;
        constexpr int kPlane = kH * (kH + 1);
        const bool inner = X0 >= kR && Y0 >= kR && X0 + kT + kR <= W && Y0 + kT + kR <= H;
        float v[3][kPer];
        int soff[kPer];  // r * (kH + 1) + c = idx + r
        if (inner) {
            const float* g = a.g + (size_t)(Y0 - kR) * W + (X0 - kR);
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * 256;
                const int r = idx / kH;
                soff[k] = idx + r;
                if (idx < kH * kH) {
                    const unsigned o = (unsigned)(r * W + (idx - r * kH));
                    v[0][k] = g[o];
                    v[1][k] = g[P + o];
                    v[2][k] = g[2 * P + o];
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int idx = threadIdx.x + k * 256;
                const int r = idx / kH;
                soff[k] = idx + r;
                if (idx < kH * kH) {
                    const size_t o = (size_t)reflect(Y0 + r - kR, H) * W + reflect(X0 + (idx - r * kH) - kR, W);
                    v[0][k] = a.g[o];
                    v[1][k] = a.g[P + o];
                    v[2][k] = a.g[2 * P + o];
                }
            }
        }
        float* sg = &s_g[0][0][0];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (threadIdx.x + k * 256 < kH * kH) {
                sg[soff[k]] = v[0][k];
                sg[kPlane + soff[k]] = v[1][k];
                sg[2 * kPlane + soff[k]] = v[2][k];
            }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kH * kT; idx += blockDim.x) {
        const int r = idx / kT, c = idx % kT;
        float h0 = 0.f, h1 = 0.f, h2 = 0.f;
#pragma unroll
        for (int t = 0; t < 2 * kR + 1; ++t) {
            const float w = a.w[t];
            h0 += w * s_g[0][r][c + t];
            h1 += w * s_g[1][r][c + t];
            h2 += w * s_g[2][r][c + t];
        }
        s_h[0][r][c] = h0;
        s_h[1][r][c] = h1;
        s_h[2][r][c] = h2;
    }
    __syncthreads();
    const float inv_n = (float)(1.0 / (double)P);
    const float k = (float)(a.lambda * a.dssim_scale);
    for (int idx = threadIdx.x; idx < kT * kT; idx += blockDim.x) {
        const int r = idx / kT, c = idx % kT;
        const int i = X0 + c, j = Y0 + r;
        if (i >= W || j >= H) continue;
        float A0 = 0.f, A1 = 0.f, A2 = 0.f;
#pragma unroll
        for (int t = 0; t < 2 * kR + 1; ++t) {
            const float w = a.w[t];
            A0 += w * s_h[0][r + t][c];
            A1 += w * s_h[1][r + t][c];
            A2 += w * s_h[2][r + t][c];
        }
        const size_t o = (size_t)j * W + i;
        const float x = a.image[o], y = a.target[o];
        const float gs = A0 + 2.f * x * A1 + y * A2;
        const float d = x - y;
        a.dl_di[o] = (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_n + k * (-gs);
    }
    finish_loss(a, true);
}

}  // namespace

void launch_loss_fwd_only(const LossLaunch& a, cudaStream_t st) {
    const dim3 grid((a.W + kT - 1) / kT, (a.H + kT - 1) / kT);
    launch_pdl(k_ssim_fwd, grid, dim3(kSsimThreads), 0, st, a);
}

void launch_loss(const LossLaunch& a, cudaStream_t st) {
    if (a.lambda == 0.0) {
        const size_t n = (size_t)a.W * a.H;
        const unsigned grid = (unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
        launch_pdl(k_l1_only, dim3(grid), dim3(256), 0, st, a);
        return;
    }
    const dim3 grid((a.W + kT - 1) / kT, (a.H + kT - 1) / kT);
    launch_pdl(k_ssim_fwd, dim3(grid), dim3(kSsimThreads), 0, st, a);
    launch_pdl(k_ssim_bwd, dim3(grid), dim3(256), 0, st, a);
}

unsigned loss_partial_blocks(int W, int H, double lambda) {
    if (lambda == 0.0) {
        const size_t n = (size_t)W * H;
        return (unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
    }
    return (unsigned)(((W + kT - 1) / kT) * ((H + kT - 1) / kT));
}

}  // namespace gpk
