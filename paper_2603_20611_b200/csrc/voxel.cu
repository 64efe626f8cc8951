// voxel.cu — 3-D voxelizer evaluation and backward (voxelize.hpp:113-240).
//
// Forward (voxelize, voxelize.hpp:126-146): one CTA per voxel tile. The
// tile's primitives (already in ascending set order from the stable radix
// sort) are staged through shared memory in batches; each thread owns one
// x-row segment (a whole 8-voxel row of an 8^3 tile, 64 threads per tile;
// 16-voxel segments for other tile widths) and, per primitive, evaluates
//     alpha * exp(-1/2 d^T Sigma^-1 d) = 2^(q(dx)),  q(dx) = (a00 dx + B) dx + C
// where B, C are per-(row, primitive) constants and log2(alpha) and
// -1/2*log2(e) are folded into C and the a's: two FMAs + one MUFU.EX2 + one
// FADD per voxel evaluation. Every voxel of every touched tile is evaluated,
// as in the reference (no clipping to the support box), accumulated in list
// order, and clamped at 0 on the write (voxelize.hpp:146).
//
// Backward (voxelize.hpp:175-205): one warp per (tile, primitive) pair; lanes
// own voxel rows, accumulate the 10 per-pair sums (d alpha, d mu, symmetric
// d Sigma^-1) and combine them with a fixed xor-shuffle tree; the pair's sums
// go to its pre-sort position so k_vchain merges a primitive's tiles in tile
// order (voxelize.hpp:207-215).
#include "common.cuh"

namespace gpk {

namespace {

constexpr float kNegHalfLog2e = -0.72134752044448170368f;
constexpr int kVoxBatch = 128;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


struct TileBox {
    int x0, y0, z0, nx, ny, nz;  // voxel origin and extent (clipped to the grid)
    int tx, ty, tz;
};

__device__ __forceinline__ TileBox tile_box(const VoxArgs& v, unsigned t) {
    TileBox b;
    b.tx = (int)(t % (unsigned)v.ntiles[0]);
    b.ty = (int)((t / (unsigned)v.ntiles[0]) % (unsigned)v.ntiles[1]);
    b.tz = (int)(t / ((unsigned)v.ntiles[0] * (unsigned)v.ntiles[1]));
    b.x0 = b.tx * v.tile[0];
    b.y0 = b.ty * v.tile[1];
    b.z0 = b.tz * v.tile[2];
    b.nx = min(v.dims[0], b.x0 + v.tile[0]) - b.x0;
    b.ny = min(v.dims[1], b.y0 + v.tile[1]) - b.y0;
    b.nz = min(v.dims[2], b.z0 + v.tile[2]) - b.z0;
    return b;
}

// SEG voxels of an x-row per thread, THREADS per CTA: (8, 64) for 8-wide
// tiles (every thread owns one full row of the 8x8x8 tile: no idle lanes, no
// evaluations past the row), (16, 128) otherwise.
template <int SEG, int THREADS>
__global__ void __launch_bounds__(THREADS) k_veval(const VoxEvalLaunch a) {
    __shared__ float4 s_p[kVoxBatch][3];  // {ox, oy, oz, log2a}, {a00, a11, a22, 2a01}, {2a02, 2a12}
    __shared__ unsigned s_range[2];
    const int tid = threadIdx.x;
    const unsigned t = blockIdx.x;
    const TileBox b = tile_box(a.v, t);
    if (tid < 2) s_range[tid] = __ldcg(&a.tile_start[t + tid]);  // (k_key_starts)
    // voxel centre of the tile origin (voxel_center, core.hpp:136-138), fp64
    const double wx0 = a.v.origin[0] + b.x0 * a.v.spacing[0];
    const double wy0 = a.v.origin[1] + b.y0 * a.v.spacing[1];
    const double wz0 = a.v.origin[2] + b.z0 * a.v.spacing[2];
    const float sx = (float)a.v.spacing[0], sy = (float)a.v.spacing[1], sz = (float)a.v.spacing[2];
    __syncthreads();
    const unsigned start = s_range[0], end = s_range[1];
    const int nseg = (b.nx + SEG - 1) / SEG;
    const int nitems = b.ny * b.nz * nseg;

    for (int ig = 0; ig < nitems; ig += THREADS) {
        const int it = ig + tid;
        const bool active = it < nitems;
        const int seg = active ? it % nseg : 0, row = active ? it / nseg : 0;
        const int ly = row % b.ny, lz = row / b.ny;
        const int lx0 = seg * SEG;
        const int len = active ? min(SEG, b.nx - lx0) : 0;
        float acc[SEG];
#pragma unroll
        for (int j = 0; j < SEG; ++j) acc[j] = 0.f;
        const float fy = ly * sy, fz = lz * sz;
        float fxs[SEG];
#pragma unroll
        for (int j = 0; j < SEG; ++j) fxs[j] = (float)(lx0 + j) * sx;
        for (unsigned bb = start; bb < end; bb += kVoxBatch) {
            const unsigned nb = min((unsigned)kVoxBatch, end - bb);
            __syncthreads();
            for (unsigned q = tid; q < nb; q += THREADS) {
                const VoxRecord r = a.records[a.vals[bb + q]];
                s_p[q][0] = make_float4((float)(wx0 - (double)r.mu[0]), (float)(wy0 - (double)r.mu[1]),
                                        (float)(wz0 - (double)r.mu[2]), r.log2a);
                s_p[q][1] = make_float4(r.a[0], r.a[1], r.a[2], r.a[3]);
                s_p[q][2] = make_float4(r.a[4], r.a[5], 0.f, 0.f);
            }
            __syncthreads();
            if (active) {
                for (unsigned k = 0; k < nb; ++k) {
                    const float4 p0 = s_p[k][0], p1 = s_p[k][1], p2 = s_p[k][2];
                    const float dy = fy + p0.y, dz = fz + p0.z;
                    const float B = fmaf(p1.w, dy, p2.x * dz);
                    const float Cc = fmaf(dy, fmaf(p1.y, dy, p2.y * dz), fmaf(p1.z * dz, dz, p0.w));
                    // two voxels of the row per packed fp32 pair (FFMA2; x + y as
                    // fma(1, x, y): each lane rounds exactly like the scalar code)
#pragma unroll
                    for (int j = 0; j < SEG; j += 2) {
                        const f32x2 dx = ffma2(f2(1.f, 1.f), f2(fxs[j], fxs[j + 1]), f2(p0.x, p0.x));
                        const float2 q = f2_unpack(ffma2(ffma2(f2(p1.x, p1.x), dx, f2(B, B)), dx, f2(Cc, Cc)));
                        const float2 s2 = f2_unpack(
                            ffma2(f2(1.f, 1.f), f2(ex2_approx(q.x), ex2_approx(q.y)), f2(acc[j], acc[j + 1])));
                        acc[j] = s2.x;
                        acc[j + 1] = s2.y;
                    }
                }
            }
        }
        if (active) {
            const size_t X = (size_t)a.v.dims[0], Y = (size_t)a.v.dims[1];
            float* out = a.volume + ((size_t)(b.z0 + lz) * Y + (b.y0 + ly)) * X + (b.x0 + lx0);
#pragma unroll
            for (int j = 0; j < SEG; ++j)
                if (j < len) out[j] = fmaxf(0.f, acc[j]);
        }
    }
}

__global__ void __launch_bounds__(128) k_vbwd(const VoxEvalLaunch a) {
    extern __shared__ float s_dl[];  // the tile's dL/dV, nx*ny*nz
    __shared__ unsigned s_range[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned t = blockIdx.x;
    const TileBox b = tile_box(a.v, t);
    if (tid < 2) s_range[tid] = __ldcg(&a.tile_start[t + tid]);  // (k_key_starts)
    const int nvox = b.nx * b.ny * b.nz;
    const size_t X = (size_t)a.v.dims[0], Y = (size_t)a.v.dims[1];
    if (!a.dl_global) {
        for (int q = tid; q < nvox; q += blockDim.x) {
            const int lx = q % b.nx, ly = (q / b.nx) % b.ny, lz = q / (b.nx * b.ny);
            s_dl[q] = a.dl_dv[((size_t)(b.z0 + lz) * Y + (b.y0 + ly)) * X + (b.x0 + lx)];
        }
    }
    const double wx0 = a.v.origin[0] + b.x0 * a.v.spacing[0];
    const double wy0 = a.v.origin[1] + b.y0 * a.v.spacing[1];
    const double wz0 = a.v.origin[2] + b.z0 * a.v.spacing[2];
    const float sx = (float)a.v.spacing[0], sy = (float)a.v.spacing[1], sz = (float)a.v.spacing[2];
    constexpr float kInvK = 1.f / kNegHalfLog2e;
    __syncthreads();
    const unsigned start = s_range[0], end = s_range[1];
    const int nrows = b.ny * b.nz;
    const int nwarps = blockDim.x >> 5;

    for (unsigned p = start + warp; p < end; p += nwarps) {
        const VoxRecord r = a.records[a.vals[p]];
        const float ox = (float)(wx0 - (double)r.mu[0]), oy = (float)(wy0 - (double)r.mu[1]),
                    oz = (float)(wz0 - (double)r.mu[2]);
        // true Sigma^-1 from the prescaled record
        const float A00 = r.a[0] * kInvK, A11 = r.a[1] * kInvK, A22 = r.a[2] * kInvK;
        const float A01 = 0.5f * r.a[3] * kInvK, A02 = 0.5f * r.a[4] * kInvK, A12 = 0.5f * r.a[5] * kInvK;
        const float alpha = exp2f(r.log2a);
        float s[10];
#pragma unroll
        for (int j = 0; j < 10; ++j) s[j] = 0.f;
        for (int row = lane; row < nrows; row += 32) {
            const int ly = row % b.ny, lz = row / b.ny;
            const float dy = fmaf((float)ly, sy, oy), dz = fmaf((float)lz, sz, oz);
            const float* dl_row = a.dl_global ? a.dl_dv + ((size_t)(b.z0 + lz) * Y + (b.y0 + ly)) * X + b.x0
                                              : s_dl + row * b.nx;
            for (int lx = 0; lx < b.nx; ++lx) {
                const float g = dl_row[lx];
                if (g == 0.f) continue;  // voxelize.hpp:192
                const float dx = fmaf((float)lx, sx, ox);
                const float sdx = fmaf(A00, dx, fmaf(A01, dy, A02 * dz));
                const float sdy = fmaf(A01, dx, fmaf(A11, dy, A12 * dz));
                const float sdz = fmaf(A02, dx, fmaf(A12, dy, A22 * dz));
                const float e = ex2_approx(kNegHalfLog2e * fmaf(dx, sdx, fmaf(dy, sdy, dz * sdz)));
                s[0] = fmaf(g, e, s[0]);
                const float w = g * alpha * e;
                s[1] = fmaf(sdx, w, s[1]);
                s[2] = fmaf(sdy, w, s[2]);
                s[3] = fmaf(sdz, w, s[3]);
                const float hw = -0.5f * w;
                s[4] = fmaf(hw * dx, dx, s[4]);
                s[5] = fmaf(hw * dy, dy, s[5]);
                s[6] = fmaf(hw * dz, dz, s[6]);
                s[7] = fmaf(hw * dx, dy, s[7]);
                s[8] = fmaf(hw * dx, dz, s[8]);
                s[9] = fmaf(hw * dy, dz, s[9]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int j = 0; j < 10; ++j) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
        if (lane == 0) {
            int tx0 = r.lo[0] / a.v.tile[0], ty0 = r.lo[1] / a.v.tile[1], tz0 = r.lo[2] / a.v.tile[2];
            const int ntx = r.hi[0] / a.v.tile[0] - tx0 + 1, nty = r.hi[1] / a.v.tile[1] - ty0 + 1;
            const unsigned pos = r.pair_base + (unsigned)(((b.tz - tz0) * nty + (b.ty - ty0)) * ntx + (b.tx - tx0));
            if (pos < a.pair_cap) {
                float* dst = a.partials + 10ull * pos;
#pragma unroll
                for (int j = 0; j < 10; ++j) dst[j] = s[j];
            }
        }
    }
}

}  // namespace

void launch_vox_eval(const VoxEvalLaunch& a, cudaStream_t st) {
    const unsigned tiles = (unsigned)a.v.ntiles[0] * a.v.ntiles[1] * a.v.ntiles[2];
    if (!tiles) return;
    if (a.v.tile[0] == 8) k_veval<8, 64><<<tiles, 64, 0, st>>>(a);
    else k_veval<16, 128><<<tiles, 128, 0, st>>>(a);
}

void launch_vox_bwd(const VoxEvalLaunch& a, cudaStream_t st) {
    const unsigned tiles = (unsigned)a.v.ntiles[0] * a.v.ntiles[1] * a.v.ntiles[2];
    const int smem = a.dl_global ? 0 : a.v.tile[0] * a.v.tile[1] * a.v.tile[2] * (int)sizeof(float);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_vbwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (tiles) k_vbwd<<<tiles, 128, smem, st>>>(a);
}

}  // namespace gpk
