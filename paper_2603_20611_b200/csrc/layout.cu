// layout.cu — record (AoS) <-> plane (SoA) transposes on the device, for the
// parameter / gradient / moment transfers across the C-ABI (gpk_set_gaussians,
// gpk_get_gaussians, gpk_get_gradients, Adam state, checkpoints).
//
// The host side speaks the reference's checkpoint record: 11 f32 per
// primitive (mu xyz, log-scale xyz, quat wxyz, raw alpha; checkpoint.hpp:14-16);
// the session keeps 11 planes of stride cap. A CTA moves 256 records
// (11 KB) with coalesced 4 B loads of the contiguous record block into shared
// memory and coalesced stores of 11 plane runs (and the reverse), so the
// transpose runs at copy bandwidth instead of the host loop's ~1 GB/s.
#include "common.cuh"

namespace gpk {

namespace {

constexpr int kLayoutThreads = 256;
constexpr int kRec = 11;

__global__ void __launch_bounds__(kLayoutThreads) k_records_to_planes(const float* __restrict__ rec, uint64_t n,
                                                                      float* __restrict__ planes, uint64_t cap) {
    __shared__ float tile[kLayoutThreads * kRec + 1];
    const uint64_t base = (uint64_t)blockIdx.x * kLayoutThreads;
    const uint64_t cnt = min((uint64_t)kLayoutThreads, n - base);
    const float* src = rec + base * kRec;
    for (uint32_t t = threadIdx.x; t < cnt * kRec; t += kLayoutThreads) tile[t] = src[t];
    __syncthreads();
    if (threadIdx.x < cnt) {
#pragma unroll
        for (int k = 0; k < kRec; ++k) planes[k * cap + base + threadIdx.x] = tile[threadIdx.x * kRec + k];
    }
}

__global__ void __launch_bounds__(kLayoutThreads) k_planes_to_records(const float* __restrict__ planes, uint64_t cap,
                                                                      uint64_t n, float* __restrict__ rec) {
    __shared__ float tile[kLayoutThreads * kRec + 1];
    const uint64_t base = (uint64_t)blockIdx.x * kLayoutThreads;
    const uint64_t cnt = min((uint64_t)kLayoutThreads, n - base);
    if (threadIdx.x < cnt) {
#pragma unroll
        for (int k = 0; k < kRec; ++k) tile[threadIdx.x * kRec + k] = planes[k * cap + base + threadIdx.x];
    }
    __syncthreads();
    float* dst = rec + base * kRec;
    for (uint32_t t = threadIdx.x; t < cnt * kRec; t += kLayoutThreads) dst[t] = tile[t];
}

}  // namespace

void launch_records_to_planes(const float* rec, uint64_t n, float* planes, uint64_t cap, cudaStream_t st) {
    if (n) k_records_to_planes<<<(unsigned)((n + kLayoutThreads - 1) / kLayoutThreads), kLayoutThreads, 0, st>>>(
        rec, n, planes, cap);
}

void launch_planes_to_records(const float* planes, uint64_t cap, uint64_t n, float* rec, cudaStream_t st) {
    if (n) k_planes_to_records<<<(unsigned)((n + kLayoutThreads - 1) / kLayoutThreads), kLayoutThreads, 0, st>>>(
        planes, cap, n, rec);
}

}  // namespace gpk
