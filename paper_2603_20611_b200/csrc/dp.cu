// dp.cu — the union-compacted gradient exchange of a data-parallel training
// step. Rank r renders slice poses[r] of the step;
// gradients are exactly zero outside the union of the step's survivors
// (grad_chain.hpp:12-22), so only the rows of that union cross NVLink:
//
//   1. every rank evaluates K_filter's certain-cull for ALL the step's poses in
//      its own cull pass (k_filter_multi, cull.cu): the union of the poses'
//      candidates (a superset of every rank's survivors) as 4 words per
//      128-Gaussian chunk — computed from identical parameters and poses, so
//      identical on every rank, with no collective;
//   2. k_union_scan + k_union_map turn it into a dense numbering: umap[i] =
//      1 + the row of Gaussian i (chunk-major, ascending index), 0 outside;
//   3. the rank's chain writes each survivor's 11 gradients into row umap[i]-1
//      of 11 row planes (zero elsewhere);
//   4. one grouped ncclAllReduce sums the planes' first `ucap` rows;
//   5. Adam (every rank, all N: momentum moves culled Gaussians,
//      optimize.hpp:202-220) reads the gradient of Gaussian i from its row —
//      identical inputs, identical replicas.
// Rows beyond the capacity `ucap` (host-sized: the all-reduce count) set an
// overflow flag: the Adam skips the step and the host grows the capacity.
#include "common.cuh"

namespace gpk {

namespace {

constexpr int kScanThreads = 1024;

// Exclusive prefix of the chunks' union counts (one CTA), the total M and the
// overflow flag (uctrl[0] = M, uctrl[1] = M > ucap).
__global__ void __launch_bounds__(kScanThreads) k_union_scan(const unsigned* __restrict__ words, unsigned nchunks,
                                                             unsigned* __restrict__ prefix, unsigned* uctrl,
                                                             uint64_t ucap) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_wsum[kScanThreads / 32];
    __shared__ unsigned s_carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (unsigned b0 = 0; b0 < nchunks; b0 += kScanThreads) {
        const unsigned b = b0 + tid;
        unsigned c = 0;
        if (b < nchunks) {
            const uint4 w = *reinterpret_cast<const uint4*>(words + 4ull * b);
            c = __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
        }
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        unsigned ex = s_carry + incl - c;
        for (int w = 0; w < warp; ++w) ex += s_wsum[w];
        if (b < nchunks) prefix[b] = ex;
        __syncthreads();
        if (tid == kScanThreads - 1) s_carry = ex + c;
        __syncthreads();
    }
    if (tid == 0) {
        uctrl[0] = s_carry;
        uctrl[1] = (uint64_t)s_carry > ucap ? 1u : 0u;
    }
}

// umap[i] for every Gaussian: 1 + its row (chunk prefix + rank among the
// chunk's union members in ascending index), 0 outside the union.
__global__ void __launch_bounds__(256) k_union_map(const unsigned* __restrict__ words,
                                                   const unsigned* __restrict__ prefix, uint32_t n,
                                                   uint32_t* __restrict__ umap) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned b = i / kFilterBlock, r = i % kFilterBlock;
    const unsigned l = r / kFilterItems, k = r % kFilterItems;  // lane l, item k of the chunk
    const uint4 w = *reinterpret_cast<const uint4*>(words + 4ull * b);
    const unsigned ww[4] = {w.x, w.y, w.z, w.w};
    const unsigned below = (1u << l) - 1u;
    unsigned rank = 0;
#pragma unroll
    for (int q = 0; q < kFilterItems; ++q) rank += __popc(ww[q] & below) + (q < (int)k ? (ww[q] >> l) & 1u : 0u);
    umap[i] = ((ww[k] >> l) & 1u) ? prefix[b] + rank + 1u : 0u;
}

// The union gradient of every Gaussian into the dense planes (full
// overwrite): the API's view of a data-parallel step's gradient.
__global__ void __launch_bounds__(256) k_union_to_dense(const uint32_t* __restrict__ umap,
                                                        const float* __restrict__ rows, uint64_t cap, uint32_t n,
                                                        uint64_t ucap, float* __restrict__ grads) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t m = umap[i];
#pragma unroll
    for (int k = 0; k < 11; ++k)
        grads[(uint64_t)k * cap + i] = (m && m - 1 < ucap) ? rows[(uint64_t)k * cap + m - 1] : 0.f;
}

}  // namespace

void launch_union_scan(const unsigned* words, unsigned nchunks, unsigned* prefix, unsigned* uctrl, uint64_t ucap,
                       cudaStream_t st) {
    launch_pdl(k_union_scan, dim3(1), dim3(kScanThreads), 0, st, words, nchunks, prefix, uctrl, ucap);
}

void launch_union_map(const unsigned* words, const unsigned* prefix, uint32_t n, uint32_t* umap, cudaStream_t st) {
    if (n) launch_pdl(k_union_map, dim3((n + 255) / 256), dim3(256), 0, st, words, prefix, n, umap);
}

void launch_union_to_dense(const uint32_t* umap, const float* rows, uint64_t cap, uint32_t n, uint64_t ucap,
                           float* grads, cudaStream_t st) {
    if (n) k_union_to_dense<<<(n + 255) / 256, 256, 0, st>>>(umap, rows, cap, n, ucap, grads);
}

}  // namespace gpk
