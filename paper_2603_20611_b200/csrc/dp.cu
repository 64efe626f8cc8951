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
#include <algorithm>

#include "common.cuh"

namespace gpk {

namespace {

constexpr int kScanThreads = 1024;  // chunks per scan block

// Exclusive prefix of the chunks' union counts: CTA k scans chunks
// [1024 k, 1024 k + 1024) into prefix[] (relative to its block) and publishes
// its block total; the last CTA (ticket) turns the totals into block offsets,
// the total M and the overflow flag (uctrl[0] = M, uctrl[1] = M > ucap).
// k_union_map adds the block offset.
__global__ void __launch_bounds__(kScanThreads) k_union_scan(const unsigned* __restrict__ words, unsigned nchunks,
                                                             unsigned* __restrict__ prefix, unsigned* uctrl,
                                                             uint64_t ucap) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    __shared__ unsigned s_wsum[kScanThreads / 32];
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nblk = gridDim.x;
    unsigned* btot = prefix + nchunks;  // block totals, then block offsets
    unsigned* boff = btot + nblk;
    unsigned* ticket = uctrl + 2;
    const unsigned b = blockIdx.x * kScanThreads + tid;
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
    unsigned ex = incl - c;
    for (int w = 0; w < warp; ++w) ex += s_wsum[w];
    if (b < nchunks) prefix[b] = ex;
    if (tid == kScanThreads - 1) btot[blockIdx.x] = ex + c;
    __syncthreads();
    if (tid == 0) s_last = ticket_acq_rel(ticket) == nblk - 1;
    __syncthreads();
    if (!s_last) return;
    unsigned carry = 0;  // (block totals: a handful per million Gaussians)
    for (unsigned k0 = 0; k0 < nblk; k0 += kScanThreads) {
        const unsigned k = k0 + tid;
        const unsigned v = k < nblk ? __ldcg(&btot[k]) : 0u;
        unsigned in2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, in2, o);
            if (lane >= o) in2 += u;
        }
        __syncthreads();
        if (lane == 31) s_wsum[warp] = in2;
        __syncthreads();
        unsigned e2 = carry + in2 - v;
        for (int w = 0; w < warp; ++w) e2 += s_wsum[w];
        if (k < nblk) boff[k] = e2;
        unsigned tot = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) tot += s_wsum[w];
        carry += tot;
    }
    if (tid == 0) {
        uctrl[0] = carry;
        uctrl[1] = (uint64_t)carry > ucap ? 1u : 0u;
        *ticket = 0;
    }
}

// umap[i] for every Gaussian: 1 + its row (block offset + chunk prefix + rank
// among the chunk's union members in ascending index), 0 outside the union.
// One thread per (chunk, lane): the lane's 4 items in one 16 B store.
// The kernel also clears the rows the chain is about to fill (11 planes of
// stride cap, the first ucap rows), so the step needs no memset nodes.
__global__ void __launch_bounds__(256) k_union_map(const unsigned* __restrict__ words,
                                                   const unsigned* __restrict__ prefix, unsigned nchunks,
                                                   uint32_t* __restrict__ umap, float* __restrict__ rows,
                                                   uint64_t cap, uint64_t ucap) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    {
        const uint64_t q4 = (ucap + 3) / 4;  // float4 per plane (cap is a multiple of 512)
        for (uint64_t e = t; e < 11 * q4; e += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t k = e / q4, j = e % q4;
            reinterpret_cast<float4*>(rows + k * cap)[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    const unsigned b = t / 32, l = t % 32;  // chunk b, lane l: items 4 l .. 4 l + 3
    if (b >= nchunks) return;
    const uint4 w = *reinterpret_cast<const uint4*>(words + 4ull * b);
    const unsigned ww[4] = {w.x, w.y, w.z, w.w};
    const unsigned nblk = (nchunks + kScanThreads - 1) / kScanThreads;
    const unsigned base = prefix[b] + prefix[nchunks + nblk + b / kScanThreads];
    const unsigned below = (1u << l) - 1u;
    unsigned rank = 0;
#pragma unroll
    for (int q = 0; q < kFilterItems; ++q) rank += __popc(ww[q] & below);
    uint32_t m[4];
#pragma unroll
    for (int k = 0; k < kFilterItems; ++k) {
        const bool in = (ww[k] >> l) & 1u;
        m[k] = in ? base + rank + 1u : 0u;
        rank += in ? 1u : 0u;
    }
    *reinterpret_cast<uint4*>(umap + (uint64_t)b * kFilterBlock + 4u * l) = make_uint4(m[0], m[1], m[2], m[3]);
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
    const unsigned nblk = std::max(1u, (nchunks + kScanThreads - 1) / kScanThreads);
    launch_pdl(k_union_scan, dim3(nblk), dim3(kScanThreads), 0, st, words, nchunks, prefix, uctrl, ucap);
}

void launch_union_map(const unsigned* words, const unsigned* prefix, uint32_t n, uint32_t* umap, float* rows,
                      uint64_t cap, uint64_t ucap, cudaStream_t st) {
    const unsigned nchunks = (n + kFilterBlock - 1) / kFilterBlock;
    if (n)
        launch_pdl(k_union_map, dim3((nchunks * 32 + 255) / 256), dim3(256), 0, st, words, prefix, nchunks, umap,
                   rows, cap, ucap);
}

void launch_union_to_dense(const uint32_t* umap, const float* rows, uint64_t cap, uint32_t n, uint64_t ucap,
                           float* grads, cudaStream_t st) {
    if (n) k_union_to_dense<<<(n + 255) / 256, 256, 0, st>>>(umap, rows, cap, n, ucap, grads);
}

}  // namespace gpk
