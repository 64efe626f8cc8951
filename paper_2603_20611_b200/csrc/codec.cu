// codec.cu — the codec's front half on the device: the
// stable Z-order sort (morton_sort, morton.hpp:15-48), the attribute
// quantization (quantize, quant.hpp:67-132) and the per-stream delta +
// zig-zag packing (detail::pack_deltas, container.hpp:136-156) that encode()
// (container.hpp:203-230) applies before LZMA. LZMA itself stays on the host.
//
// Built over the public C-ABI (the resident parameter planes, the session
// stream), like the fit driver:
//   k_morton_codes  per primitive: position normalized to the bbox, rounded
//                   to `bits` levels per axis (lround, quantize_unit), x/y/z
//                   bit-interleaved into a u64 code; value = set index.
//   radix sort      stable LSD over the 3*bits code bits, 8-bit digits:
//                   k_rs_hist (per-block digit counts) -> k_rs_scan (one CTA,
//                   digit-major exclusive scan) -> k_rs_scatter (in-block
//                   ranks from __match_any_sync + per-warp digit counts, items
//                   taken in index order, so equal codes keep their order —
//                   std::stable_sort's contract).
//   k_quant_check   log-scale min / max per axis (fp32-exact values, so
//                   atomics on their order-preserving integer images are
//                   exact) and the first non-finite / zero-quaternion index.
//   k_quantize      the four u32 streams, in sorted order, with the
//                   reference's fp64 expressions (--fmad=false).
//   k_pack_deltas   value minus the previous value of the same component,
//                   wrapped to [-2^(b-1), 2^(b-1)), zig-zag, ceil(b/8) bytes
//                   little endian — every element independent.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gpile_b200.h"
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 4;
constexpr int kBlockItems = kThreads * kItems;
constexpr int kDigits = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t quant_value(double u, int bits) {
    const double levels = (double)((1u << bits) - 1);
    const double c = fmin(1.0, fmax(0.0, u));
    return (uint32_t)lround(c * levels);
}

__global__ void k_morton_codes(const float* __restrict__ p, uint64_t cap, uint64_t n, gpk_bounds bb, int bits,
                               unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t q[3];
    for (int d = 0; d < 3; ++d) {
        const double ext = bb.max[d] - bb.min[d];
        const double rel = (double)p[d * cap + i] - bb.min[d];
        q[d] = quant_value(ext > 0.0 ? rel / ext : 0.0, bits);
    }
    unsigned long long code = 0;
    for (int b = 0; b < bits; ++b) {
        code |= (unsigned long long)((q[0] >> b) & 1u) << (3 * b);
        code |= (unsigned long long)((q[1] >> b) & 1u) << (3 * b + 1);
        code |= (unsigned long long)((q[2] >> b) & 1u) << (3 * b + 2);
    }
    keys[i] = code;
    vals[i] = (uint32_t)i;
}

__global__ void __launch_bounds__(kThreads) k_rs_hist(const unsigned long long* __restrict__ keys, uint64_t n,
                                                      int shift, unsigned nb, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kDigits];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kBlockItems;
    for (int r = 0; r < kItems; ++r) {
        const uint64_t i = base + (uint64_t)r * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// One CTA: exclusive scan of `total` u32 in place (chunk per thread).
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* __restrict__ a, uint64_t total) {
    __shared__ uint32_t part[1024];
    const uint64_t chunk = (total + 1023) / 1024;
    const uint64_t lo = threadIdx.x * chunk, hi = min(total, lo + chunk);
    uint32_t sum = 0;
    for (uint64_t k = lo; k < hi; ++k) sum += a[k];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        const uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - sum;
    for (uint64_t k = lo; k < hi; ++k) {
        const uint32_t v = a[k];
        a[k] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(kThreads) k_rs_scatter(const unsigned long long* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, uint64_t n, int shift,
                                                         unsigned nb, const uint32_t* __restrict__ goff,
                                                         unsigned long long* __restrict__ kout,
                                                         uint32_t* __restrict__ vout) {
    __shared__ uint32_t run[kDigits];
    __shared__ uint32_t wcnt[kWarps][kDigits];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    run[threadIdx.x] = goff[(uint64_t)threadIdx.x * nb + blockIdx.x];
    for (int w = 0; w < kWarps; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kBlockItems;
    for (int r = 0; r < kItems; ++r) {
        const uint64_t i = base + (uint64_t)r * kThreads + threadIdx.x;
        const bool valid = i < n;
        unsigned long long key = 0;
        uint32_t val = 0;
        unsigned d = 0xffffu;  // invalid items match only each other and are not counted
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = (unsigned)(key >> shift) & 0xffu;
        }
        const unsigned mask = __match_any_sync(0xffffffffu, d);
        const unsigned rank = __popc(mask & ((1u << lane) - 1u));
        if (valid && rank == 0) wcnt[warp][d] = __popc(mask);
        __syncthreads();
        if (valid) {
            uint32_t off = run[d] + rank;
            for (unsigned w = 0; w < warp; ++w) off += wcnt[w][d];
            kout[off] = key;
            vout[off] = val;
        }
        __syncthreads();
        uint32_t add = 0;
        for (int w = 0; w < kWarps; ++w) {
            add += wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = 0;
        }
        run[threadIdx.x] += add;
        __syncthreads();
    }
}

// float -> u32 whose unsigned order is the float order
__device__ __forceinline__ unsigned ordered(float f) {
    const unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float unordered(unsigned u) {
    const unsigned b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

struct QuantCheck {
    unsigned smin[3], smax[3];
    unsigned long long bad_ls;     // first index with a non-finite log-scale
    unsigned long long bad_param;  // 2 * index + (0 non-finite parameter, 1 zero quaternion)
};

// Over sorted positions j (perm) so error indices are the quantized set's.
__global__ void k_quant_check(const float* __restrict__ p, uint64_t cap, uint64_t n, const uint32_t* __restrict__ perm,
                              QuantCheck* c) {
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t i = perm ? perm[j] : j;
    bool ls_bad = false;
    for (int d = 0; d < 3; ++d) {
        const float v = p[(3 + d) * cap + i];
        if (!isfinite(v)) {
            ls_bad = true;
            continue;
        }
        atomicMin(&c->smin[d], ordered(v));
        atomicMax(&c->smax[d], ordered(v));
    }
    if (ls_bad) atomicMin(&c->bad_ls, (unsigned long long)j);
    // quant.hpp:104-110: mu[d], quat[d] for d < 3 and alpha_raw
    bool pbad = !isfinite(p[10 * cap + i]);
    for (int d = 0; d < 3; ++d) pbad |= !isfinite(p[d * cap + i]) || !isfinite(p[(6 + d) * cap + i]);
    double qn2 = 0.0;
    for (int k = 0; k < 4; ++k) {
        const double q = (double)p[(6 + k) * cap + i];
        qn2 += q * q;
    }
    const bool qzero = !(sqrt(qn2) > 0.0);
    if (pbad || qzero) atomicMin(&c->bad_param, 2ull * j + (pbad ? 0ull : 1ull));
}

struct QuantArgs {
    const float* p;
    uint64_t cap, n;
    const uint32_t* perm;
    gpk_bounds bb;
    double smin[3], smax[3];
    gpk_quant_spec spec;
    uint32_t *pos, *opa, *ls, *quat;
};

__global__ void k_quantize(const QuantArgs a) {
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.n) return;
    const uint64_t i = a.perm ? a.perm[j] : j;
    const float* p = a.p;
    for (int d = 0; d < 3; ++d) {
        const double e = a.bb.max[d] - a.bb.min[d];
        const double rel = (double)p[d * a.cap + i] - a.bb.min[d];
        a.pos[3 * j + d] = quant_value(e > 0.0 ? rel / e : 0.0, a.spec.pos_bits);
    }
    const double alpha = 1.0 / (1.0 + exp(-(double)p[10 * a.cap + i]));  // alpha_activation (core.hpp:21)
    a.opa[j] = quant_value(alpha, a.spec.opacity_bits);
    for (int d = 0; d < 3; ++d) {
        const double range = a.smax[d] - a.smin[d];
        const double u = range > 0.0 ? ((double)p[(3 + d) * a.cap + i] - a.smin[d]) / range : 0.0;
        a.ls[3 * j + d] = quant_value(u, a.spec.scale_bits);
    }
    double q[4];
    for (int k = 0; k < 4; ++k) q[k] = (double)p[(6 + k) * a.cap + i];
    const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (fabs(qn - 1.0) > 1e-2) {
        const double inv = 1.0 / qn;
        for (int k = 0; k < 4; ++k) q[k] = q[k] * inv;
    }
    for (int k = 0; k < 4; ++k) {  // canonical_half_sphere (quant.hpp:53-62)
        if (q[k] > 0.0) break;
        if (q[k] < 0.0) {
            for (int m = 0; m < 4; ++m) q[m] = q[m] * -1.0;
            break;
        }
    }
    for (int k = 0; k < 4; ++k) a.quat[4 * j + k] = quant_value((q[k] + 1.0) * 0.5, a.spec.quat_bits);
}

__global__ void k_pack_deltas(const uint32_t* __restrict__ v, uint64_t total, int components, int bits,
                              uint8_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int width = (bits + 7) / 8;
    const long long modulus = 1ll << bits, half = modulus >> 1;
    const long long prev = i >= (uint64_t)components ? (long long)v[i - components] : 0ll;
    long long s = (long long)v[i] - prev;
    if (s < -half) s += modulus;
    if (s >= half) s -= modulus;
    const unsigned long long zz = (unsigned long long)((s << 1) ^ (s >> 63));
    for (int b = 0; b < width; ++b) out[i * width + b] = (uint8_t)((zz >> (8 * b)) & 0xffu);
}

// ---- decode direction: detail::unpack_deltas (container.hpp:158-181) + dequantize (quant.hpp:134-176)
struct UnpackStream {
    const uint8_t* bytes;
    uint32_t* values;
    uint64_t count;   // primitives
    int comps, bits;
};

// zig-zag bytes -> signed deltas (as u32, wrapping); flags an out-of-range delta
__global__ void k_unzigzag(const UnpackStream u, unsigned* bad) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= u.count * (uint64_t)u.comps) return;
    const int width = (u.bits + 7) / 8;
    unsigned long long zz = 0;
    for (int b = 0; b < width; ++b) zz |= (unsigned long long)u.bytes[i * width + b] << (8 * b);
    if (zz >= (1ull << u.bits)) atomicOr(bad, 1u);
    const long long sv = (long long)((zz >> 1) ^ (~(zz & 1) + 1));
    u.values[i] = (uint32_t)(unsigned long long)sv;
}

// per-component running sum mod 2^bits: CTA c scans component c (chunk per
// thread, then a block scan of the chunk sums; u32 wrap-around is exact mod 2^bits)
__global__ void __launch_bounds__(1024) k_delta_scan(const UnpackStream u) {
    __shared__ uint32_t part[1024];
    const int c = blockIdx.x;
    const uint64_t n = u.count, chunk = (n + 1023) / 1024;
    const uint64_t lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
    uint32_t sum = 0;
    for (uint64_t k = lo; k < hi; ++k) sum += u.values[k * u.comps + c];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const uint32_t v = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - sum;
    const uint32_t mask = (uint32_t)((1ull << u.bits) - 1);
    for (uint64_t k = lo; k < hi; ++k) {
        run += u.values[k * u.comps + c];
        u.values[k * u.comps + c] = run & mask;
    }
}

struct DequantArgs {
    const uint32_t *pos, *opa, *ls, *quat;
    uint64_t n;
    gpk_bounds bb;
    double smin[3], smax[3];
    gpk_quant_spec spec;
    float* rec;  // n x 11 records
};

__device__ __forceinline__ double dequant_value(uint32_t q, int bits) { return (double)q / (double)((1u << bits) - 1); }

__global__ void k_dequantize(const DequantArgs a) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    float* r = a.rec + 11 * i;
    for (int d = 0; d < 3; ++d) {
        const double ext = a.bb.max[d] - a.bb.min[d];
        r[d] = (float)(a.bb.min[d] + dequant_value(a.pos[3 * i + d], a.spec.pos_bits) * ext);
        r[3 + d] = (float)(a.smin[d] + dequant_value(a.ls[3 * i + d], a.spec.scale_bits) * (a.smax[d] - a.smin[d]));
    }
    double al = dequant_value(a.opa[i], a.spec.opacity_bits);  // alpha_activation_inverse (core.hpp:23-27)
    al = fmin(1.0 - 1e-12, fmax(1e-12, al));
    r[10] = (float)log(al / (1.0 - al));
    double q[4];
    for (int k = 0; k < 4; ++k) q[k] = dequant_value(a.quat[4 * i + k], a.spec.quat_bits) * 2.0 - 1.0;
    const bool nz = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]) > 0.0;
    for (int k = 0; k < 4; ++k) r[6 + k] = nz ? (float)q[k] : (k == 0 ? 1.0f : 0.0f);
}

struct Dev {
    void* p = nullptr;
    ~Dev() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t b) { return cudaMalloc(&p, std::max<size_t>(b, 16)); }
};

int fail(int code, const std::string& m) { return gpk::set_last_error(code, m); }

#define CTRY(x)                                 \
    do {                                        \
        const int _s = (x);                     \
        if (_s != GPK_OK) return _s;            \
    } while (0)
#define CCK(x)                                                                     \
    do {                                                                           \
        const cudaError_t _e = (x);                                                \
        if (_e != cudaSuccess) return fail(GPK_ERR_CUDA, cudaGetErrorString(_e));  \
    } while (0)

struct Resident {
    const float* p = nullptr;
    uint64_t cap = 0, n = 0;
    gpk_bounds bb{};
    cudaStream_t st = nullptr;
};

int resident(gpk_session* s, Resident& r) {
    void* ptr = nullptr;
    uint64_t bytes = 0;
    CTRY(gpk_gaussian_count(s, &r.n));
    CTRY(gpk_get_bounds(s, &r.bb));
    void* stv = nullptr;
    CTRY(gpk_session_get_stream(s, &stv));
    r.st = static_cast<cudaStream_t>(stv);
    CTRY(gpk_session_synchronize(s));
    CTRY(gpk_device_buffer(s, GPK_BUF_PARAMS, &ptr, &bytes));
    r.p = static_cast<const float*>(ptr);
    r.cap = bytes / 44;
    return GPK_OK;
}

int validate_spec(const gpk_quant_spec* q) {
    const int b[5] = {q->pos_bits, q->opacity_bits, q->scale_bits, q->quat_bits, q->morton_bits};
    for (int v : b)
        if (v < 4 || v > 21) return fail(GPK_ERR_INVALID_ARGUMENT, "QuantSpec: bit widths must be in [4, 21]");
    return GPK_OK;
}

unsigned grid(uint64_t n, int t = kThreads) { return (unsigned)std::max<uint64_t>(1, (n + t - 1) / t); }

// Stable Z-order permutation into perm (device, n u32).
int morton_perm(const Resident& r, int bits, uint32_t* perm) {
    const uint64_t n = r.n;
    if (n == 0) return GPK_OK;
    Dev k0, k1, v1, hist;
    CCK(k0.alloc(n * 8));
    CCK(k1.alloc(n * 8));
    CCK(v1.alloc(n * 4));
    const unsigned nb = (unsigned)((n + kBlockItems - 1) / kBlockItems);
    CCK(hist.alloc((size_t)kDigits * nb * 4));
    auto* ka = static_cast<unsigned long long*>(k0.p);
    auto* kb = static_cast<unsigned long long*>(k1.p);
    uint32_t* va = perm;
    uint32_t* vb = static_cast<uint32_t*>(v1.p);
    k_morton_codes<<<grid(n), kThreads, 0, r.st>>>(r.p, r.cap, n, r.bb, bits, ka, va);
    CCK(cudaGetLastError());
    const int passes = (3 * bits + 7) / 8;
    for (int ps = 0; ps < passes; ++ps) {
        const int shift = 8 * ps;
        k_rs_hist<<<nb, kThreads, 0, r.st>>>(ka, n, shift, nb, static_cast<uint32_t*>(hist.p));
        k_rs_scan<<<1, 1024, 0, r.st>>>(static_cast<uint32_t*>(hist.p), (uint64_t)kDigits * nb);
        k_rs_scatter<<<nb, kThreads, 0, r.st>>>(ka, va, n, shift, nb, static_cast<uint32_t*>(hist.p), kb, vb);
        CCK(cudaGetLastError());
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (va != perm) CCK(cudaMemcpyAsync(perm, va, n * 4, cudaMemcpyDeviceToDevice, r.st));
    CCK(cudaStreamSynchronize(r.st));
    return GPK_OK;
}

// quantize (quant.hpp:67-132) of the resident set in perm order (or set order)
// into device streams; scale ranges out.
int quantize_dev(const Resident& r, const gpk_quant_spec* spec, const uint32_t* perm, uint32_t* pos, uint32_t* opa,
                 uint32_t* ls, uint32_t* quat, double smin[3], double smax[3]) {
    const uint64_t n = r.n;
    Dev chk;
    CCK(chk.alloc(sizeof(QuantCheck)));
    QuantCheck init;
    for (int d = 0; d < 3; ++d) {
        init.smin[d] = 0xffffffffu;
        init.smax[d] = 0u;
    }
    init.bad_ls = init.bad_param = ~0ull;
    CCK(cudaMemcpyAsync(chk.p, &init, sizeof init, cudaMemcpyHostToDevice, r.st));
    if (n) k_quant_check<<<grid(n), kThreads, 0, r.st>>>(r.p, r.cap, n, perm, static_cast<QuantCheck*>(chk.p));
    CCK(cudaGetLastError());
    QuantCheck c;
    CCK(cudaMemcpyAsync(&c, chk.p, sizeof c, cudaMemcpyDeviceToHost, r.st));
    CCK(cudaStreamSynchronize(r.st));
    if (c.bad_ls != ~0ull)
        return fail(GPK_ERR_INVALID_ARGUMENT, "quantize: non-finite log-scale at primitive " + std::to_string(c.bad_ls));
    if (c.bad_param != ~0ull)
        return fail(GPK_ERR_INVALID_ARGUMENT, std::string(c.bad_param & 1 ? "quantize: zero quaternion at primitive "
                                                                          : "quantize: non-finite parameter at primitive ") +
                                                  std::to_string(c.bad_param >> 1));
    QuantArgs a;
    a.p = r.p;
    a.cap = r.cap;
    a.n = n;
    a.perm = perm;
    a.bb = r.bb;
    a.spec = *spec;
    for (int d = 0; d < 3; ++d) {
        // scale_min / max start at 0 and take the first primitive's values
        // (quant.hpp:79-90): with n > 0 that is the plain min / max
        a.smin[d] = n ? (double)unordered(c.smin[d]) : 0.0;
        a.smax[d] = n ? (double)unordered(c.smax[d]) : 0.0;
        if (!(a.smax[d] > a.smin[d])) a.smax[d] = a.smin[d];
        smin[d] = a.smin[d];
        smax[d] = a.smax[d];
    }
    a.pos = pos;
    a.opa = opa;
    a.ls = ls;
    a.quat = quat;
    if (n) k_quantize<<<grid(n), kThreads, 0, r.st>>>(a);
    CCK(cudaGetLastError());
    return GPK_OK;
}

}  // namespace

extern "C" {

int gpk_morton_sort(gpk_session* s, int32_t bits, uint64_t* perm_out) {
    if (!s) return fail(GPK_ERR_INVALID_ARGUMENT, "null session");
    if (bits < 1 || bits > 21) return fail(GPK_ERR_INVALID_ARGUMENT, "morton_sort: bits must be in [1, 21]");
    Resident r;
    CTRY(resident(s, r));
    if (r.n && !perm_out) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    Dev perm;
    CCK(perm.alloc(r.n * 4));
    CTRY(morton_perm(r, bits, static_cast<uint32_t*>(perm.p)));
    std::vector<uint32_t> h(r.n);
    if (r.n) CCK(cudaMemcpy(h.data(), perm.p, r.n * 4, cudaMemcpyDeviceToHost));
    for (uint64_t k = 0; k < r.n; ++k) perm_out[k] = h[k];
    return GPK_OK;
}

int gpk_quantize(gpk_session* s, const gpk_quant_spec* spec, int32_t morton_order, uint32_t* positions,
                 uint32_t* opacities, uint32_t* log_scales, uint32_t* quats, double scale_min[3],
                 double scale_max[3]) {
    if (!s || !spec || !scale_min || !scale_max) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    CTRY(validate_spec(spec));
    Resident r;
    CTRY(resident(s, r));
    const uint64_t n = r.n;
    if (n && (!positions || !opacities || !log_scales || !quats))
        return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    Dev perm, streams;
    CCK(perm.alloc(n * 4));
    CCK(streams.alloc(n * 11 * 4));
    if (morton_order) CTRY(morton_perm(r, spec->morton_bits, static_cast<uint32_t*>(perm.p)));
    uint32_t* sp = static_cast<uint32_t*>(streams.p);
    CTRY(quantize_dev(r, spec, morton_order ? static_cast<uint32_t*>(perm.p) : nullptr, sp, sp + 3 * n,
                      sp + 4 * n, sp + 7 * n, scale_min, scale_max));
    if (n) {
        CCK(cudaMemcpyAsync(positions, sp, n * 12, cudaMemcpyDeviceToHost, r.st));
        CCK(cudaMemcpyAsync(opacities, sp + 3 * n, n * 4, cudaMemcpyDeviceToHost, r.st));
        CCK(cudaMemcpyAsync(log_scales, sp + 4 * n, n * 12, cudaMemcpyDeviceToHost, r.st));
        CCK(cudaMemcpyAsync(quats, sp + 7 * n, n * 16, cudaMemcpyDeviceToHost, r.st));
    }
    CCK(cudaStreamSynchronize(r.st));
    return GPK_OK;
}

uint64_t gpk_stream_bytes(uint64_t count, int32_t components, int32_t bits) {
    return count * (uint64_t)components * (uint64_t)((bits + 7) / 8);
}

int gpk_encode_streams(gpk_session* s, const gpk_quant_spec* spec, uint8_t* positions, uint8_t* opacities,
                       uint8_t* log_scales, uint8_t* quats, double scale_min[3], double scale_max[3]) {
    if (!s || !spec || !scale_min || !scale_max) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    CTRY(validate_spec(spec));
    Resident r;
    CTRY(resident(s, r));
    const uint64_t n = r.n;
    if (n && (!positions || !opacities || !log_scales || !quats))
        return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    Dev perm, streams, bytes;
    CCK(perm.alloc(n * 4));
    CCK(streams.alloc(n * 11 * 4));
    CTRY(morton_perm(r, spec->morton_bits, static_cast<uint32_t*>(perm.p)));
    uint32_t* sp = static_cast<uint32_t*>(streams.p);
    CTRY(quantize_dev(r, spec, static_cast<uint32_t*>(perm.p), sp, sp + 3 * n, sp + 4 * n, sp + 7 * n, scale_min,
                      scale_max));
    struct S {
        const uint32_t* v;
        int comps, bits;
        uint8_t* host;
    } st[4] = {{sp, 3, spec->pos_bits, positions},
               {sp + 3 * n, 1, spec->opacity_bits, opacities},
               {sp + 4 * n, 3, spec->scale_bits, log_scales},
               {sp + 7 * n, 4, spec->quat_bits, quats}};
    uint64_t total = 0;
    for (const S& x : st) total += gpk_stream_bytes(n, x.comps, x.bits);
    CCK(bytes.alloc(total));
    uint64_t off = 0;
    for (const S& x : st) {
        const uint64_t cnt = n * (uint64_t)x.comps, b = gpk_stream_bytes(n, x.comps, x.bits);
        uint8_t* dst = static_cast<uint8_t*>(bytes.p) + off;
        if (cnt) k_pack_deltas<<<grid(cnt), kThreads, 0, r.st>>>(x.v, cnt, x.comps, x.bits, dst);
        CCK(cudaGetLastError());
        if (b) CCK(cudaMemcpyAsync(x.host, dst, b, cudaMemcpyDeviceToHost, r.st));
        off += b;
    }
    CCK(cudaStreamSynchronize(r.st));
    return GPK_OK;
}

// unpack_deltas of the four streams + dequantize (the decode side of
// container.hpp:232-260 after LZMA): records out (n x 11 f32, host), and the
// decoded set loaded into the session when load != 0.
int gpk_decode_streams(gpk_session* s, const gpk_quant_spec* spec, uint64_t n, const gpk_bounds* bbox,
                       const double scale_min[3], const double scale_max[3], const uint8_t* positions,
                       const uint8_t* opacities, const uint8_t* log_scales, const uint8_t* quats,
                       float* records_out, int32_t load) {
    if (!s || !spec || !bbox || !scale_min || !scale_max) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    if (n && (!positions || !opacities || !log_scales || !quats)) return fail(GPK_ERR_INVALID_ARGUMENT, "null argument");
    CTRY(validate_spec(spec));
    void* stv = nullptr;
    CTRY(gpk_session_get_stream(s, &stv));
    CTRY(gpk_session_synchronize(s));  // selects the session's device
    cudaStream_t st = static_cast<cudaStream_t>(stv);
    const int comps[4] = {3, 1, 3, 4};
    const int bits[4] = {spec->pos_bits, spec->opacity_bits, spec->scale_bits, spec->quat_bits};
    const uint8_t* host[4] = {positions, opacities, log_scales, quats};
    const char* names[4] = {"positions", "opacities", "log_scales", "quats"};
    Dev raw, vals, rec, bad;
    uint64_t rb = 0;
    for (int k = 0; k < 4; ++k) rb += gpk_stream_bytes(n, comps[k], bits[k]);
    CCK(raw.alloc(rb));
    CCK(vals.alloc(n * 11 * 4));
    CCK(rec.alloc(n * 44));
    CCK(bad.alloc(16));
    CCK(cudaMemsetAsync(bad.p, 0, 16, st));
    uint64_t off = 0, voff = 0;
    uint32_t* vp[4];
    for (int k = 0; k < 4; ++k) {
        const uint64_t b = gpk_stream_bytes(n, comps[k], bits[k]);
        uint8_t* dst = static_cast<uint8_t*>(raw.p) + off;
        if (b) CCK(cudaMemcpyAsync(dst, host[k], b, cudaMemcpyHostToDevice, st));
        UnpackStream u{dst, static_cast<uint32_t*>(vals.p) + voff, n, comps[k], bits[k]};
        vp[k] = u.values;
        if (n) {
            k_unzigzag<<<grid(n * comps[k]), kThreads, 0, st>>>(u, static_cast<unsigned*>(bad.p) + k);
            k_delta_scan<<<comps[k], 1024, 0, st>>>(u);
        }
        CCK(cudaGetLastError());
        off += b;
        voff += n * comps[k];
    }
    unsigned flags[4];
    CCK(cudaMemcpyAsync(flags, bad.p, 16, cudaMemcpyDeviceToHost, st));
    CCK(cudaStreamSynchronize(st));
    for (int k = 0; k < 4; ++k)
        if (flags[k])
            return fail(GPK_ERR_CORRUPT_CONTAINER, std::string("container: out-of-range delta in ") + names[k]);
    DequantArgs a;
    a.pos = vp[0];
    a.opa = vp[1];
    a.ls = vp[2];
    a.quat = vp[3];
    a.n = n;
    a.bb = *bbox;
    for (int d = 0; d < 3; ++d) {
        a.smin[d] = scale_min[d];
        a.smax[d] = scale_max[d];
    }
    a.spec = *spec;
    a.rec = static_cast<float*>(rec.p);
    if (n) k_dequantize<<<grid(n), kThreads, 0, st>>>(a);
    CCK(cudaGetLastError());
    std::vector<float> tmp;
    float* out = records_out;
    if (!out && load) {
        tmp.resize(n * 11);
        out = tmp.data();
    }
    if (out && n) CCK(cudaMemcpyAsync(out, rec.p, n * 44, cudaMemcpyDeviceToHost, st));
    CCK(cudaStreamSynchronize(st));
    if (load) CTRY(gpk_set_gaussians(s, n, out, bbox));
    return GPK_OK;
}

}  // extern "C"
