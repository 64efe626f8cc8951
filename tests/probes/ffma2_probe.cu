// Throughput probe: FFMA vs FFMA2 (fma.rn.f32x2) on sm_100a, independent chains.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__global__ void k1(float* out, float s, int iters) {
    float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
    float t = 0; for (int i = 0; i < 8; ++i) t += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = t; }
__global__ void k2(float* out, float s, int iters) {
    unsigned long long a[8]; for (int i = 0; i < 8; ++i) a[i] = f2(threadIdx.x * 0.001f + i, i * 0.5f);
    const unsigned long long ss = f2(s, s), hh = f2(0.5f, 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(ss), "l"(hh));
    float t = 0; for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t; }
// mixed: per iteration 8 FMA + 2 MUFU.EX2 + 4 integer ops
__global__ void k3(float* out, float s, int iters, int packed) {
    float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    unsigned m = threadIdx.x; float e = 0.f;
    for (int it = 0; it < iters; ++it) {
        if (packed) {
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                unsigned long long v = f2(a[i], a[i + 1]);
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v) : "l"(f2(s, s)), "l"(f2(0.5f, 0.5f)));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(a[i]), "=f"(a[i + 1]) : "l"(v));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
        }
        float y0, y1; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a[0] * -1e-3f));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(a[1] * -1e-3f));
        e += y0 + y1; m = (m * 1664525u + 1013904223u) ^ (m >> 3);
    }
    float t = e + (float)(m & 1); for (int i = 0; i < 8; ++i) t += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = t; }
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 20000; float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); k1<<<148 * 8, 256>>>(out, 0.999f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); double fl = 148.0 * 8 * 256 * iters * 8;
        printf("FFMA : %.3f ms  %.1f Gfma/s  (%.1f per clk per SM at 1.965 GHz)\n", ms, fl / ms / 1e6, fl / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(a); k2<<<148 * 8, 256>>>(out, 0.999f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); fl *= 2;
        printf("FFMA2: %.3f ms  %.1f Gfma/s  (%.1f per clk per SM)\n", ms, fl / ms / 1e6, fl / (ms * 1e-3) / 148 / 1.965e9);
        for (int p = 0; p < 2; ++p) {
            cudaEventRecord(a); k3<<<148 * 8, 256>>>(out, 0.999f, iters, p); cudaEventRecord(b); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("mixed packed=%d: %.3f ms\n", p, ms);
        }
    }
    return 0;
}
