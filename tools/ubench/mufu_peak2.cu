// MUFU ex2 peak with independent (non-MUFU-chained) inputs: u_i <- u_i + d,
// acc_i += ex2(u_i), 16 lanes of state per thread (8 float2), packed updates.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k(float* out, int iters) {
    float2 u[8], acc[8];
    const float2 dlt = make_float2(-1e-7f, -2e-7f);
#pragma unroll
    for (int c = 0; c < 8; ++c) { u[c] = make_float2(-0.001f * c - threadIdx.x * 1e-5f, -0.5f - 0.001f * c); acc[c] = make_float2(0.f, 0.f); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            acc[c] = __fadd2_rn(acc[c], make_float2(ex2f(u[c].x), ex2f(u[c].y)));
            u[c] = __fadd2_rn(u[c], dlt);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c].x + acc[c].y;
    if (s == 1234.5f) out[blockIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 1 << 20);
    for (int wps : {8, 16, 32, 64}) {
        int threads = 256, blocks = 148 * wps / 8;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int iters = 2048;
        k<<<blocks, threads>>>(out, 8);
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a); k<<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("warps/SM %2d: %.3f Tex2/s (%.1f per SM per clk at 1965 MHz)\n", wps,
               (double)blocks * threads * iters * 16 / (best * 1e-3) / 1e12,
               (double)blocks * threads * iters * 16 / (best * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
