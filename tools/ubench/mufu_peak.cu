// MUFU ex2 peak on this GPU: independent chains per thread (latency hidden),
// several occupancies; plus the same loop with one FFMA2 per two ex2.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int CH>
__global__ void chains(float* out, int iters) {
    float a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = -(threadIdx.x * 1e-4f + 0.01f * c);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = ex2f(-a[c]);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c];
    if (s == 1234.5f) out[blockIdx.x] = s;
}
template <int CH>
void run(int wps) {
    float* out; cudaMalloc(&out, 1 << 20);
    int threads = 256, blocks = 148 * wps / 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2048;
    chains<CH><<<blocks, threads>>>(out, 8);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        chains<CH><<<blocks, threads>>>(out, iters);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("chains %2d warps/SM %2d: %.3f Tex2/s\n", CH, wps, (double)blocks * threads * iters * CH / (best * 1e-3) / 1e12);
    cudaFree(out);
}
int main() {
    for (int w : {8, 16, 32, 64}) { run<4>(w); run<8>(w); run<16>(w); }
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock attr %d kHz\n", clk);
    return 0;
}
