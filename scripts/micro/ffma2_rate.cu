// Issue/pipe rate of FFMA vs packed FFMA2 (sm_100a) -- 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void k1(float* out, int iters, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], a, b);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k2(float* out, int iters, float a, float b) {
    unsigned long long x[8];
    unsigned long long A, B;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
    for (int i = 0; i < 8; ++i) { float v = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(v)); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], A, B);
    float s = 0;
    for (int i = 0; i < 8; ++i) { float l, h; asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(x[i])); s += l + h; }
    if (s == 1.2345f) out[0] = s;
}
// mixed: one FFMA2 + one FFMA per step (does FFMA2 share the pipe with FFMA?)
__global__ void k3(float* out, int iters, float a, float b) {
    unsigned long long x[4]; float y[4];
    unsigned long long A, B;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
    for (int i = 0; i < 4; ++i) { float v = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(v)); y[i] = v; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) { x[i] = fma2(x[i], A, B); y[i] = __fmaf_rn(y[i], a, b); }
    float s = 0;
    for (int i = 0; i < 4; ++i) { float l, h; asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(x[i])); s += l + h + y[i]; }
    if (s == 1.2345f) out[0] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k1<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
            if (kind == 1) k2<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
            if (kind == 2) k3<<<blocks, threads>>>(out, iters, 0.999f, 1e-4f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double lanes_fma = double(blocks) * threads * iters * 16 * 8;           // k1: 8 FFMA/step
            if (kind == 1) lanes_fma *= 2;                                          // k2: 8 FFMA2 = 16 FMA
            if (kind == 2) lanes_fma = double(blocks) * threads * iters * 16 * 12;  // k3: 4 FFMA2 + 4 FFMA
            double instr = double(blocks) * threads / 32 * iters * 16 * 8;          // warp instructions
            printf("%s rep %d: %.3f ms  %.1f TFLOP/s  %.2f warp-instr/clk/SM @1.965GHz\n",
                   kind == 0 ? "FFMA " : kind == 1 ? "FFMA2" : "mixed", rep, ms, 2 * lanes_fma / ms / 1e9,
                   instr / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    return 0;
}
