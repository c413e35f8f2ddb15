// FP32 pipe peak probe: scalar FFMA chains vs packed FFMA2 (fma.rn.f32x2) chains, all SMs.
// Prints lane-FMA/s for each; used to set the roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;

__global__ void k_ffma(float *out, float a, float b) {
    float x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float *out, float a, float b) {
    unsigned long long x[CH];
    unsigned long long A, Bv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(Bv) : "f"(b));
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float lo = threadIdx.x * 1e-3f + i, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(lo), "f"(hi));
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(Bv));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
        s += lo + hi;
    }
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_fadd_fmul(float *out, float a, float b) {  // the Eq. 1 mix: 3 FADD, 1 FMUL, 2 FFMA
    float x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const float dx = x[i] - a, dy = x[i] - b, dz = x[i] - 0.25f;
            x[i] = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx))) * 1e-3f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out;
    cudaMalloc(&out, 4);
    dim3 grid(sms * 8), block(256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double thr = (double)grid.x * block.x;
    for (int k = 0; k < 3; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (k == 0) k_ffma<<<grid, block>>>(out, 0.999f, 1e-3f);
            if (k == 1) k_ffma2<<<grid, block>>>(out, 0.999f, 1e-3f);
            if (k == 2) k_fadd_fmul<<<grid, block>>>(out, 0.999f, 1e-3f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double lanes = thr * ITERS * CH * (k == 1 ? 2 : 1) * (k == 2 ? 6 : 1);
        printf("%s: %.3f ms, %.2f T lane-ops/s (%s)\n", k == 0 ? "FFMA " : (k == 1 ? "FFMA2" : "dist6"), ms,
               lanes / (ms * 1e-3) / 1e12, k == 2 ? "6 FP32 instr per Eq.1 distance" : "FMA lanes");
    }
    printf("SMs %d, attr clock %d kHz, nominal 128 lanes/SM/clk -> %.2f T lane-ops/s at 1965 MHz\n", sms, clk,
           sms * 128.0 * 1.965e9 / 1e12);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
