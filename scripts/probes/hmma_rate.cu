// Probe: legacy mma.sync m16n8k16 (f16 x f16 -> f32) throughput on B200, per SM and per warp count.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hmma hmma_rate.cu && /tmp/hmma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(float *out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = a0 + 11;
    float acc[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                         : "r"(a0 + c), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1 + c));
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    if (s == 12345.f) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *o;
    cudaMalloc(&o, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int wps : {4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k<8><<<sms, 32 * wps>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = (double)sms * wps * iters * 8;
            if (rep) printf("warps/SM %2d: %.3f ms, %.1f mma/clk/SM (at 1.965 GHz), %.1f TFLOP/s f16\n", wps, ms,
                            mmas / sms / (ms * 1e-3 * 1.965e9), mmas * 4096 / (ms * 1e-3) / 1e12);
        }
    }
    // latency: one warp, one chain
    cudaEventRecord(e0);
    k<1><<<1, 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dependent chain latency: %.1f clk per mma\n", ms * 1e-3 * 1.965e9 / iters);
    return 0;
}
