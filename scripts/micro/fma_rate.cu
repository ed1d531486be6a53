// Microbenchmark: FP32 FMA issue throughput on sm_100a, FFMA vs FFMA2
// (packed fp32x2), with a broadcast scalar multiplier as in the spline
// contraction.  Prints FMA/clk/SM for each variant.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) fma_kernel(float *out, float w0, float w1, int iters) {
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = threadIdx.x * 1e-3f + e;
    const float wa = w0 + threadIdx.x * 1e-9f, wb = w1;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // scalar FFMA, register operands
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = __fmaf_rn(wa, acc[e], wb);
        } else {          // packed FFMA2: (wa, wa) * acc2 + (wb, wb)
            float2 *a2 = reinterpret_cast<float2 *>(acc);
            const float2 w2 = make_float2(wa, wa), b2 = make_float2(wb, wb);
#pragma unroll
            for (int e = 0; e < 8; ++e) a2[e] = __ffma2_rn(w2, a2[e], b2);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 16; ++e) s += acc[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * 148 * 8 * 256 * 4);
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int blocksPerSM : {4, 8}) {
            dim3 grid(sms * blocksPerSM);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) fma_kernel<0><<<grid, 256>>>(out, 1.0001f, 0.5f, iters);
                else fma_kernel<1><<<grid, 256>>>(out, 1.0001f, 0.5f, iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double fmas = (double)grid.x * 256 * iters * 16;
            printf("mode=%s blocks/SM=%d  %.3f ms  %.2f TFMA/s  = %.1f FMA/clk/SM at max clock %d MHz\n",
                   mode ? "FFMA2" : "FFMA ", blocksPerSM, ms, fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3),
                   clk / 1000);
        }
    }
    return 0;
}
