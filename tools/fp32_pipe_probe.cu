// Measures sustained FP32 issue throughput on this GPU for the instruction forms the compat filter uses:
// scalar FFMA (3-register), packed FFMA2 (f32x2), and an FFMA2 + scalar FFMA mix.  Each thread runs 8
// independent dependency chains; the reported figure is lane-FMAs per SM per clock (nominal B200: 128).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipe_probe tools/fp32_pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
template <int MODE>
__global__ void k(float* out, int iters, float s) {
    float f[8];
    u64 v[8];
    for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 1e-3f + i; v[i] = ((u64)__float_as_uint(f[i]) << 32) | __float_as_uint(f[i] + 1); }
    const u64 m = ((u64)__float_as_uint(s) << 32) | __float_as_uint(s);
    const u64 a = ((u64)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) f[i] = fmaf(f[i], s, f[(i + 1) & 7]);
            if (MODE == 1) v[i] = ffma2(v[i], m, v[(i + 1) & 7]);
            if (MODE == 2) { if (i & 1) f[i] = fmaf(f[i], s, f[(i + 1) & 7]); else v[i] = ffma2(v[i], m, v[(i + 1) & 7]); }
            if (MODE == 3) v[i] = ffma2(v[i], m, a);
            if (MODE == 4) {  // one operand a scalar broadcast (.F32), as in the compat/score loops
                const u64 bs = ((u64)__float_as_uint(f[i]) << 32) | __float_as_uint(f[i]);
                v[i] = ffma2(v[i], bs, v[(i + 1) & 7]);
            }
        }
    }
    float acc = 0.f;
    for (int i = 0; i < 8; ++i) acc += f[i] + __uint_as_float((unsigned)v[i]) + __uint_as_float((unsigned)(v[i] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
    const int iters = 20000;
    const char* names[5] = {"FFMA scalar (3-reg)", "FFMA2 (3-reg pairs)", "mix FFMA2 + FFMA", "FFMA2 (const pair)",
                            "FFMA2 (scalar bcast)"};
    const double lanes_per_inst[5] = {1, 2, 1.5, 2, 2};
    for (int mode = 0; mode < 5; ++mode) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<sms * 8, 256>>>(out, iters, 1.0001f);
            if (mode == 1) k<1><<<sms * 8, 256>>>(out, iters, 1.0001f);
            if (mode == 2) k<2><<<sms * 8, 256>>>(out, iters, 1.0001f);
            if (mode == 3) k<3><<<sms * 8, 256>>>(out, iters, 1.0001f);
            if (mode == 4) k<4><<<sms * 8, 256>>>(out, iters, 1.0001f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double insts = (double)sms * 8 * 256 / 32 * iters * 8;  // warp instructions
        const double lane_fma = insts * 32 * lanes_per_inst[mode];
        printf("%-24s %8.3f ms  %7.2f T lane-FMA/s  (%.1f per SM per clk at %d MHz nominal clock attr)\n", names[mode], ms,
               lane_fma / ms / 1e9, lane_fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
