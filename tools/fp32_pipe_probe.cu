// Measures sustained FP32 issue throughput on this GPU for the instruction forms the compat filter and
// the scoring loop use: scalar FFMA, packed FFMA2 / FADD2 / FMUL2 (f32x2), FFMA2 with a scalar broadcast
// operand, and mixes of packed FP with 32-bit integer logic (LOP3 / SHF) in the compat loop's proportions.
// Each thread runs 8 independent dependency chains (MODE 9: 2 chains); the reported figure is lane-FP ops
// per SM per clock (nominal B200: 128) and, for the mixes, the ALU instructions issued alongside.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipe_probe tools/fp32_pipe_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
    u64 d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
    u64 d;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
template <int MODE>
__global__ void k(float* out, int iters, float s) {
    float f[8];
    u64 v[8];
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = threadIdx.x * 1e-3f + i;
        v[i] = ((u64)__float_as_uint(f[i]) << 32) | __float_as_uint(f[i] + 1);
        w[i] = threadIdx.x * 7 + i;
    }
    const u64 m = ((u64)__float_as_uint(s) << 32) | __float_as_uint(s);
    const u64 a = ((u64)__float_as_uint(0.999f) << 32) | __float_as_uint(0.999f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) f[i] = fmaf(f[i], s, f[(i + 1) & 7]);
            if (MODE == 1) v[i] = ffma2(v[i], m, v[(i + 1) & 7]);
            if (MODE == 2) { if (i & 1) f[i] = fmaf(f[i], s, f[(i + 1) & 7]); else v[i] = ffma2(v[i], m, v[(i + 1) & 7]); }
            if (MODE == 3) v[i] = ffma2(v[i], m, a);
            if (MODE == 4) {  // an operand pair re-packed from a scalar in the loop (ptxas emits IMAD/MOV)
                const u64 bs = ((u64)__float_as_uint(f[i]) << 32) | __float_as_uint(f[i]);
                v[i] = ffma2(v[i], bs, v[(i + 1) & 7]);
            }
            if (MODE == 5) v[i] = fadd2(v[i], v[(i + 1) & 7]);
            if (MODE == 6) v[i] = fmul2(v[i], v[(i + 1) & 7]);
            if (MODE == 7) {  // 5 FP2 + 2 LOP3 (the compat loop's 20 : 8 ratio)
                v[i] = ffma2(v[i], m, v[(i + 1) & 7]);
                if ((i & 3) == 0) {
                    w[i] = (w[i] & ~(uint32_t)v[i]) ^ (w[(i + 3) & 7] >> 1);
                    w[(i + 1) & 7] = __funnelshift_l((uint32_t)(v[i] >> 32), w[(i + 1) & 7], 1);
                }
                if ((i & 3) == 2) w[i] = w[i] & (uint32_t)v[i] & 0x7fffffffu;
            }
            if (MODE == 8) {  // 1 FP2 : 1 ALU
                v[i] = ffma2(v[i], m, v[(i + 1) & 7]);
                w[i] = __funnelshift_l((uint32_t)v[i], w[i], 1);
            }
            if (MODE == 9) {  // only 2 independent chains per thread
                v[i & 1] = ffma2(v[i & 1], m, a);
            }
        }
    }
    float acc = 0.f;
    for (int i = 0; i < 8; ++i)
        acc += f[i] + __uint_as_float((unsigned)v[i]) + __uint_as_float((unsigned)(v[i] >> 32)) + (float)w[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
    const int iters = 20000;
    const int NM = 10;
    const char* names[NM] = {"FFMA scalar (3-reg)", "FFMA2 (3-reg pairs)", "mix FFMA2 + FFMA", "FFMA2 (const pair)",
                             "FFMA2 (pair re-packed)", "FADD2 (pairs)", "FMUL2 (pairs)", "FFMA2 + LOP3/SHF 5:2",
                             "FFMA2 + SHF 1:1", "FFMA2 2 chains/thread"};
    const double lanes_per_inst[NM] = {1, 2, 1.5, 2, 2, 2, 2, 2, 2, 2};
    for (int mode = 0; mode < NM; ++mode) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: k<0><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 1: k<1><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 2: k<2><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 3: k<3><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 4: k<4><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 5: k<5><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 6: k<6><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 7: k<7><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 8: k<8><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
                case 9: k<9><<<sms * 8, 256>>>(out, iters, 1.0001f); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double insts = (double)sms * 8 * 256 / 32 * iters * 8;  // FP warp instructions
        const double lane_fma = insts * 32 * lanes_per_inst[mode];
        printf("%-24s %8.3f ms  %7.2f T lane-FP/s  (%.1f per SM per clk at %d MHz clock attr)\n", names[mode], ms,
               lane_fma / ms / 1e9, lane_fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
