// =====================================================================================================
// SC^2 on the dense block: Ĝ = C ⊙ (C·C) (Eq. 2) restricted to the "heavy" rows H (the
// high-degree rows — on registration workloads the inliers, whose mutual compatibility is dense).
// C·C over H is a dense binary contraction, so it runs on the 5th-gen tensor cores:
//   X = C[H, :] as uint8 0/1 (K-major, [h][K]),  D = X · X^T  (exact: int32 accumulate, K <= 32768)
// with tcgen05.mma kind::i8 (M=128, N=256, K=32 per instruction), operands staged by TMA
// (cp.async.bulk.tensor, 128B swizzle) through a 4-stage mbarrier pipeline, the accumulator in TMEM
// (256 columns) and a 4-warp epilogue (tcgen05.ld 32x32b) that stores D as uint16 for the assembly pass.
// Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread MMA issuer, warps 2..5 =
// epilogue.  Which rows are heavy only changes speed, never the result (Σ_k splits exactly).
// =====================================================================================================
#pragma once
#include <cuda.h>
#include <cstdint>

namespace trk {

constexpr int MMA_BM = 128;
constexpr int MMA_BN = 256;
constexpr int MMA_BK = 128;  // bytes = int8 elements per stage per row
constexpr int MMA_STAGES = 4;
constexpr int MMA_A_BYTES = MMA_BM * MMA_BK;  // 16 KB
constexpr int MMA_B_BYTES = MMA_BN * MMA_BK;  // 32 KB
constexpr int MMA_STAGE_BYTES = MMA_A_BYTES + MMA_B_BYTES;
constexpr int MMA_SMEM_BYTES = MMA_STAGES * MMA_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int MMA_THREADS = 192;

// Instruction descriptor: c_format S32 (bits 4-5 = 2), a/b format u8 (0), both K-major, N>>3 at bit 17,
// M>>4 at bit 24 (CUTLASS UMMA::InstrDescriptor layout).
constexpr uint32_t MMA_IDESC = (2u << 4) | ((uint32_t)(MMA_BN >> 3) << 17) | ((uint32_t)(MMA_BM >> 4) << 24);

// Shared-memory matrix descriptor for a K-major operand in the canonical 128B-swizzle layout: 8-row
// atoms of 128 B, stride between atoms (SBO) 1024 B, LBO 16 B (unused when swizzled), version 1 (sm100),
// layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    return (uint64_t)((smem_addr >> 4) & 0x3fffu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tm, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Per-pair heavy-set bookkeeping lives in PairState (heavy_h); tile (rb, cb) enumeration over the blocks
// that touch the strict upper triangle (some b > a): cb >= rb/2.
__device__ __forceinline__ bool mma_tile_coords(int t, int hp, int* rb_out, int* cb_out) {
    const int RB = hp / MMA_BM, CB = hp / MMA_BN;
    for (int rb = 0; rb < RB; ++rb) {
        const int c0 = rb / 2;
        const int cnt = CB - c0;
        if (t < cnt) { *rb_out = rb; *cb_out = c0 + t; return true; }
        t -= cnt;
    }
    return false;
}

__global__ void __launch_bounds__(MMA_THREADS, 1) k_sc2_mma(const __grid_constant__ CUtensorMap tmX, WS ws) {
    extern __shared__ uint8_t smem_raw[];
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    if (d.n == 0) return;
    const int h = ws.st[p].heavy_h;
    if (h == 0) return;
    const int hp = (h + MMA_BN - 1) / MMA_BN * MMA_BN;
    int rb, cb;
    if (!mma_tile_coords(blockIdx.x, hp, &rb, &cb)) return;
    // K = every column (32 W, a multiple of 128), or the non-sparse columns padded to 128 (sc2_variant bit 2)
    const int KB = (ws.sc2_variant & 4) ? (ws.st[p].n_dense + MMA_BK - 1) / MMA_BK : d.W * 32 / MMA_BK;

    const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t tiles = (base + 1023u) & ~1023u;  // 1024-byte aligned for the 128B swizzle
    const uint32_t bars = tiles + MMA_STAGES * MMA_STAGE_BYTES;
    // barriers: full[s] at bars + 8s, empty[s] at bars + 64 + 8s, accum at bars + 128; tmem ptr at bars + 192
    const uint32_t full0 = bars, empty0 = bars + 64, accum = bars + 128, tptr = bars + 192;
    uint8_t* gen_tptr = smem_raw + (tptr - base);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < MMA_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(accum, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    }
    if (warp == 1) {  // TMEM: 256 columns × 128 lanes of 32-bit = one M128×N256 int32 accumulator
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(tptr));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gen_tptr);

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % MMA_STAGES;
                const int round = kb / MMA_STAGES;
                if (round > 0) mbar_wait(empty0 + 8 * s, (round - 1) & 1);
                const uint32_t a_dst = tiles + s * MMA_STAGE_BYTES;
                const uint32_t b_dst = a_dst + MMA_A_BYTES;
                mbar_expect_tx(full0 + 8 * s, MMA_STAGE_BYTES);
                tma_load_3d(a_dst, &tmX, full0 + 8 * s, kb * MMA_BK, rb * MMA_BM, p);
                tma_load_3d(b_dst, &tmX, full0 + 8 * s, kb * MMA_BK, cb * MMA_BN, p);
                tma_load_3d(b_dst + MMA_A_BYTES, &tmX, full0 + 8 * s, kb * MMA_BK, cb * MMA_BN + 128, p);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // single-thread MMA issuer
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % MMA_STAGES;
                mbar_wait(full0 + 8 * s, (kb / MMA_STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a_src = tiles + s * MMA_STAGE_BYTES;
                const uint32_t b_src = a_src + MMA_A_BYTES;
#pragma unroll
                for (int k = 0; k < MMA_BK / 32; ++k) {
                    umma_i8(tmem, umma_desc_sw128(a_src + 32 * k), umma_desc_sw128(b_src + 32 * k), MMA_IDESC,
                            (kb | k) ? 1u : 0u);
                }
                umma_commit(empty0 + 8 * s);  // frees the smem stage once these MMAs completed
            }
            umma_commit(accum);
        }
    } else {  // epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
        const int q = warp & 3;
        mbar_wait(accum, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int a = rb * MMA_BM + q * 32 + lane;  // output row = TMEM lane
        uint16_t* D = ws.heavy_D + p * ws.heavy_D_stride + (int64_t)a * ws.heavy_cap;
#pragma unroll 1
        for (int c = 0; c < MMA_BN / 32; ++c) {
            uint32_t v[32];
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (a < h) {
                uint4* dst = reinterpret_cast<uint4*>(D + cb * MMA_BN + c * 32);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint4 o;
                    o.x = (v[8 * k + 0] & 0xffffu) | (v[8 * k + 1] << 16);
                    o.y = (v[8 * k + 2] & 0xffffu) | (v[8 * k + 3] << 16);
                    o.z = (v[8 * k + 4] & 0xffffu) | (v[8 * k + 5] << 16);
                    o.w = (v[8 * k + 6] & 0xffffu) | (v[8 * k + 7] << 16);
                    dst[k] = o;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

// CUDA-core cross-check of the same contraction (sc2_path = 2): D = X X^T with __dp4a, 64×64 tiles.
__global__ void __launch_bounds__(256) k_sc2_dp4a(WS ws) {
    __shared__ uint32_t sa[64][33];
    __shared__ uint32_t sb[64][33];
    const int p = blockIdx.z;
    const PairDesc d = ws.desc[p];
    if (d.n == 0) return;
    const int h = ws.st[p].heavy_h;
    const int a0 = blockIdx.y * 64, b0 = blockIdx.x * 64;
    if (a0 >= h || b0 >= h || b0 + 63 < a0) return;
    const int K = (ws.sc2_variant & 4) ? (ws.st[p].n_dense + MMA_BK - 1) / MMA_BK * MMA_BK : d.W * 32;
    const uint8_t* X = ws.heavy_X + p * ws.heavy_X_stride;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    uint32_t acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 128) {
        for (int e = threadIdx.x; e < 64 * 32; e += 256) {
            const int r = e >> 5, w = e & 31;
            sa[r][w] = *reinterpret_cast<const uint32_t*>(X + (int64_t)(a0 + r) * ws.heavy_Kcap + k0 + 4 * w);
            sb[r][w] = *reinterpret_cast<const uint32_t*>(X + (int64_t)(b0 + r) * ws.heavy_Kcap + k0 + 4 * w);
        }
        __syncthreads();
        for (int w = 0; w < 32; ++w)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __dp4a(sa[ty * 4 + i][w], sb[tx * 4 + j][w], acc[i][j]);
        __syncthreads();
    }
    uint16_t* D = ws.heavy_D + p * ws.heavy_D_stride;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            D[(int64_t)(a0 + ty * 4 + i) * ws.heavy_cap + b0 + tx * 4 + j] = (uint16_t)acc[i][j];
}

}  // namespace trk
