// =====================================================================================================
// SC^2 on the dense block: Ĝ = C ⊙ (C·C) (Eq. 2) restricted to the "heavy" rows H (the
// high-degree rows — on registration workloads the inliers, whose mutual compatibility is dense).
// C·C over H is a dense binary contraction, so it runs on the 5th-gen tensor cores:
//   X = C[H, :] (K-major, [h][K]),  D = X · X^T  (exact: every product is 0 or 1, every count < 2^24)
// by default as packed e2m1 (bit → 1.0 / 0.0) with tcgen05.mma kind::mxf4.block_scale (M=128, N=240,
// K=64 per instruction, unit UE8M0 block scales in TMEM, fp32 accumulate); option mma_fp4 = 0 runs uint8
// 0/1 operands with kind::i8 (M=128, N=256, K=32, int32 accumulate).  Operands are staged by TMA
// (cp.async.bulk.tensor, 128B swizzle) through a 4-stage mbarrier pipeline.
// Persistent: one CTA per SM walks the (pair, tile) list of the whole batch (or one rank's tile range of a
// split pair); the accumulator is double buffered in TMEM (2 × 256 columns) so the epilogue of tile t
// overlaps the MMAs of tile t+1.  The epilogue (16 warps, 4 per TMEM lane quarter, tcgen05.ld 32x32b)
// does not store D: it transposes 32×32 chunks through shared memory (lane = column), keeps the entries
// that are O2 edges — b > a and C[H_a][H_b] = 1, tested on row H_a's upper words — and writes each
// straight to its slot in the compact edge list, rowptr(H_a) + rank of H_b in U_{H_a} (prefix counts
// per word from k_expand).  Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + single-thread
// MMA issuer, warps 2..17 = epilogue.  Which rows are heavy only changes speed.
// =====================================================================================================
#pragma once
#include <cuda.h>
#include <cstdint>

namespace trk {

constexpr int MMA_BM = 128;
constexpr int MMA_BN = 256;
constexpr int MMA_BK = 128;  // bytes = int8 elements per stage per row
constexpr int MMA_STAGES = 4;
constexpr int MMA_TILE_RING = 4;  // dynamic tile ids in flight between the producer and the consumers
constexpr int MMA_A_BYTES = MMA_BM * MMA_BK;  // 16 KB
constexpr int MMA_B_BYTES = MMA_BN * MMA_BK;  // 32 KB
constexpr int MMA_STAGE_BYTES = MMA_A_BYTES + MMA_B_BYTES;
constexpr int MMA_EPI_WARPS = 16;  // 4 per TMEM lane quarter; sub-warp k drains 32-column chunks k, k+4
constexpr int MMA_EPI_SUB = MMA_EPI_WARPS / 4;
constexpr int MMA_TABLE_PAIRS = 1024;  // pair table in shared memory (larger batches: k_tile_table's global one)
constexpr int MMA_SMEM_BYTES = MMA_STAGES * MMA_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                               (2 * MMA_TABLE_PAIRS + 1) * 4 /*tile prefix + |H| per pair*/ +
                               MMA_EPI_WARPS * 16 * 34 * 2 /*transpose*/ + MMA_EPI_WARPS * 32 * 4 /*row bases*/;
constexpr int MMA_THREADS = 64 + 32 * MMA_EPI_WARPS;

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
// X tiles are re-read by every tile of their pair (35 per config-E pair): loaded with an L2 evict_last policy
// so the pair's operand block stays in L2 while the edge stores stream past it.
__device__ __forceinline__ uint64_t l2_tile_policy(int which) {
    uint64_t pol;
    if (which == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else if (which == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tm, uint32_t bar, int c0, int c1, int c2,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// Block-scaled instruction descriptor (CUTLASS UMMA::InstrDescriptorBlockScaled): a/b format E2M1 (1) at
// bits 7 / 10, N>>3 at 17, scale format UE8M0 at 23, M>>4 at 24, scale-factor ids 0, K = 64.
constexpr uint32_t MMA_IDESC_MXF4 = (1u << 7) | (1u << 10) | ((uint32_t)(240 >> 3) << 17) | (1u << 23) |
                                    ((uint32_t)(MMA_BM >> 4) << 24);
__device__ __forceinline__ void umma_mxf4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t tmem_sf, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(tmem_sf));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Tiles (rb, cb) of one pair: 128-row × TN-column blocks (TN = 256 for int8, 240 for the block-scaled
// fp4 path) that touch the strict upper triangle (some b > a): cb >= rb·128 / TN.
__device__ __forceinline__ int mma_tile_count(int h, int TN) {
    const int RB = (h + MMA_BM - 1) / MMA_BM, CB = (h + TN - 1) / TN;
    int t = 0;
    for (int rb = 0; rb < RB; ++rb) t += CB - rb * MMA_BM / TN;
    return t;
}
__device__ __forceinline__ void mma_tile_coords(int t, int h, int TN, int* rb_out, int* cb_out) {
    const int RB = (h + MMA_BM - 1) / MMA_BM, CB = (h + TN - 1) / TN;
    for (int rb = 0; rb < RB; ++rb) {
        const int c0 = rb * MMA_BM / TN;
        const int cnt = CB - c0;
        if (t < cnt) { *rb_out = rb; *cb_out = c0 + t; return; }
        t -= cnt;
    }
    *rb_out = *cb_out = 0;
}
// Global tile g of the batch -> (pair, rb, cb) from the tile-count prefix and |H| per pair: a shared-memory
// table built once per CTA for batches up to MMA_TABLE_PAIRS, else k_tile_table's global one (L1-cached);
// each role walks its tiles in increasing g, so the pair cursor only moves forward.
struct TableCursor {
    const int32_t* pre;  // [batch + 1] exclusive prefix of the pairs' tile counts
    const int32_t* hh;   // [batch] |H| per pair
    int TN;
    int p = 0;
    __device__ bool locate(int batch, int g, int* pp, int* rb, int* cb, int* h) {
        if (g >= pre[batch]) return false;
        while (pre[p + 1] <= g) ++p;
        *pp = p;
        *h = hh[p];
        mma_tile_coords(g - pre[p], *h, TN, rb, cb);
        return true;
    }
};

// The batch's tile table for batches beyond the shared-memory table (k_sc2_mma reads it through L1): one
// block, a scan of the pairs' tile counts.
__global__ void __launch_bounds__(1024) k_tile_table(WS ws, int batch, int TN) {
    __shared__ int s_w[32];
    __shared__ int s_carry;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) s_carry = 0;
    __syncthreads();
    for (int q0 = 0; q0 < batch; q0 += 1024) {
        const int q = q0 + t;
        const int hq = (q < batch && ws.desc[q].n != 0) ? ws.st[q].heavy_h : 0;
        const int c = hq ? mma_tile_count(hq, TN) : 0;
        const int x = warp_incl_scan(c);
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const int y = s_w[lane];
            s_w[lane] = warp_incl_scan(y) - y;
        }
        __syncthreads();
        if (q < batch) {
            ws.tile_tab[q + 1] = s_carry + s_w[warp] + x;
            ws.tile_tab[batch + 1 + q] = hq;
        }
        __syncthreads();
        if (t == 1023) s_carry += s_w[31] + x;
        __syncthreads();
    }
    if (t == 0) ws.tile_tab[0] = 0;
}

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// FP4: X holds packed e2m1 (1.0 / 0.0 per bit, two per byte) and the contraction runs as
// tcgen05.mma kind::mxf4.block_scale (K = 64 per instruction, every block scale 2^0 in TMEM, fp32
// accumulate — exact for counts < 2^24) on 128×240 tiles, so the two accumulators (columns 0 and 256)
// leave TMEM columns 496.. for the scale factors.
template <bool FP4>
__global__ void __launch_bounds__(MMA_THREADS, 1) k_sc2_mma(const __grid_constant__ CUtensorMap tmX, WS ws, int batch) {
    constexpr int TN = FP4 ? 240 : MMA_BN;  // tile columns
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t tiles = (base + 1023u) & ~1023u;  // 1024-byte aligned for the 128B swizzle
    const uint32_t bars = tiles + MMA_STAGES * MMA_STAGE_BYTES;
    // barriers: full[s] at bars + 8s, empty[s] at bars + 64 + 8s, tmem_full[2] at bars + 128,
    // tmem_empty[2] at bars + 144; tile ring: tile_full[r] at bars + 32 + 8r, tile_empty[r] at bars + 96 + 8r,
    // tile ids at bars + 160 + 4r; tmem ptr at bars + 192
    const uint32_t full0 = bars, empty0 = bars + 64, tfull0 = bars + 128, tempty0 = bars + 144, tptr = bars + 192;
    const uint32_t gfull0 = bars + 32, gempty0 = bars + 96;
    volatile int32_t* s_tg = reinterpret_cast<volatile int32_t*>(smem_raw + (bars + 160 - base));
    uint8_t* gen_tptr = smem_raw + (tptr - base);
    uint16_t* s_vt = reinterpret_cast<uint16_t*>(smem_raw + (bars + 256 - base));  // [warps][16][34] (Ĝ < 65536)
    int32_t* s_eb = reinterpret_cast<int32_t*>(s_vt + MMA_EPI_WARPS * 16 * 34);     // [warps][32] edge-list bases
    int32_t* s_tpre = s_eb + MMA_EPI_WARPS * 32;                                    // [batch + 1] tile prefix
    int32_t* s_th = s_tpre + MMA_TABLE_PAIRS + 1;                                 // [batch] |H|
    const bool smem_table = batch <= MMA_TABLE_PAIRS;
    const int32_t* t_pre = smem_table ? s_tpre : ws.tile_tab;
    const int32_t* t_h = smem_table ? s_th : ws.tile_tab + batch + 1;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // warp: provably uniform

    if (threadIdx.x == 0) {
        for (int s = 0; s < MMA_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, MMA_EPI_WARPS);  // one arrive per epilogue warp
        }
        for (int r = 0; r < MMA_TILE_RING; ++r) {
            mbar_init(gfull0 + 8 * r, 1);
            mbar_init(gempty0 + 8 * r, 1 + MMA_EPI_WARPS);  // the MMA issuer and every epilogue warp read it
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    }
    if (warp == 1) {  // TMEM: 2 × 256 columns × 128 lanes of 32-bit = two M128×N256 int32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tptr));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (smem_table) {  // tile counts per pair, then their exclusive prefix (warp 0)
        for (int q = threadIdx.x; q < batch; q += blockDim.x) {
            const int hq = (ws.desc[q].n == 0) ? 0 : ws.st[q].heavy_h;
            s_th[q] = hq;
            s_tpre[q + 1] = hq ? mma_tile_count(hq, TN) : 0;
        }
        __syncthreads();
        if (warp == 0) {
            int carry = 0;
            for (int q0 = 0; q0 < batch; q0 += 32) {
                const int c = (q0 + lane < batch) ? s_tpre[q0 + lane + 1] : 0;
                const int incl = warp_incl_scan(c);
                if (q0 + lane < batch) s_tpre[q0 + lane + 1] = carry + incl;
                carry += __shfl_sync(FULL, incl, 31);
            }
            if (lane == 0) s_tpre[0] = 0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gen_tptr);
    // global tile range of this launch: every tile, or this rank's share of a split pair (batch 1, table)
    int g_lo = 0, g_hi = 0x7fffffff;
    if (ws.split_world > 1) split_range(ws, t_pre[batch], &g_lo, &g_hi);
    // Dynamic tile scheduling: the producer takes the next global tile from ws.tile_ctr and publishes it in a
    // shared-memory ring read by the MMA issuer and the epilogue warps (−1 = no more tiles).  The CTAs then
    // work on one narrow window of the (pair, tile) list at any time, so a pair's X rows are fetched from
    // HBM about once and re-read from L2 by its other tiles (static striding let the CTAs drift apart).
    auto tile_get = [&](int lt) {  // consumers: wait for the ring slot of tile lt, read it
        const int r = lt % MMA_TILE_RING;
        mbar_wait(gfull0 + 8 * r, (lt / MMA_TILE_RING) & 1);
        return s_tg[r];
    };
    auto tile_release = [&](int lt) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gempty0 + 8 * (lt % MMA_TILE_RING)) : "memory");
    };
    if constexpr (FP4) {  // block scales: UE8M0 127 (= 1.0) in every byte of columns 496..511
        if (warp >= 2 && warp < 6) {
            const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 496u;
            const uint32_t one = 0x7f7f7f7fu;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    taddr),
                "r"(one)
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            TableCursor tc{t_pre, t_h, TN};
            int it = 0;
            int p, rb, cb, h;
            const uint64_t pol = l2_tile_policy(ws.mma_l2);
            for (int lt = 0;; ++lt) {
                const int r = lt % MMA_TILE_RING;
                if (lt >= MMA_TILE_RING) mbar_wait(gempty0 + 8 * r, (lt / MMA_TILE_RING - 1) & 1);
                int g = g_lo + atomicAdd(ws.tile_ctr, 1);
                if (!(g < g_hi && tc.locate(batch, g, &p, &rb, &cb, &h))) g = -1;
                s_tg[r] = g;
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gfull0 + 8 * r) : "memory");
                if (g < 0) break;
                const int KB = FP4 ? (ws.desc[p].W * 16 + MMA_BK - 1) / MMA_BK : ws.desc[p].W * 32 / MMA_BK;
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % MMA_STAGES;
                    const int round = it / MMA_STAGES;
                    if (round > 0) mbar_wait(empty0 + 8 * s, (round - 1) & 1);
                    const uint32_t a_dst = tiles + s * MMA_STAGE_BYTES;
                    const uint32_t b_dst = a_dst + MMA_A_BYTES;
                    mbar_expect_tx(full0 + 8 * s, MMA_STAGE_BYTES);
                    tma_load_3d(a_dst, &tmX, full0 + 8 * s, kb * MMA_BK, rb * MMA_BM, ws.pair_base + p, pol);
                    tma_load_3d(b_dst, &tmX, full0 + 8 * s, kb * MMA_BK, cb * TN, ws.pair_base + p, pol);
                    tma_load_3d(b_dst + MMA_A_BYTES, &tmX, full0 + 8 * s, kb * MMA_BK, cb * TN + 128, ws.pair_base + p, pol);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // single-thread MMA issuer
            TableCursor tc{t_pre, t_h, TN};
            int it = 0;
            int p, rb, cb, h;
            for (int lt = 0;; ++lt) {
                const int g = tile_get(lt);
                tile_release(lt);
                if (g < 0) break;
                tc.locate(batch, g, &p, &rb, &cb, &h);
                const int KB = FP4 ? (ws.desc[p].W * 16 + MMA_BK - 1) / MMA_BK : ws.desc[p].W * 32 / MMA_BK;
                const int acc = lt & 1;
                if (lt >= 2) mbar_wait(tempty0 + 8 * acc, ((lt >> 1) - 1) & 1);  // epilogue drained it
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t tacc = tmem + (uint32_t)(acc * MMA_BN);
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % MMA_STAGES;
                    mbar_wait(full0 + 8 * s, (it / MMA_STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t a_src = tiles + s * MMA_STAGE_BYTES;
                    const uint32_t b_src = a_src + MMA_A_BYTES;
#pragma unroll
                    for (int k = 0; k < MMA_BK / 32; ++k) {
                        if constexpr (FP4)
                            umma_mxf4(tacc, umma_desc_sw128(a_src + 32 * k), umma_desc_sw128(b_src + 32 * k),
                                      MMA_IDESC_MXF4, tmem + 496u, (kb | k) ? 1u : 0u);
                        else
                            umma_i8(tacc, umma_desc_sw128(a_src + 32 * k), umma_desc_sw128(b_src + 32 * k), MMA_IDESC,
                                    (kb | k) ? 1u : 0u);
                    }
                    umma_commit(empty0 + 8 * s);  // frees the smem stage once these MMAs completed
                }
                umma_commit(tfull0 + 8 * acc);  // accumulator complete
            }
        }
    } else {  // epilogue: warp w owns TMEM lane quarter w % 4 and the chunks c ≡ (w - 2) / 4 mod MMA_EPI_SUB
        const int q = warp & 3;
        const int ew = warp - 2;           // 0 .. MMA_EPI_WARPS-1
        const int sub = ew >> 2;
        constexpr int NCH = MMA_BN / 32;
        const int last_c = sub + (NCH - 1 - sub) / MMA_EPI_SUB * MMA_EPI_SUB;
        TableCursor tc{t_pre, t_h, TN};
        auto locate = [&](int gq, int* pp, int* rbp, int* cbp, int* hp) {
            return gq >= 0 && tc.locate(batch, gq, pp, rbp, cbp, hp);
        };
        auto epi_tile = [&](int lt) {  // every lane reads the slot; lane 0 releases it for the warp
            const int gq = tile_get(lt);
            __syncwarp();
            if (lane == 0) tile_release(lt);
            return gq;
        };
        // per-warp tile metadata in registers (no block barrier between tiles): the heavy ids of this warp's
        // columns (lane = column of chunks sub and sub + MMA_EPI_SUB) and its rows' edge-list bases (lane =
        // row, in this warp's shared-memory slot); tile t+1's are loaded while tile t is drained
        static_assert(MMA_BN / 32 == 2 * MMA_EPI_SUB, "two chunks per epilogue warp");
        auto col_id = [&](const int32_t* hlq, int cbq, int hq, int c) {
            const int k = c * 32 + lane;
            return (k < TN && cbq * TN + k < hq) ? __ldg(hlq + cbq * TN + k) : -1;
        };
        int p, rb, cb, h;
        int g = epi_tile(0);
        bool have = locate(g, &p, &rb, &cb, &h);
        int jb0 = -1, jb1 = -1;
        if (have) {
            const int32_t* hlist = ws.heavy_list + p * ws.heavy_cap;
            jb0 = col_id(hlist, cb, h, sub);
            jb1 = col_id(hlist, cb, h, sub + MMA_EPI_SUB);
            const int a = rb * MMA_BM + q * 32 + lane;
            s_eb[ew * 32 + lane] = a < h ? __ldg(ws.rowptr + p * ws.rp_stride + __ldg(hlist + a)) : -1;
        }
        __syncwarp();
        for (int lt = 0; have; ++lt) {
            const int acc = lt & 1;
            int pn, rbn, cbn, hn;
            const int gn = epi_tile(lt + 1);
            const bool next = locate(gn, &pn, &rbn, &cbn, &hn);
            int jbn0 = -1, jbn1 = -1, ja_n = -1, eb_n = -1;
            if (next) {
                const int32_t* hln = ws.heavy_list + pn * ws.heavy_cap;
                jbn0 = col_id(hln, cbn, hn, sub);
                jbn1 = col_id(hln, cbn, hn, sub + MMA_EPI_SUB);
                const int an = rbn * MMA_BM + q * 32 + lane;
                if (an < hn) ja_n = __ldg(hln + an);
                const int c0 = cbn * TN, c1 = min(hn, c0 + TN) - 1;
                if (sub == 0 && an < min(hn, c1)) {  // L2 prefetch of the next tile's (U word, prefix) row segment
                    const int64_t Wn = ws.desc[pn].W;
                    const int64_t w0 = __ldg(hln + c0) >> 5, w1 = __ldg(hln + c1) >> 5;
                    const int64_t s0 = ((an * Wn + w0) * 8) & ~15ll, e0 = ((an * Wn + w1 + 1) * 8 + 15) & ~15ll;
                    const char* upn = reinterpret_cast<const char*>(ws.heavy_UP + pn * ws.heavy_UP_stride);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(upn + s0), "r"((uint32_t)(e0 - s0))
                                 : "memory");
                }
            }
            const int W = ws.desc[p].W;
            const uint2* up0 = ws.heavy_UP + p * ws.heavy_UP_stride;
            uint32_t* edges = ws.edges + p * ws.edges_stride;
            asm("" : "+l"(edges));  // keep the base in registers (ptxas otherwise recomputes it per store)
            uint16_t* vt = s_vt + ew * 16 * 34;  // this warp's 16×32 transpose buffer
            const int bt = cb * TN;
            mbar_wait(tfull0 + 8 * acc, (lt >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int c = sub; c < NCH; c += MMA_EPI_SUB) {
                const int b = bt + c * 32 + lane;
                const int jb = (c == sub) ? jb0 : jb1;
                const int a0 = rb * MMA_BM + q * 32;
                // rows r < lim of this warp are heavy rows (a0 + r < h) below the lane's column (b > a0 + r)
                const int lim = jb >= 0 ? min(b - a0, h - a0) : 0;
                if (__all_sync(FULL, lim <= 0)) {  // the chunk holds no upper pair (below the diagonal / beyond H)
                    if (c == last_c) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * acc) : "memory");
                    }
                    if (c == sub && ja_n >= 0) eb_n = __ldg(ws.rowptr + pn * ws.rp_stride + ja_n);
                    continue;
                }
                uint32_t v[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * MMA_BN + c * 32);
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
                if (c == last_c) {  // my chunks drained: hand the accumulator back to the MMA issuer
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * acc) : "memory");
                }
                // transpose through shared memory: afterwards lane = column, loop over the warp's 32 rows, so
                // the UP reads and edge stores of one row are coalesced
                const uint32_t bit = 1u << (jb & 31);
                const uint32_t jhi = (uint32_t)jb << 16, bm1 = bit - 1u;
                const char* upl = reinterpret_cast<const char*>(up0 + (size_t)a0 * W + (jb >= 0 ? (jb >> 5) : 0));
                const size_t W8 = (size_t)W * sizeof(uint2);
#pragma unroll
                for (int rh = 0; rh < 32; rh += 16) {  // rows rh .. rh+15 through a 16-row transpose buffer
                    __syncwarp();
                    if ((lane & 16) == rh) {  // two 16-bit values per 32-bit store
                        uint32_t* vr = reinterpret_cast<uint32_t*>(vt + (lane & 15) * 34);
#pragma unroll
                        for (int k = 0; k < 32; k += 2) {
                            uint32_t lo = v[k], hi = v[k + 1];
                            if constexpr (FP4) {  // exact integer-valued fp32 (< 2^23): + 2^23 puts it in the low mantissa bits
                                unsigned long long pr2 = (unsigned long long)lo | ((unsigned long long)hi << 32);
                                asm("add.rn.f32x2 %0, %0, %1;" : "+l"(pr2) : "l"(0x4b0000004b000000ull));
                                lo = (uint32_t)pr2;
                                hi = (uint32_t)(pr2 >> 32);
                            }
                            vr[k >> 1] = __byte_perm(lo, hi, 0x5410);  // low halves of both
                        }
                    }
                    __syncwarp();
                    uint2 u[16];
                    const char* pr = upl + rh * W8;
                    // 16 rows' words in flight at once; unconditional (rows < heavy_cap, a multiple of 128, are
                    // inside the buffer) and masked by lim afterwards
#pragma unroll
                    for (int r = 0; r < 16; ++r, pr += W8) u[r] = __ldg(reinterpret_cast<const uint2*>(pr));
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        const uint32_t x = u[r].x;
                        const uint32_t slot = (uint32_t)(s_eb[ew * 32 + rh + r] + (int)u[r].y) + __popc(x & bm1);
                        if (rh + r < lim && (x & bit)) __stcs(edges + slot, jhi | vt[r * 34 + lane]);
                    }
                }
                __syncwarp();
                if (c == sub && ja_n >= 0) eb_n = __ldg(ws.rowptr + pn * ws.rp_stride + ja_n);
            }
            g = gn;
            p = pn, rb = rbn, cb = cbn, h = hn;
            jb0 = jbn0, jb1 = jbn1;
            s_eb[ew * 32 + lane] = eb_n;  // private to this warp: its reads of tile t are done
            __syncwarp();
            have = next;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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
    const int K = d.W * 32;
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

// Edge emission from D for the CUDA-core path: one warp per heavy row a, lanes over the columns b > a
// (same test and slot as the tensor-core epilogue).
__global__ void __launch_bounds__(256) k_emit_hh(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    if (d.n == 0) return;
    const int h = ws.st[p].heavy_h;
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a >= h) return;
    const int32_t* hlist = ws.heavy_list + p * ws.heavy_cap;
    const int ja = hlist[a];
    const int ebase = ws.rowptr[p * ws.rp_stride + ja];
    const uint2* up = ws.heavy_UP + p * ws.heavy_UP_stride + (int64_t)a * d.W;
    const uint16_t* Drow = ws.heavy_D + p * ws.heavy_D_stride + (int64_t)a * ws.heavy_cap;
    uint32_t* edges = ws.edges + p * ws.edges_stride;
    for (int b = a + 1 + lane; b < h; b += 32) {
        const int jb = hlist[b];
        const uint2 u = up[jb >> 5];
        const uint32_t bit = 1u << (jb & 31);
        if (u.x & bit) edges[ebase + (int)u.y + __popc(u.x & (bit - 1u))] = ((uint32_t)jb << 16) | Drow[b];
    }
}

}  // namespace trk
