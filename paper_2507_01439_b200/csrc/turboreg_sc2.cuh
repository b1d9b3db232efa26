// a3 SC^2 weights and the O2 edge lists (Eq. 2, Def. 2): degrees, heavy/sparse split, assembly.
// Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_compat.cuh"

namespace trk {

// ------------------------------------------------------------------------------------------ a3 SC^2
// Eq. 2 for every O2 edge (i < j), written as (j << 16 | Ĝ_ij) to edges[rowptr(i) + rank of j
// in U_i] (compact, rank-indexed rows).  Three passes write disjoint sets of edges:
//   * both endpoints heavy → the tensor-core epilogue (k_sc2_mma; k_emit_hh on the cross-check path);
//   * one endpoint dense (heavy, or degree > list_max) → k_sc2 below, from the dense row's side;
//   * both sparse → k_sc2_light.
// The pivot passes (turboreg_select.cuh) then histogram the positive weights for the radix select (Eq. 4).
constexpr int SC2_WARPS = 8;
// k_degree: rows per 8-warp block — 64 for small batches (enough blocks to fill the GPU), 256 for batches
// of >= 256 pairs (fewer, longer blocks: 1623 config-E pairs 1.34 -> 1.28 us/pair)
constexpr int DEG_ROWS_PER_BLOCK = 64, DEG_ROWS_PER_BLOCK_BIG = 256;  // k_degree: rows per 8-warp block
constexpr int SEL_WARPS = 8;
constexpr int SEL_ROWS_PER_BLOCK = 128;
#ifndef TRK_LIST_MAX
#define TRK_LIST_MAX 64
#endif
constexpr int LIST_MAX = TRK_LIST_MAX;  // rows with degree <= list_max keep a sorted uint16 neighbour list: 64, or
constexpr int LIST_MAX_BIG = 256;  // 256 for rows of more than 256 words (N > 8192, where outliers' degrees grow)
template <int WPL>
constexpr int list_max_of() { return WPL >= 16 ? LIST_MAX_BIG : LIST_MAX; }
constexpr int MMA_BK_ = 128;  // K granularity of the tensor-core block (= MMA_BK)
template <int WPL>
constexpr int sc2_qcap() { return WPL >= 8 ? 256 : 32 * WPL; }  // sparse-neighbour queue entries per warp
template <int WPL>
constexpr int sc2_warp_words() { return 64 * WPL + sc2_qcap<WPL>(); }  // row i, its U_i rank prefix, queue
template <int WPL>
constexpr int sc2_smem_bytes() { return (SC2_WARPS * sc2_warp_words<WPL>() + 2 * 32 * WPL) * 4; }

// Dense rows (not sparse: heavy, or degree > list_max), one warp per row i, SC2_BLOCKS_PER_PAIR blocks of
// warps striding over the pair's dense rows.  Row i's edges come from three sources:
//   (1) i, j both heavy: written by the tensor-core epilogue (k_sc2_mma) or k_emit_hh, not here;
//   (2) j sparse (degree <= list_max, sorted neighbour list L_j), on EITHER side of i:
//       Ĝ_ij = |L_j ∩ N(i)|, one edge per lane, list entries tested against row i's bitmap in shared
//       memory.  For j > i the result goes to row i's slot; for j < i to row j's slot, whose rank
//       (entries of L_j below i, minus those up to j) falls out of the same pass over L_j;
//   (3) both dense but not both heavy (rare since H takes every non-sparse row that fits its cap):
//       warp-cooperative popcount(row_i AND row_j).
// Sparse-sparse edges are k_sc2_light's.  Every O2 edge is therefore written exactly once.
// Blocks per pair: at least 64 (512 warps over its dense rows), 16 for batches of >= 128 pairs, where the
// grid is large anyway and fewer blocks amortise each block's staging of the row-class masks (1623 pairs:
// k_sc2 2.68 -> 2.49 us/pair)
constexpr int SC2_BLOCKS_PER_PAIR = 64, SC2_BLOCKS_PER_PAIR_BIG = 16;

// |L ∩ N(i)| for a sorted list L of <= LM uint16 entries (16-byte aligned, zero padded) against row i's
// bitmap in shared memory.  Entries past len are zeros, so a chunk is processed whole and the pad's bit 0
// tests are subtracted once (row i's own bit 0 is read once).  64 entries (8 chunks) are loaded before any
// is tested.
template <int LM>
__device__ __forceinline__ uint32_t list_bitmap_count(const uint16_t* L, int len, const uint32_t* sr) {
    const int nch = (len + 7) >> 3;
    uint32_t cnt = 0;
#pragma unroll 1
    for (int c0 = 0; c0 < nch; c0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
            v[c] = (c0 + c < nch) ? __ldg(reinterpret_cast<const uint4*>(L) + c0 + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c0 + c < nch) {
                const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t k0 = wv[e] & 0xffffu, k1 = wv[e] >> 16;
                    cnt += ((sr[k0 >> 5] >> (k0 & 31)) & 1u) + ((sr[k1 >> 5] >> (k1 & 31)) & 1u);
                }
            }
        }
        if (LM <= 64) break;
    }
    return cnt - (uint32_t)(nch * 8 - len) * (sr[0] & 1u);
}

// As list_bitmap_count, also returning lt = #{x in L : x < i} (pads included) for the edge's slot.  The
// comparison runs on both uint16 entries of a word at once: with c = 0x8000 + i − 1 in each half, the half
// c − x lies in [1, 0xfffe] for x, i < 2^15, so no borrow crosses halves and its bit 15 is [x < i].
template <int LM>
__device__ __forceinline__ uint32_t list_bitmap_count_lt(const uint16_t* L, int len, const uint32_t* sr, int i,
                                                         int* lt) {
    const int nch = (len + 7) >> 3;
    uint32_t cnt = 0, acc = 0;
    const uint32_t c1 = 0x8000u + (uint32_t)i - 1u, cpair = c1 | (c1 << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < nch; c0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
            v[c] = (c0 + c < nch) ? __ldg(reinterpret_cast<const uint4*>(L) + c0 + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c0 + c < nch) {
                const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t k0 = wv[e] & 0xffffu, k1 = wv[e] >> 16;
                    cnt += ((sr[k0 >> 5] >> (k0 & 31)) & 1u) + ((sr[k1 >> 5] >> (k1 & 31)) & 1u);
                    acc += ((cpair - wv[e]) >> 15) & 0x10001u;
                }
            }
        }
        if (LM <= 64) break;
    }
    *lt = (int)((acc & 0xffffu) + (acc >> 16));
    return cnt - (uint32_t)(nch * 8 - len) * (sr[0] & 1u);
}

// Edge between dense row i (bitmap sr and the exclusive prefix sp of U_i's popcounts per word in shared
// memory; U_i's words are sr's above i) and sparse row j, on either side of i: one code path for both sides.
// For j < i the edge lives in row j at rank #{x in L_j : j < x < i} = lt − pads − #{x in L_j : x < j}, the
// last being deg(j) − |U_j| = deg_full[j] − (rowptr[j + 1] − rowptr[j]).
template <int LM>
__device__ __forceinline__ void sc2_sparse_edge(const WS& ws, const uint16_t* lists, const int32_t* deg_full,
                                                const int32_t* rowptr, uint32_t* edges, uint32_t* erow,
                                                const int32_t* sp, const uint32_t* sr, int i, int j) {
    const uint16_t* L = lists + (int64_t)j * LM;
    const int len = deg_full[j];
    int lt;
    const uint32_t c = list_bitmap_count_lt<LM>(L, len, sr, i, &lt);
    const int wj = j >> 5;
    uint32_t* dst;
    if (j > i) {
        dst = erow + sp[wj] + __popc(upper_mask(sr[wj], wj, i) & ((1u << (j & 31)) - 1u));
    } else {
        const int r0 = rowptr[j], r1 = rowptr[j + 1];
        const int pads = ((len + 7) & ~7) - len;
        dst = edges + r0 + (lt - pads - (len - (r1 - r0)));
    }
    *dst = ((uint32_t)((j > i) ? j : i) << 16) | c;
}

template <int WPL>
#ifndef TRK_SC2_MINB
#define TRK_SC2_MINB 4
#endif
__global__ void __launch_bounds__(SC2_WARPS * 32, (WPL >= 16 ? 2 : WPL >= 8 ? 3 : TRK_SC2_MINB)) k_sc2(WS ws, int cpi) {
    constexpr int G = 4;
    constexpr int QCAP = sc2_qcap<WPL>();  // sparse-neighbour queue (a round adds at most 32 entries)
    extern __shared__ uint32_t s_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // block: heavy mask, sparse mask; per warp: row i, rank prefix of U_i per word, queue (U_i's words are
    // row i's above i, recomputed where needed: a smaller footprint keeps large-N rows at 2 blocks per SM)
    uint32_t* hm = s_dyn;
    uint32_t* lm = s_dyn + 32 * WPL;
    uint32_t* sr = s_dyn + 64 * WPL + warp * sc2_warp_words<WPL>();
    int32_t* sp = reinterpret_cast<int32_t*>(sr + 32 * WPL);
    uint32_t* sq = sr + 64 * WPL;
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int nd = ws.st[p].n_dense;
    const int W = d.W;
    const int nchunks = (W + 31) >> 5;
    const int mstride = ws.bits_stride / ws.row_stride;
    for (int w = threadIdx.x; w < 32 * WPL; w += blockDim.x) {
        hm[w] = (w < W) ? ws.heavy_mask[p * mstride + w] : 0u;
        lm[w] = (w < W) ? ws.light_mask[p * mstride + w] : 0u;
    }
    __syncthreads();
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    const int32_t* deg_full = ws.deg_full + p * ws.row_stride;
    const uint16_t* lists = ws.lists + p * ws.lists_stride;
    const int32_t* hpos = ws.hpos + p * ws.row_stride;
    const int32_t* rowptr = ws.rowptr + p * ws.rp_stride;
    uint32_t* edges = ws.edges + p * ws.edges_stride;
    const int nw = gridDim.x * SC2_WARPS;
    // work item = (dense row, group of cpi 32-word chunks of its row): rows with many dense neighbours
    // are spread over several warps
    const int ngrp = (nchunks + cpi - 1) / cpi;
    int it_lo, it_hi;  // this rank's items (all of them unless the pair is split over ranks)
    split_range(ws, nd * ngrp, &it_lo, &it_hi);
    for (int item = it_lo + blockIdx.x * SC2_WARPS + warp; item < it_hi; item += nw) {
        const int kq = item / ngrp, c_lo = (item - kq * ngrp) * cpi, c_hi = min(nchunks, c_lo + cpi);
        const int i = ws.dense_list[p * ws.row_stride + kq];
        const uint32_t* ri = bits + (int64_t)i * W;
        const int hi = hpos[i];
        uint32_t* erow = edges + rowptr[i];
        uint32_t reg[WPL];
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            const int w = lane + 32 * k;
            reg[k] = (w < W) ? ri[w] : 0u;
        }
        {
            int carry = 0;
#pragma unroll
            for (int k = 0; k < WPL; ++k) {
                const int w = lane + 32 * k;
                const uint32_t u = (w < W) ? upper_mask(reg[k], w, i) : 0u;
                const int cnt = __popc(u);
                const int incl = warp_incl_scan(cnt);
                sr[w] = reg[k];
                sp[w] = carry + incl - cnt;
                carry += __shfl_sync(FULL, incl, 31);
            }
        }
        __syncwarp();
        // (2) sparse neighbours on both sides, queued (one edge per lane) and (3) dense-dense upper
        // neighbours that are not both heavy (warp-cooperative popcount).  A chunk's sparse neighbours enter
        // the queue in one pass: each lane writes its word's bits at its prefix offset (virtual positions
        // from nq; full windows of QCAP entries are processed as they fill).
        int nq = 0;
        for (int c = c_lo; c < c_hi; ++c) {
            const int w = c * 32 + lane;
            const uint32_t lmw = (w < W) ? lm[w] : 0u;
            const uint32_t srw = (w < W) ? sr[w] : 0u;
            uint32_t ul = srw & lmw;
            uint32_t ud = (w < W) ? upper_mask(srw, w, i) & ~lmw : 0u;
            if (hi >= 0 && w < W) ud &= ~hm[w];
            const int cl = __popc(ul);
            const int incl = warp_incl_scan(cl);
            const int vend = nq + __shfl_sync(FULL, incl, 31);
            int o = nq + incl - cl, qbase = 0;
            while (vend - qbase > QCAP) {  // rare: the queue fills inside this chunk
                while (ul && o < qbase + QCAP) {
                    const int b = 31 - __clz(ul);
                    ul &= ~(0xffffffffu << b);
                    sq[o++ - qbase] = (uint32_t)(w * 32 + b);
                }
                __syncwarp();
                for (int t = lane; t < QCAP; t += 32) sc2_sparse_edge<list_max_of<WPL>()>(ws, lists, deg_full, rowptr, edges, erow, sp, sr, i, (int)sq[t]);
                __syncwarp();
                qbase += QCAP;
            }
            while (ul) {
                const int b = 31 - __clz(ul);
                ul &= ~(0xffffffffu << b);
                sq[o++ - qbase] = (uint32_t)(w * 32 + b);
            }
            nq = vend - qbase;
            while (__any_sync(FULL, ud != 0u)) {
                int jd = -1;
                if (ud) {
                    jd = w * 32 + __ffs(ud) - 1;
                    ud &= ud - 1u;
                }
                unsigned lb = __ballot_sync(FULL, jd >= 0);
                while (lb) {
                    int jj[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        int src = -1;
                        if (lb) {
                            src = __ffs(lb) - 1;
                            lb &= lb - 1u;
                        }
                        jj[g] = __shfl_sync(FULL, jd, src < 0 ? 0 : src);
                        if (src < 0) jj[g] = -1;
                    }
                    uint32_t part[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        part[g] = 0u;
                        if (jj[g] >= 0) {
                            const uint32_t* rj = bits + (int64_t)jj[g] * W;
#pragma unroll
                            for (int k = 0; k < WPL; ++k) {
                                const int wk = lane + 32 * k;
                                if (wk < W) part[g] += __popc(reg[k] & __ldg(rj + wk));
                            }
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (jj[g] < 0) break;
                        const uint32_t tot = __reduce_add_sync(FULL, part[g]);
                        if (lane == g) {
                            const int j = jj[g], wj = j >> 5;
                            erow[sp[wj] + __popc(upper_mask(sr[wj], wj, i) & ((1u << (j & 31)) - 1u))] =
                                ((uint32_t)j << 16) | tot;
                        }
                    }
                }
            }
        }
        __syncwarp();
        for (int t = lane; t < nq; t += 32) sc2_sparse_edge<list_max_of<WPL>()>(ws, lists, deg_full, rowptr, edges, erow, sp, sr, i, (int)sq[t]);
        __syncwarp();
    }
}

// Row classes for the SC^2 assembly: sparse rows (a list, not heavy) go to k_sc2_light, the rest to k_sc2.
__global__ void __launch_bounds__(1024) k_rowclass(WS ws) {
    // one pass, 4 consecutive rows per thread (all loads issued up front): a block scan of (light flag,
    // upper degree) gives both the light/dense lists and the CSR row pointers
    constexpr int RPT = 4;
    __shared__ int s_wf[32], s_wu[32];
    __shared__ int s_cf, s_cu;
    const int p = blockIdx.x;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int32_t* deg = ws.deg_full + p * ws.row_stride;
    const int32_t* hpos = ws.hpos + p * ws.row_stride;
    const int32_t* udeg = ws.deg + p * ws.row_stride;
    int32_t* L = ws.light_list + p * ws.row_stride;
    int32_t* Dn = ws.dense_list + p * ws.row_stride;
    int32_t* rp = ws.rowptr + p * ws.rp_stride;
    uint32_t* lmask = ws.light_mask + p * (ws.bits_stride / ws.row_stride);
    if (ws.st[p].edge_overflow) {  // no room for this pair's edges: every row empty, nothing assembled
        for (int i = t; i <= n; i += 1024) rp[i] = 0;
        for (int w = t; w < d.W; w += 1024) lmask[w] = 0u;
        if (t == 0) { ws.st[p].n_light = 0; ws.st[p].n_dense = 0; ws.st[p].edges = 0; }
        return;
    }
    if (t == 0) s_cf = s_cu = 0;
    __syncthreads();
    for (int r0 = 0; r0 < n; r0 += 1024 * RPT) {
        const int ib = r0 + t * RPT;
        int fl[RPT], ud[RPT], fs = 0, us = 0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int i = ib + k;
            fl[k] = (i < n && hpos[i] < 0 && deg[i] <= ws.list_max) ? 1 : 0;
            ud[k] = i < n ? udeg[i] : 0;
            fs += fl[k];
            us += ud[k];
        }
        const int xf = warp_incl_scan(fs), xu = warp_incl_scan(us);
        if (lane == 31) { s_wf[warp] = xf; s_wu[warp] = xu; }
        __syncthreads();
        if (warp == 0) {
            const int yf = s_wf[lane], yu = s_wu[lane];
            const int zf = warp_incl_scan(yf), zu = warp_incl_scan(yu);
            s_wf[lane] = zf - yf;
            s_wu[lane] = zu - yu;
        }
        __syncthreads();
        int pf = s_cf + s_wf[warp] + xf - fs, pu = s_cu + s_wu[warp] + xu - us;
        uint32_t nib = 0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int i = ib + k;
            if (i < n) {
                if (fl[k]) L[pf] = i;
                else Dn[i - pf] = i;
                rp[i] = pu;
            }
            pf += fl[k];
            pu += ud[k];
            nib |= (uint32_t)fl[k] << k;
        }
        // light-row bitset: 8 threads x 4 rows = one 32-bit word
        uint32_t wbits = nib << (RPT * (lane & 7));
        wbits |= __shfl_xor_sync(FULL, wbits, 1);
        wbits |= __shfl_xor_sync(FULL, wbits, 2);
        wbits |= __shfl_xor_sync(FULL, wbits, 4);
        const int w = ib >> 5;
        if ((lane & 7) == 0 && w < d.W) lmask[w] = wbits;  // words past n (up to W) are written as 0
        __syncthreads();
        if (t == 1023) { s_cf = pf; s_cu = pu; }
        __syncthreads();
    }
    if (t == 0) {
        ws.st[p].n_light = s_cf;
        ws.st[p].n_dense = n - s_cf;
        rp[n] = s_cu;
        ws.st[p].edges = s_cu;
    }
}

// NEXT(1) split mode: every rank assembles only its share of the edges, so the pair's E edge words are
// cleared first (the ranks' arrays are then summed: each word is written by exactly one rank).
__global__ void __launch_bounds__(256) k_zero_edges(WS ws) {
    const int p = blockIdx.y;
    if (ws.desc[p].n == 0) return;
    const int E = ws.st[p].edges;
    uint32_t* e = ws.edges + p * ws.edges_stride;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < E; k += gridDim.x * blockDim.x) e[k] = 0u;
}

// SC^2 edges of the sparse rows, packed for full lanes: a warp takes LG sparse rows (bitmaps and lists
// staged in shared memory), enumerates all their upper edges, and pushes them into two queues — j sparse
// (|L_j ∩ N(i)| against row i's bitmap) and j dense (|L_i ∩ N(j)| against row j's words) — each flushed
// 32 edges at a time, one edge per lane.
// 16-byte asynchronous global -> shared copy (LDGSTS), completed by cp.async.wait_all.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}

template <int WPL>
#ifndef TRK_LIGHT_LG
#define TRK_LIGHT_LG 8
#endif
constexpr int light_rows() { return WPL >= 16 ? 2 : TRK_LIGHT_LG; }  // LG: sparse rows per warp group
template <int WPL, int LG = light_rows<WPL>()>
constexpr int light_warp_words() {
    return LG * 32 * WPL + LG * (list_max_of<WPL>() / 2) + 64 + 64 + 4 * LG;
}
template <int WPL, int LG = light_rows<WPL>()>
constexpr int light_smem_bytes() { return (8 * light_warp_words<WPL, LG>() + 32 * WPL) * 4; }  // + sparse-row mask

template <int WPL>
__device__ __forceinline__ void light_flush(const WS& ws, int p, const uint32_t* bm, const int32_t* meta,
                                            const uint32_t* q, int cnt) {
    const int lane = threadIdx.x & 31;
    const uint16_t* lists = ws.lists + p * ws.lists_stride;
    const int32_t* deg_full = ws.deg_full + p * ws.row_stride;
    if (lane < cnt) {
        constexpr int LM = list_max_of<WPL>();
        const uint32_t e = q[lane];
        const int j = (int)(e & 0xffffu), t = (int)((e >> 16) & 255), r = (int)(e >> 24);
        const int i = meta[4 * r], lo = meta[4 * r + 2];
        const uint32_t c = list_bitmap_count<LM>(lists + (int64_t)j * LM, deg_full[j], bm + r * 32 * WPL);
        ws.edges[p * ws.edges_stride + ws.rowptr[p * ws.rp_stride + i] + (t - lo)] = ((uint32_t)j << 16) | c;
    }
}

// LG (sparse rows per warp group): light_rows<WPL>() for batches; 2 when a small batch would leave SMs idle
#ifndef TRK_LIGHT_MINB
#define TRK_LIGHT_MINB 4  // shared memory allows 4 blocks per SM anyway: up to 64 registers
#endif
template <int WPL, int LG = light_rows<WPL>()>
__global__ void __launch_bounds__(256, TRK_LIGHT_MINB) k_sc2_light(WS ws) {
    extern __shared__ uint32_t s_dyn[];
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int W = d.W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nl = ws.st[p].n_light;
    int gr_lo, gr_hi;  // this rank's groups of LG sparse rows (all of them unless the pair is split)
    split_range(ws, (nl + LG - 1) / LG, &gr_lo, &gr_hi);
    if (gr_lo + (int)blockIdx.x * 8 >= gr_hi) return;  // the whole block is idle
    // the sparse-row mask in shared memory: the enumeration below tests one bit per list entry
    uint32_t* s_lm = s_dyn + 8 * light_warp_words<WPL, LG>();
    {
        const uint32_t* lmg = ws.light_mask + p * (ws.bits_stride / ws.row_stride);
        for (int w = threadIdx.x; w < W; w += blockDim.x) s_lm[w] = lmg[w];
        __syncthreads();
    }
    const int gi = gr_lo + blockIdx.x * 8 + warp;
    if (gi >= gr_hi) return;
    const int g0 = gi * LG;
    const int nr = min(LG, nl - g0);
    constexpr int LM = list_max_of<WPL>();
    uint32_t* bm = s_dyn + warp * light_warp_words<WPL, LG>();
    uint16_t* ls = reinterpret_cast<uint16_t*>(bm + LG * 32 * WPL);
    uint32_t* qL = bm + LG * 32 * WPL + LG * (LM / 2);
    uint32_t* qD = qL + 64;
    int32_t* meta = reinterpret_cast<int32_t*>(qD + 64);
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    const uint16_t* lists = ws.lists + p * ws.lists_stride;
    const int32_t* deg_full = ws.deg_full + p * ws.row_stride;
    const int32_t* light = ws.light_list + p * ws.row_stride;
    // stage the group's bitmaps and lists with asynchronous 16-byte copies (all rows in flight at once);
    // per-row meta (i, d, lo)
    int my_i = 0, my_d = 0, my_lo = 0;
    if (lane < nr) {
        my_i = light[g0 + lane];
        my_d = deg_full[my_i];
        my_lo = my_d - ws.deg[p * ws.row_stride + my_i];  // neighbours below i: degree minus |U_i|
        meta[4 * lane] = my_i;
        meta[4 * lane + 1] = my_d;
    }
    __syncwarp();
    const int W4 = W >> 2;  // 16-byte chunks of a bit row (W is a multiple of 4)
    for (int idx = lane; idx < nr * W4; idx += 32) {
        const int r = idx / W4, c = idx - r * W4;
        cp_async16(bm + r * 32 * WPL + 4 * c, bits + (int64_t)meta[4 * r] * W + 4 * c);
    }
    for (int idx = lane; idx < nr * (LM / 8); idx += 32) {
        const int r = idx / (LM / 8), c = idx - r * (LM / 8);
        uint16_t* dst = ls + r * LM + 8 * c;
        if (c * 8 < meta[4 * r + 1]) cp_async16(dst, lists + (int64_t)meta[4 * r] * LM + 8 * c);
        else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if (lane < nr) {
        meta[4 * lane] = my_i; meta[4 * lane + 1] = my_d; meta[4 * lane + 2] = my_lo;
    }
    // edge prefix over rows: pref(r) = Σ_{r' < r} (d − lo)
    const int my_up = (lane < nr) ? my_d - my_lo : 0;
    const int incl = warp_incl_scan(my_up);
    const int my_pref = incl - my_up;
    const int M = __shfl_sync(FULL, incl, 31);
    if (lane < nr) meta[4 * lane + 3] = my_pref;
    __syncwarp();
    int nL = 0;
    for (int e0 = 0; e0 < M; e0 += 32) {
        const int e = e0 + lane;
        bool isL = false;
        uint32_t packed = 0;
        if (e < M) {
            int r = 0;
            for (int rr = 1; rr < nr; ++rr)
                if (meta[4 * rr + 3] <= e) r = rr;
            const int lo = meta[4 * r + 2];
            const int pr = meta[4 * r + 3];
            const int t = lo + (e - pr);
            const int j = ls[r * LM + t];
            packed = (uint32_t)j | ((uint32_t)t << 16) | ((uint32_t)r << 24);
            isL = (s_lm[j >> 5] >> (j & 31)) & 1u;  // sparse j; dense j is k_sc2's edge
        }
        const unsigned bL = __ballot_sync(FULL, isL);
        if (isL) qL[nL + __popc(bL & ((1u << lane) - 1u))] = packed;
        nL += __popc(bL);
        __syncwarp();
        if (nL >= 32) {
            light_flush<WPL>(ws, p, bm, meta, qL, 32);
            __syncwarp();
            if (lane < nL - 32) qL[lane] = qL[32 + lane];
            nL -= 32;
            __syncwarp();
        }
    }
    light_flush<WPL>(ws, p, bm, meta, qL, nL);
}

// The pivot passes stream the pair's compact O2 edge array (E words) with a grid stride: coalesced,
// no per-row bookkeeping.
constexpr int SEL_BLOCKS_PER_PAIR = 8;  // (or more for small batches, to fill the GPU)

// Histogram of Ĝ >> 7 over positive O2 weights (the high digit of the pivot radix select, Eq. 4).
// The three edge passes below stream the pair's compact O2 edge array (edges_stride is a multiple of 4
// words) as uint4: EDGE_VEC edges per thread per round, all loads issued before any is consumed.
constexpr int EDGE_VEC = 8;
__device__ __forceinline__ void load_edges8(const uint32_t* edges, int e, int E, uint32_t (&v)[EDGE_VEC]) {
    if (e + EDGE_VEC <= E) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(edges + e));
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(edges + e) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < EDGE_VEC; ++k) v[k] = (e + k < E) ? __ldg(edges + e + k) : 0u;
    }
}

__global__ void __launch_bounds__(256) k_hist_hi(WS ws) {
    // one histogram column per lane (bin-major, lane-minor: s_hist[bin * 32 + lane]): the 32 lanes of a
    // warp never collide on an address or a bank, so the runs of equal bins need no warp aggregation
    __shared__ int s_hist[256 * 32];
    const int p = blockIdx.y;
    if (ws.desc[p].n == 0) return;
    PairState* st = ws.st + p;
    const int E = st->edges;
    const int lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < 256 * 32; b += blockDim.x) s_hist[b] = 0;
    __syncthreads();
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) * EDGE_VEC; e < E; e += gridDim.x * blockDim.x * EDGE_VEC) {
        uint32_t v[EDGE_VEC];
        load_edges8(edges, e, E, v);
        // consecutive weights come from one row and cluster in one bin: add runs, not single edges
        int run_bin = -1, run = 0;
#pragma unroll
        for (int k = 0; k < EDGE_VEC; ++k) {
            const uint32_t w = v[k] & 0xffffu;
            const int bin = w ? (int)(w >> 7) : -1;
            if (bin != run_bin) {
                if (run_bin >= 0) atomicAdd(&s_hist[run_bin * 32 + lane], run);  // other warps may share it
                run_bin = bin;
                run = 0;
            }
            ++run;
        }
        if (run_bin >= 0) atomicAdd(&s_hist[run_bin * 32 + lane], run);
    }
    __syncthreads();
    for (int b = threadIdx.x >> 5; b < 256; b += blockDim.x >> 5) {  // warp per bin: sum the 32 columns
        const int c = (int)__reduce_add_sync(FULL, (unsigned)s_hist[b * 32 + lane]);
        if (lane == 0 && c) atomicAdd(&st->hist_hi[b], c);
    }
}

// ------------------------------------------------------------------------------------------ a3 heavy split
// Full degrees (popcount of each bit row), their sum and maximum, and the sorted uint16 neighbour list of
// every row with degree <= list_max (zero-padded to a 16-byte chunk); one warp per row.
// Degrees and the sorted lists of sparse rows.  Lane l owns 8 consecutive words [g + 8l, g + 8l + 8) of a
// 256-word group (two 16-byte loads), so lane order is column order and one warp scan of the per-lane
// counts places every lane's entries; only rows with degree <= list_max extract their set bits.
__device__ __forceinline__ void deg_load8(const uint32_t* ri, int w0, int W, uint32_t (&v)[8]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint4 q = (w0 + 4 * h < W) ? __ldg(reinterpret_cast<const uint4*>(ri + w0 + 4 * h)) : make_uint4(0, 0, 0, 0);
        v[4 * h] = q.x; v[4 * h + 1] = q.y; v[4 * h + 2] = q.z; v[4 * h + 3] = q.w;
    }
}
__device__ __forceinline__ void deg_extract8(const uint32_t (&v)[8], int w0, int pos, uint16_t* L) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint32_t x = v[k];
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1u;
            L[pos++] = (uint16_t)((w0 + k) * 32 + b);
        }
    }
}
__global__ void __launch_bounds__(256, 6) k_degree(WS ws, int rows_per_block) {
    __shared__ unsigned long long s_sum;
    __shared__ int s_max;
    __shared__ uint4 s_list[SEL_WARPS][LIST_MAX / 8];  // a sparse row's list (rows of <= 256 words: list_max 64)
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    if (threadIdx.x == 0) { s_sum = 0ull; s_max = 0; }
    __syncthreads();
    const int W = d.W, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    unsigned mine = 0;
    int mx = 0;
    const int row0 = blockIdx.x * rows_per_block, row1 = min(row0 + rows_per_block, n);
    uint16_t* lists = ws.lists + p * ws.lists_stride;
    auto finish_row = [&](int i, int deg, int ucnt, bool pad = true) {  // ucnt: the row's total |U_i|
        uint16_t* L = lists + (int64_t)i * ws.list_max;
        if (pad && deg <= ws.list_max)
            for (int t = deg + lane; t < ((deg + 7) & ~7); t += 32) L[t] = 0;  // pad to a 16-byte chunk
        if (lane == 0) { ws.deg_full[p * ws.row_stride + i] = deg; ws.deg[p * ws.row_stride + i] = ucnt; }
        mine += deg;
        mx = max(mx, deg);
    };
    if (W <= 256) {  // the whole row in registers (WPL = ceil(W/32) words per lane, no idle lanes)
        auto rows = [&](auto wpl) {
            constexpr int WPL = decltype(wpl)::value;
            const int w0 = WPL * lane;
            uint32_t vn[WPL];
            auto load = [&](int i) {
                const uint32_t* ri = bits + (int64_t)i * W;
#pragma unroll
                for (int k = 0; k < WPL; ++k) vn[k] = (w0 + k < W) ? __ldg(ri + w0 + k) : 0u;
            };
            if (row0 + warp < row1) load(row0 + warp);
            for (int i = row0 + warp; i < row1; i += SEL_WARPS) {
                uint32_t v[WPL];
#pragma unroll
                for (int k = 0; k < WPL; ++k) v[k] = vn[k];
                if (i + SEL_WARPS < row1) load(i + SEL_WARPS);
                int cnt = 0;
#pragma unroll
                for (int k = 0; k < WPL; ++k) cnt += __popc(v[k]);
                const int deg = (int)__reduce_add_sync(FULL, (unsigned)cnt);
                // |U_i| = deg - #neighbours below i (no self loop)
                const int wi = i >> 5;
                const uint32_t mb = (1u << (i & 31)) - 1u;
                int bl = 0;
#pragma unroll
                for (int k = 0; k < WPL; ++k) {
                    const int w = w0 + k;
                    bl += __popc(v[k] & (w < wi ? 0xffffffffu : (w == wi ? mb : 0u)));
                }
                const int ucnt = deg - (int)__reduce_add_sync(FULL, (unsigned)bl);
                const bool smem_list = ws.list_max == LIST_MAX;  // (a batch with rows above 256 words: 256)
                if (deg <= ws.list_max && !smem_list) {
                    uint16_t* L = lists + (int64_t)i * ws.list_max;
                    int pos = warp_incl_scan(cnt) - cnt;
#pragma unroll
                    for (int k = 0; k < WPL; ++k) {
                        uint32_t x = v[k];
                        while (x) {
                            const int b = __ffs(x) - 1;
                            x &= x - 1u;
                            L[pos++] = (uint16_t)((w0 + k) * 32 + b);
                        }
                    }
                }
                if (deg <= ws.list_max && smem_list) {  // sorted list built in shared memory, written as 16-byte chunks
                    uint16_t* sl = reinterpret_cast<uint16_t*>(s_list[warp]);
                    if (lane < LIST_MAX / 8) s_list[warp][lane] = make_uint4(0u, 0u, 0u, 0u);
                    const int incl = warp_incl_scan(cnt);
                    int pos = incl - cnt;
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < WPL; ++k) {
                        uint32_t x = v[k];
                        while (x) {
                            const int b = __ffs(x) - 1;
                            x &= x - 1u;
                            sl[pos++] = (uint16_t)((w0 + k) * 32 + b);
                        }
                    }
                    __syncwarp();
                    if (lane < ((deg + 7) >> 3))
                        reinterpret_cast<uint4*>(lists + (int64_t)i * ws.list_max)[lane] = s_list[warp][lane];
                    __syncwarp();
                }
                if (ws.uprefix) {  // SC^2 mode: rank of any j in U_i = uprefix[i][j>>5] + popc(U_i word below j)
                    int uc[WPL], ul = 0;
#pragma unroll
                    for (int k = 0; k < WPL; ++k) { uc[k] = __popc(upper_mask(v[k], w0 + k, i)); ul += uc[k]; }
                    int run = warp_incl_scan(ul) - ul;
                    uint16_t* up = ws.uprefix + p * ws.bits_stride + (int64_t)i * W + w0;
#pragma unroll
                    for (int k = 0; k < WPL; ++k) {
                        if (w0 + k < W) up[k] = (uint16_t)run;
                        run += uc[k];
                    }
                }
                finish_row(i, deg, ucnt, !smem_list);
            }
        };
        switch ((W + 31) >> 5) {
            case 1: rows(std::integral_constant<int, 1>{}); break;
            case 2: rows(std::integral_constant<int, 2>{}); break;
            case 3: rows(std::integral_constant<int, 3>{}); break;
            case 4: rows(std::integral_constant<int, 4>{}); break;
            case 5: rows(std::integral_constant<int, 5>{}); break;
            case 6: rows(std::integral_constant<int, 6>{}); break;
            case 7: rows(std::integral_constant<int, 7>{}); break;
            default: rows(std::integral_constant<int, 8>{}); break;
        }
    } else {  // n > 8192: count first, extract in a second pass if sparse
        for (int i = row0 + warp; i < row1; i += SEL_WARPS) {
            const uint32_t* ri = bits + (int64_t)i * W;
            int deg = 0, ucnt = 0;
            for (int g = 0; g < W; g += 256) {
                uint32_t v[8];
                const int w0 = g + 8 * lane;
                deg_load8(ri, w0, W, v);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    deg += __popc(v[k]);
                    ucnt += __popc(upper_mask(v[k], w0 + k, i));
                }
            }
            deg = __reduce_add_sync(FULL, (unsigned)deg);
            if (ws.uprefix) {
                int carry = 0;
                for (int g = 0; g < W; g += 256) {
                    uint32_t v[8];
                    const int w0 = g + 8 * lane;
                    deg_load8(ri, w0, W, v);
                    int uc[8], tot = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) { uc[k] = __popc(upper_mask(v[k], w0 + k, i)); tot += uc[k]; }
                    const int incl = warp_incl_scan(tot);
                    int run = carry + incl - tot;
                    uint16_t* up = ws.uprefix + p * ws.bits_stride + (int64_t)i * W + w0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (w0 + k < W) up[k] = (uint16_t)run;
                        run += uc[k];
                    }
                    carry += __shfl_sync(FULL, incl, 31);
                }
            }
            if (deg <= ws.list_max) {
                int carry = 0;
                for (int g = 0; g < W; g += 256) {
                    uint32_t v[8];
                    const int w0 = g + 8 * lane;
                    deg_load8(ri, w0, W, v);
                    int cnt = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) cnt += __popc(v[k]);
                    const int incl = warp_incl_scan(cnt);
                    deg_extract8(v, w0, carry + incl - cnt, lists + (int64_t)i * ws.list_max);
                    carry += __shfl_sync(FULL, incl, 31);
                }
            }
            finish_row(i, deg, (int)__reduce_add_sync(FULL, (unsigned)ucnt));
        }
    }
    if (lane == 0 && mine) { atomicAdd(&s_sum, (unsigned long long)mine); atomicMax(&s_max, mx); }
    __syncthreads();
    if (threadIdx.x == 0 && s_sum) { atomicAdd(&ws.st[p].deg_sum, s_sum); atomicMax(&ws.st[p].deg_max, s_max); }
}

// One block per pair: H = rows with degree >= θ, θ = max(heavy_min_deg, ⌈max degree / 3⌉), raised until
// |H| <= heavy_cap; |H| < heavy_min_rows ⇒ no tensor-core block.  Ordered compaction (H in index order, so
// i < j ⇔ hpos(i) < hpos(j)).
__global__ void __launch_bounds__(1024) k_heavy(WS ws) {
    // rows 0 .. 8191 are held in registers (8 consecutive rows per thread, loaded once for every count and
    // the compaction); longer rows' tails are re-read
    constexpr int RC = 8, NC = 1024 * RC;
    __shared__ int s_w[32];
    __shared__ int s_carry, s_cnt;
    const int p = blockIdx.x;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    PairState* st = ws.st + p;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int32_t* deg = ws.deg_full + p * ws.row_stride;
    int32_t* hpos = ws.hpos + p * ws.row_stride;
    int dv[RC];
#pragma unroll
    for (int k = 0; k < RC; ++k) dv[k] = (t * RC + k < n) ? deg[t * RC + k] : -1;
    auto count_ge = [&](int th) {  // #rows with degree >= th (block-wide)
        if (t == 0) s_cnt = 0;
        __syncthreads();
        int c = 0;
#pragma unroll
        for (int k = 0; k < RC; ++k) c += dv[k] >= th;
        for (int i = NC + t; i < n; i += 1024) c += deg[i] >= th;
        c = __reduce_add_sync(FULL, (unsigned)c);
        if (lane == 0 && c) atomicAdd(&s_cnt, c);
        __syncthreads();
        const int r = s_cnt;
        __syncthreads();
        return r;
    };
    int thr = max(ws.heavy_min_deg, (st->deg_max + 2) / 3);
    int cnt = count_ge(thr);
    if (cnt > ws.heavy_cap) {  // smallest threshold whose row count fits the block: binary search
        int lo = thr, hi = st->deg_max + 1;  // count(lo) > cap >= count(hi) = 0
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (count_ge(mid) > ws.heavy_cap) lo = mid; else hi = mid;
        }
        thr = hi;
        cnt = count_ge(thr);
    }
    // widen H to every non-sparse row (degree > list_max) that fits the cap (heavy_widen = 0: only when that
    // costs no extra 256-row block of the tensor-core contraction): those rows' dense-dense edges then come
    // from the tensor cores instead of the latency-bound popcount path (1623 config-E pairs: k_sc2 3.17 ->
    // 2.68 us/pair for +0.04 on the block; N = 32 768: 3.96 -> 2.69 ms per pair)
    {
        const int thr2 = ws.heavy_widen > 1 ? ws.heavy_widen : max(ws.heavy_min_deg, ws.list_max + 1);
        if (thr2 < thr) {
            const int cnt2 = count_ge(thr2);
            if (cnt2 <= ws.heavy_cap && (ws.heavy_widen || (cnt2 + 255) / 256 <= (cnt + 255) / 256)) {
                thr = thr2;
                cnt = cnt2;
            }
        }
    }
    // E = Σ deg / 2 beyond the context's edge capacity: the pair is skipped (no tensor-core block, no
    // edges; k_rowclass empties its rows; k_finalize reports status 8 with the true E)
    const bool ovf = (long long)(st->deg_sum >> 1) > ws.edges_stride;
    const bool use = !ovf && ws.sc2_path != 1 && cnt >= ws.heavy_min_rows && cnt <= ws.heavy_cap;
    if (t == 0) { s_carry = 0; st->heavy_h = use ? cnt : 0; st->heavy_thr = thr; st->edge_overflow = ovf ? 1 : 0; }
    int32_t* hl = ws.heavy_list + p * ws.heavy_cap;
    uint32_t* hmask = ws.heavy_mask + p * (ws.bits_stride / ws.row_stride);
    // ordered compaction of the register-held rows: block scan of the per-thread counts
    {
        int fs = 0;
#pragma unroll
        for (int k = 0; k < RC; ++k) fs += (use && dv[k] >= thr) ? 1 : 0;
        const int x = warp_incl_scan(fs);
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const int y = s_w[lane];
            s_w[lane] = warp_incl_scan(y) - y;
        }
        __syncthreads();
        int pos = s_w[warp] + x - fs;
        uint32_t byte = 0;
#pragma unroll
        for (int k = 0; k < RC; ++k) {
            const int i = t * RC + k;
            const bool f = use && dv[k] >= thr;
            if (i < n) hpos[i] = f ? pos : -1;
            if (f) hl[pos++] = i;
            byte |= (uint32_t)f << k;
        }
        uint32_t wbits = byte << (RC * (lane & 3));  // 4 threads x 8 rows = one 32-bit word
        wbits |= __shfl_xor_sync(FULL, wbits, 1);
        wbits |= __shfl_xor_sync(FULL, wbits, 2);
        const int w = (t * RC) >> 5;
        if ((lane & 3) == 0 && w < d.W) hmask[w] = wbits;
        if (t == 1023) s_carry = pos;
        __syncthreads();
    }
    for (int r0 = NC; r0 < n; r0 += 1024) {
        const int i = r0 + t;
        const int f = (use && i < n && deg[i] >= thr) ? 1 : 0;
        int x = warp_incl_scan(f);
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int y = s_w[lane];
            int yi = warp_incl_scan(y);
            s_w[lane] = yi - y;
        }
        __syncthreads();
        const int pos = s_carry + s_w[warp] + x - f;
        if (i < n) hpos[i] = f ? pos : -1;
        if (f) hl[pos] = i;
        const unsigned fb = __ballot_sync(FULL, f);
        if (lane == 0) {
            const int wi = (r0 + warp * 32) >> 5;
            if (wi < d.W) hmask[wi] = fb;
        }
        __syncthreads();
        if (t == 1023) s_carry = pos + f;
        __syncthreads();
    }
}

// X[a][k] = C[H_a][k] as uint8 0/1 over all columns (rows a in [|H|, round_up(|H|, 256)) are zero), and
// for a < |H| the upper words of row H_a with their exclusive prefix popcounts (UP), from which the
// tensor-core epilogue reads the O2 test and the edge-list rank of every (H_a, H_b).  One warp per X row.
template <bool FP4>
__global__ void __launch_bounds__(256, 8) k_expand(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    if (d.n == 0) return;
    const int h = ws.st[p].heavy_h;
    if (h == 0) return;
    // rows the tiles read: int8 128×256 tiles reach round_up(h, 256); fp4 128×240 tiles (whose B tile is
    // loaded as 256 rows) reach round_up(h, 240) + 16
    const int xrows = (int)(ws.heavy_X_stride / ws.heavy_Kcap);  // allocated X rows (beyond: TMA zero fill)
    const int hp = min(xrows, FP4 ? max((h + 255) / 256 * 256, (h + 239) / 240 * 240 + 16) : (h + 255) / 256 * 256);
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a >= hp) return;
    const int W = d.W;
    const int ia = (a < h) ? ws.heavy_list[p * ws.heavy_cap + a] : -1;
    const uint32_t* row = (a < h) ? ws.bits + p * ws.bits_stride + (int64_t)ia * W : nullptr;
    uint8_t* X = ws.heavy_X + p * ws.heavy_X_stride + (int64_t)a * ws.heavy_Kcap;
    uint2* up = ws.heavy_UP + p * ws.heavy_UP_stride + (int64_t)a * W;
    int carry = 0;
    // rows up to 256 words: every word of the row is loaded before the first is expanded
    constexpr int PRE = 8;
    uint32_t pre[PRE];
    if (W <= 32 * PRE) {
#pragma unroll
        for (int k = 0; k < PRE; ++k) pre[k] = (row && 32 * k + lane < W) ? __ldg(row + 32 * k + lane) : 0u;
    }
#pragma unroll 1
    for (int w0 = 0; w0 < W; w0 += 32) {  // 32 bytes per bit word (two 16-byte stores)
        const int w = w0 + lane;
        uint32_t v;
        if (W <= 32 * PRE) {
            v = pre[0];
#pragma unroll
            for (int k = 1; k < PRE; ++k) v = (w0 == 32 * k) ? pre[k] : v;
        } else {
            v = (row && w < W) ? row[w] : 0u;
        }
        if (w < W) {
            if constexpr (FP4) {  // e2m1: bit k -> nibble k = 0x2 (1.0) or 0 (0.0), 16 bytes per word
                uint32_t b[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {  // byte q's 8 bits -> 8 nibbles: bit pairs select bytes of a table
                    uint32_t x = (v >> (8 * q)) & 0xffu;
                    x = (x | (x << 4)) & 0x0f0fu;  // selector nibble m = bits 2m, 2m+1
                    x = (x | (x << 2)) & 0x3333u;
                    b[q] = __byte_perm(0x22200200u, 0u, x);  // 00 -> 0x00, 01 -> 0x02, 10 -> 0x20, 11 -> 0x22
                }
                reinterpret_cast<uint4*>(X)[w] = make_uint4(b[0], b[1], b[2], b[3]);
            } else {
                uint32_t b[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t nib = (v >> (4 * q)) & 0xfu;
                    b[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
                }
                uint4* dst = reinterpret_cast<uint4*>(X + 32 * w);
                dst[0] = make_uint4(b[0], b[1], b[2], b[3]);
                dst[1] = make_uint4(b[4], b[5], b[6], b[7]);
            }
        }
        if (row) {
            const uint32_t u = (w < W) ? upper_mask(v, w, ia) : 0u;
            const int cnt = __popc(u);
            const int incl = warp_incl_scan(cnt);
            if (w < W) up[w] = make_uint2(u, (uint32_t)(carry + incl - cnt));
            carry += __shfl_sync(FULL, incl, 31);
        }
    }
    if constexpr (FP4) {  // the last 128-byte K block of an fp4 row may extend past 16 W bytes: zero it
        const int tail = (16 * W + 127) / 128 * 128;
        for (int b = 16 * W + 16 * lane; b < tail; b += 16 * 32) *reinterpret_cast<uint4*>(X + b) = make_uint4(0, 0, 0, 0);
    }
}

}  // namespace trk
