// a5 Pivot-Guided Search (Alg. 1 L5-13, Eqs. 5-7) and the SC^2-mode canonical list.
// Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_select.cuh"

namespace trk {

// ------------------------------------------------------------------------------------------ a5 PGS
// Alg. 1 L5-13, Eqs. 5-7.  One warp per pivot (i, j): the O2 common neighbours are
// M = U_i ∧ U_j (z > j > i; for a pivot C_ij = 1, so Ĝ_iz > 0 ⇔ C_iz, reading r10), scanned word-parallel;
// Ĝ_iz and Ĝ_jz are gathered from the rank-indexed edge lists (rank = prefix popcount of U_i / U_j below
// z, from a warp scan).  S = Ĝ_ij + Ĝ_iz + Ĝ_jz; the top-K2 by (S desc, z asc) are kept (readings r7, r8):
// per-lane register lists (K2 <= KL) merged by K2 warp argmax rounds, or K2 threshold rounds otherwise.
constexpr int PGS_WARPS = 8;
constexpr int PGS_KL = 8;
#ifndef TRK_PGS_QCAP
#define TRK_PGS_QCAP 128
#endif
constexpr int PGS_QCAP = TRK_PGS_QCAP;  // per-warp candidate queue (entries) of the O2 scan

// Candidate keys (reading r8: S desc, z asc) in 32 bits: S = Ĝ_ij + Ĝ_iz + Ĝ_jz < 3·2^15 takes 17 bits and
// z < 2^15 (n <= 32768) the low 15, stored as 32767 − z; every candidate key is > 0 (S >= Ĝ_ij >= 1).
constexpr uint32_t PGS_ZMAX = 32767u;
// (Ĝ_a + Ĝ_b) << 15 from two edge words (z << 16 | Ĝ): the Ĝ fields shifted to the top add without a carry
// out (Ĝ_a + Ĝ_b < 2^16) and the z fields fall off.
__device__ __forceinline__ uint32_t pgs_pair_sum15(uint32_t a, uint32_t b) { return ((a << 16) + (b << 16)) >> 1; }

// Candidates of a 32-word chunk are flattened across the warp before their weights are gathered: every lane
// writes its own candidates (z, rank in U_i, rank in U_j) to the warp's shared-memory queue at its prefix
// offset, then the lanes take the queue entries round-robin, so the gathers and the top-K2 insertions run
// on all 32 lanes whatever the distribution of candidates over the words (a chunk with more than PGS_QCAP
// candidates, i.e. one where most words hold several, has each lane walk its own word: highest bit first,
// one mask ~(−1 << b) giving both the remaining bits and the rank prefixes).
template <typename F>
__device__ __forceinline__ void pgs_scan_candidates(const uint32_t* ri, const uint32_t* rj, int W, int i, int j,
                                                    const uint32_t* ei, const uint32_t* ej, int wij, uint2* sq, F&& f) {
    const int lane = threadIdx.x & 31;
    int carry_i = 0, carry_j = 0;
    const int nchunks = (W + 31) >> 5;
    const uint32_t wbase = ((uint32_t)wij << 15) + PGS_ZMAX;
    for (int c = (i + 1) >> 10; c < nchunks; ++c) {  // chunks holding no bit > i contribute nothing
        const int w = c * 32 + lane;
        const uint32_t ui = (w < W) ? upper_mask(ri[w], w, i) : 0u;
        const uint32_t uj = (w < W) ? upper_mask(rj[w], w, j) : 0u;
        const int pi = __popc(ui), pj = __popc(uj);
        const int sij = warp_incl_scan(pi | (pj << 16));  // both prefix scans in one (each sum <= 1024)
        const int exi = carry_i + (sij & 0xffff) - pi, exj = carry_j + (sij >> 16) - pj;
        const int tij = __shfl_sync(FULL, sij, 31);
        carry_i += tij & 0xffff;
        carry_j += tij >> 16;
        uint32_t m = ui & uj;
        const int cm = __popc(m);
        const int incl = warp_incl_scan(cm);
        const int total = __shfl_sync(FULL, incl, 31);
        if (total == 0) continue;
        if (total <= PGS_QCAP) {
            int o = incl - cm;
            while (m) {  // this lane's candidates into the queue
                const int b = 31 - __clz(m);
                const uint32_t below = ~(0xffffffffu << b);
                m &= below;
                const uint32_t rk_i = (uint32_t)(exi + __popc(ui & below)), rk_j = (uint32_t)(exj + __popc(uj & below));
                sq[o++] = make_uint2((uint32_t)(w * 32 + b) | (rk_i << 16), rk_j);
            }
            __syncwarp();
            for (int k = lane; k < total; k += 64) {  // two queue entries per lane in flight
                const uint2 e0 = sq[k];
                const bool two = k + 32 < total;
                const uint2 e1 = two ? sq[k + 32] : e0;
                const uint32_t a0 = __ldg(ei + (e0.x >> 16)), b0 = __ldg(ej + e0.y);
                const uint32_t a1 = __ldg(ei + (e1.x >> 16)), b1 = __ldg(ej + e1.y);
                f(pgs_pair_sum15(a0, b0) + wbase - (e0.x & 0xffffu));
                if (two) f(pgs_pair_sum15(a1, b1) + wbase - (e1.x & 0xffffu));
            }
            __syncwarp();
        } else {
            const uint32_t* pei = ei + exi;
            const uint32_t* pej = ej + exj;
            const uint32_t zb = wbase - (uint32_t)(w * 32);
            while (m) {
                const int b = 31 - __clz(m);
                const uint32_t below = ~(0xffffffffu << b);
                m &= below;
                const uint32_t a = __ldg(pei + __popc(ui & below)), e = __ldg(pej + __popc(uj & below));
                f(pgs_pair_sum15(a, e) + zb - (uint32_t)b);
            }
        }
    }
}

// SC^2 (undirected) mode, reading r9: N(i,j) = {z ∉ {i,j} : C_iz ∧ C_jz} on both sides of the pivot
// (Table 5 row 10).  Ĝ_iz for z > i is row i's rank-indexed entry; for z < i the edge lives in row
// z at rank uprefix[z][i>>5] + popc(U_z word below i).
__device__ __forceinline__ uint32_t sc2_lower_weight(const WS& ws, int q, int W, int z, int x) {
    const int wx = x >> 5;
    const uint32_t u = upper_mask(__ldg(ws.bits + q * ws.bits_stride + (int64_t)z * W + wx), wx, z);
    const int rk = (int)__ldg(ws.uprefix + q * ws.bits_stride + (int64_t)z * W + wx) + __popc(u & ((1u << (x & 31)) - 1u));
    return __ldg(ws.edges + q * ws.edges_stride + ws.rowptr[q * ws.rp_stride + z] + rk) & 0xffffu;
}
template <typename F>
__device__ __forceinline__ void pgs_scan_candidates_sc2(const WS& ws, int q, const uint32_t* ri, const uint32_t* rj,
                                                        int W, int i, int j, const uint32_t* ei, const uint32_t* ej,
                                                        int wij, F&& f) {
    const int lane = threadIdx.x & 31;
    int carry_i = 0, carry_j = 0;
    const int nchunks = (W + 31) >> 5;
    for (int c = 0; c < nchunks; ++c) {
        const int w = c * 32 + lane;
        const uint32_t vi = (w < W) ? ri[w] : 0u, vj = (w < W) ? rj[w] : 0u;
        const uint32_t ui = (w < W) ? upper_mask(vi, w, i) : 0u;
        const uint32_t uj = (w < W) ? upper_mask(vj, w, j) : 0u;
        const int pi = __popc(ui), pj = __popc(uj);
        const int si = warp_incl_scan(pi), sj = warp_incl_scan(pj);
        const int exi = carry_i + si - pi, exj = carry_j + sj - pj;
        carry_i += __shfl_sync(FULL, si, 31);
        carry_j += __shfl_sync(FULL, sj, 31);
        uint32_t m = vi & vj;  // C_ii = C_jj = 0 and C_ij = 1: i and j are never in both rows
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1u;
            const uint32_t below = (1u << b) - 1u;
            const int z = w * 32 + b;
            const uint32_t wiz = (z > i) ? (__ldg(ei + exi + __popc(ui & below)) & 0xffffu) : sc2_lower_weight(ws, q, W, z, i);
            const uint32_t wjz = (z > j) ? (__ldg(ej + exj + __popc(uj & below)) & 0xffffu) : sc2_lower_weight(ws, q, W, z, j);
            f(((uint32_t)(wij + (int)wiz + (int)wjz) << 15) + PGS_ZMAX - (uint32_t)z);
        }
    }
}

// A clique as (i, j, z) ascending (O2 mode: z > j > i already; SC^2 mode: z anywhere) and S.
__device__ __forceinline__ int4 sorted_clique(int i, int j, int z, int S) {
    const int a = min(i, min(j, z)), c = max(i, max(j, z));
    return make_int4(a, i + j + z - a - c, c, S);
}

// Per-lane sorted top-KL lists (KL >= K2) merged by K2 warp argmax rounds.
template <int KL, int MODE>
__device__ __forceinline__ int pgs_topk_list(const WS& ws, int q, const uint32_t* ri, const uint32_t* rj, int W, int i,
                                             int j, const uint32_t* ei, const uint32_t* ej, int wij, int K2, int4* out,
                                             uint2* sq) {
    const int lane = threadIdx.x & 31;
    uint32_t top[KL];
#pragma unroll
    for (int r = 0; r < KL; ++r) top[r] = 0u;
    auto insert = [&](uint32_t key) {
        if (key > top[KL - 1]) {  // sorted insertion, descending
            uint32_t k = key;
#pragma unroll
            for (int r = 0; r < KL; ++r) {
                const uint32_t hi = max(k, top[r]);
                k = min(k, top[r]);
                top[r] = hi;
            }
        }
    };
    if constexpr (MODE == 1) pgs_scan_candidates_sc2(ws, q, ri, rj, W, i, j, ei, ej, wij, insert);
    else pgs_scan_candidates(ri, rj, W, i, j, ei, ej, wij, sq, insert);
    int emitted = 0;
    for (int r = 0; r < K2; ++r) {
        const uint32_t head = top[0];
        const uint32_t best = __reduce_max_sync(FULL, head);
        if (best == 0u) break;
        if (head == best) {  // keys are unique (distinct z), exactly one lane pops
#pragma unroll
            for (int s2 = 0; s2 < KL - 1; ++s2) top[s2] = top[s2 + 1];
            top[KL - 1] = 0u;
        }
        if (lane == 0) out[r] = sorted_clique(i, j, (int)(PGS_ZMAX - (best & PGS_ZMAX)), (int)(best >> 15));
        ++emitted;
    }
    return emitted;
}

// KL: per-lane top list length (2, 4, PGS_KL; 0 = K2 threshold rounds), fixed per launch so each
// instantiation only holds the registers its own branch needs (occupancy: the kernel is latency-bound).
#ifndef TRK_PGS_MINB
#define TRK_PGS_MINB 6
#endif
template <int MODE, int KL>
__global__ void __launch_bounds__(PGS_WARPS * 32, (KL == 2 ? TRK_PGS_MINB : 4)) k_pgs(WS ws) {
    __shared__ uint2 s_q[PGS_WARPS][PGS_QCAP];
    const int q = blockIdx.y;
    const PairDesc d = ws.desc[q];
    const int n = d.n;
    if (n == 0) return;
    const int W = d.W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pv = blockIdx.x * PGS_WARPS + warp;
    const int K1 = ws.k1, K2 = ws.k2;
    if (pv >= K1) return;
    int4* out = ws.cliq + q * ws.cl_stride + (int64_t)pv * K2;
    // the pivot slot is read before |P| is known (both loads in flight; slots >= |P| are never used)
    const int4 pvt = ws.piv[q * ws.piv_stride + pv];
    const int P = ws.st[q].npiv;
    int pv_lo, pv_hi;  // this rank's pivots (all of them unless the pair is split): others leave empty slots
    split_range(ws, P, &pv_lo, &pv_hi);
    if (pv >= P || pv < pv_lo || pv >= pv_hi) {
        for (int r = lane; r < K2; r += 32) out[r] = make_int4(-1, -1, -1, 0);
        return;
    }
    const int i = pvt.x, j = pvt.y, wij = pvt.z;
    const uint32_t* bits = ws.bits + q * ws.bits_stride;
    const uint32_t* ri = bits + (int64_t)i * W;
    const uint32_t* rj = bits + (int64_t)j * W;
    const uint32_t* edges = ws.edges + q * ws.edges_stride;
    const uint32_t* ei = edges + ws.rowptr[q * ws.rp_stride + i];
    const uint32_t* ej = edges + ws.rowptr[q * ws.rp_stride + j];
    uint2* sq = s_q[warp];
    int emitted = 0;
    if constexpr (KL > 0) {
        emitted = pgs_topk_list<KL, MODE>(ws, q, ri, rj, W, i, j, ei, ej, wij, K2, out, sq);
    } else {
        uint32_t thr = 0xffffffffu;
        for (int r = 0; r < K2; ++r) {
            uint32_t mine = 0u;
            auto take = [&](uint32_t key) {
                if (key < thr) mine = max(mine, key);
            };
            if constexpr (MODE == 1) pgs_scan_candidates_sc2(ws, q, ri, rj, W, i, j, ei, ej, wij, take);
            else pgs_scan_candidates(ri, rj, W, i, j, ei, ej, wij, sq, take);
            const uint32_t best = __reduce_max_sync(FULL, mine);
            if (best == 0u) break;
            if (lane == 0) out[r] = sorted_clique(i, j, (int)(PGS_ZMAX - (best & PGS_ZMAX)), (int)(best >> 15));
            thr = best;
            ++emitted;
        }
    }
    for (int r = emitted + lane; r < K2; r += 32) out[r] = make_int4(-1, -1, -1, 0);
}

}  // namespace trk
