// a4 pivot selection (Eq. 4, Alg. 1 L4).  Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_sc2.cuh"

namespace trk {

// ------------------------------------------------------------------------------------------ a4 pivots
// Eq. 4: α_K1 = K1-th largest O2 weight; all edges > α plus the lexicographically first
// K1 - #(> α) edges of weight α (readings r4, r5).  Found by a two-digit radix select over the
// histograms, then an ordered (row-major = lexicographic) compaction.

// Block-wide: hist[0..nb) (nb <= blockDim.x, blockDim.x a multiple of 32, <= 1024).  Finds the bin b with
// suffix(b) >= K > suffix(b+1); if the total < K, b = lowest.  Returns (b, suffix(b+1)) to every thread.
__device__ void block_suffix_select(const int* hist, int nb, int K, int lowest, int* out_b, int* out_above,
                                    int* out_total) {
    __shared__ int s_w[32];
    __shared__ int s_res[3];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int bin = nb - 1 - t;  // reversed so an inclusive prefix is a suffix sum
    const int v = (t < nb) ? hist[bin] : 0;
    int incl = warp_incl_scan(v);
    if (lane == 31) s_w[warp] = incl;
    if (t == 0) { s_res[0] = lowest; s_res[1] = 0; }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int x = lane < nw ? s_w[lane] : 0;
        int xi = warp_incl_scan(x);
        if (lane < nw) s_w[lane] = xi - x;  // exclusive warp offsets
        if (lane == nw - 1) s_res[2] = xi;  // total
    }
    __syncthreads();
    incl += s_w[warp];
    const int excl = incl - v;  // = suffix(bin + 1)
    if (t < nb && bin >= lowest && incl >= K && excl < K) { s_res[0] = bin; s_res[1] = excl; }
    __syncthreads();
    const int total = s_res[2];
    if (total < K) {  // never crosses: take everything from `lowest` up
        // suffix(lowest + 1) is needed; recompute from the scan
        if (t < nb && bin == lowest) s_res[1] = excl;
        __syncthreads();
        if (t == 0) s_res[0] = lowest;
        __syncthreads();
    }
    *out_b = s_res[0];
    *out_above = s_res[1];
    *out_total = total;
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_hist_lo(WS ws) {
    __shared__ int s_lo[128];
    const int p = blockIdx.y;
    if (ws.desc[p].n == 0) return;
    PairState* st = ws.st + p;
    int b1, above, total;
    block_suffix_select(st->hist_hi, 256, ws.k1, 0, &b1, &above, &total);
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->b1 = b1; st->above = above; st->epos = total; }
    for (int b = threadIdx.x; b < 128; b += blockDim.x) s_lo[b] = 0;
    __syncthreads();
    const int E = st->edges;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) * EDGE_VEC; e < E; e += gridDim.x * blockDim.x * EDGE_VEC) {
        uint32_t v[EDGE_VEC];
        load_edges8(edges, e, E, v);
#pragma unroll
        for (int k = 0; k < EDGE_VEC; ++k) {
            const uint32_t w = v[k] & 0xffffu;
            if (w && (int)(w >> 7) == b1) atomicAdd(&s_lo[w & 127u], 1);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 128; b += blockDim.x)
        if (s_lo[b]) atomicAdd(&st->hist_lo[b], s_lo[b]);
}

// α, #(> α) and `need` from the two histograms (identical in every block).
__device__ void pivot_threshold(WS& ws, PairState* st, int* alpha, int* c_gt, int* need) {
    const int b1 = st->b1, above = st->above;
    int l, above_l, tot_l;
    const int lowest = (b1 == 0) ? 1 : 0;  // weight 0 is never a pivot
    block_suffix_select(st->hist_lo, 128, ws.k1 - above, lowest, &l, &above_l, &tot_l);
    *alpha = b1 * 128 + l;
    *c_gt = above + above_l;
    *need = ws.k1 - *c_gt;
}

// One block per pair: α, #(> α) and `need` into the pair state.
__global__ void __launch_bounds__(256) k_alpha(WS ws) {
    const int p = blockIdx.x;
    if (ws.desc[p].n == 0) return;
    PairState* st = ws.st + p;
    int alpha, c_gt, need;
    pivot_threshold(ws, st, &alpha, &c_gt, &need);
    if (threadIdx.x == 0) { st->alpha = alpha; st->c_gt = c_gt; st->need = need; }
}

// Every edge with weight > α, or == α, is a pivot candidate: its key ((0x7fff − w) << 30 | i << 15 | j)
// orders candidates by (w desc, i asc, j asc) (readings r4, r5).  Warp-aggregated append.
__global__ void __launch_bounds__(256) k_collect(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    PairState* st = ws.st + p;
    const int alpha = st->alpha;
    const int E = st->edges;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    unsigned long long* cand = ws.cand + (int64_t)p * PIV_CAP;
    const int lane = threadIdx.x & 31;
    for (int e0 = (blockIdx.x * blockDim.x + threadIdx.x) * EDGE_VEC; __any_sync(FULL, e0 < E);
         e0 += gridDim.x * blockDim.x * EDGE_VEC) {
        uint32_t v[EDGE_VEC];
        load_edges8(edges, e0, E, v);  // zero past E: weight 0 never qualifies
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < EDGE_VEC; ++k) {
            const int w = (int)(v[k] & 0xffffu);
            m |= (w >= alpha && w > 0) ? (1u << k) : 0u;
        }
        const int cnt = __popc(m);
        const int incl = warp_incl_scan(cnt);
        const int tot = __shfl_sync(FULL, incl, 31);
        if (tot == 0) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(&st->ncand, tot);
        base = __shfl_sync(FULL, base, 0) + incl - cnt;
#pragma unroll
        for (int k = 0; k < EDGE_VEC; ++k) {
            if (!((m >> k) & 1u)) continue;
            // (i, j) lexicographic = edge position order (rows are contiguous, j increasing within a row),
            // so the key carries the position; k_pivot_sort resolves (i, j) for the K1 winners only
            const int slot = base++;
            if (slot < PIV_CAP)
                cand[slot] = ((unsigned long long)(0x7fff - (int)(v[k] & 0xffffu)) << 30) | (unsigned)(e0 + k);
        }
    }
}

// One block per pair: bitonic sort of the candidates, the first min(K1, #candidates) become the pivots.
constexpr int SORT_RP_CAP = 16384;  // rowptr entries staged in shared memory after the keys
__global__ void __launch_bounds__(1024) k_pivot_sort(WS ws) {
    extern __shared__ unsigned long long s_key[];
    const int p = blockIdx.x;
    if (ws.desc[p].n == 0) return;
    PairState* st = ws.st + p;
    const int m = st->ncand;
    if (m > PIV_CAP) {
        if (threadIdx.x == 0) st->cand_overflow = 1;
        return;
    }
    int m2 = 64;
    while (m2 < m) m2 <<= 1;
    const unsigned long long* cand = ws.cand + (int64_t)p * PIV_CAP;
    for (int k = threadIdx.x; k < m2; k += blockDim.x) s_key[k] = (k < m) ? cand[k] : ~0ull;
    __syncthreads();
    // bitonic sort; for m2 <= 2048 each warp holds 64 consecutive keys in registers (lane: keys base + lane
    // and base + lane + 32), so strides <= 32 run on shuffles and only strides >= 64 go through shared memory
    auto smem_stage = [&](int size, int stride) {
        for (int k = threadIdx.x; k < m2 / 2; k += blockDim.x) {
            const int lo = 2 * k - (k & (stride - 1));
            const int hi = lo + stride;
            const bool up = (lo & size) == 0;
            const unsigned long long a = s_key[lo], b = s_key[hi];
            if ((a > b) == up) { s_key[lo] = b; s_key[hi] = a; }
        }
        __syncthreads();
    };
    if (m2 <= 2048) {
        const int lane = threadIdx.x & 31, base = 64 * (threadIdx.x >> 5);
        const bool act = base < m2;
        const int ea = base + lane, eb = ea + 32;
        unsigned long long a = ~0ull, b = ~0ull;
        auto reg_stages = [&](int size) {  // strides min(size/2, 32) .. 1 of one bitonic merge step
            for (int stride = min(size >> 1, 32); stride > 0; stride >>= 1) {
                if (stride == 32) {
                    if ((a > b) == ((ea & size) == 0)) { const unsigned long long x = a; a = b; b = x; }
                } else {
                    const unsigned long long pa = __shfl_xor_sync(FULL, a, stride), pb = __shfl_xor_sync(FULL, b, stride);
                    a = (((ea & stride) == 0) == ((ea & size) == 0)) ? min(a, pa) : max(a, pa);
                    b = (((eb & stride) == 0) == ((eb & size) == 0)) ? min(b, pb) : max(b, pb);
                }
            }
        };
        if (act) { a = s_key[ea]; b = s_key[eb]; }
        for (int size = 2; size <= 64; size <<= 1) reg_stages(size);
        if (act) { s_key[ea] = a; s_key[eb] = b; }
        __syncthreads();
        for (int size = 128; size <= m2; size <<= 1) {
            for (int stride = size >> 1; stride >= 64; stride >>= 1) smem_stage(size, stride);
            if (act) { a = s_key[ea]; b = s_key[eb]; }
            reg_stages(size);
            if (act) { s_key[ea] = a; s_key[eb] = b; }
            __syncthreads();
        }
    } else {
        for (int size = 2; size <= m2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) smem_stage(size, stride);
    }
    // keys are ((0x7fff - w) << 30 | edge position): the row of a winner comes from a binary search of its
    // position in rowptr (staged in shared memory when it fits), j from the edge word
    const int P = min(ws.k1, m);
    const int n = ws.desc[p].n;
    const int32_t* rpg = ws.rowptr + p * ws.rp_stride;
    int32_t* s_rp = reinterpret_cast<int32_t*>(s_key + PIV_CAP);
    const bool staged = n + 1 <= SORT_RP_CAP;
    if (staged)
        for (int k = threadIdx.x; k <= n; k += blockDim.x) s_rp[k] = rpg[k];
    __syncthreads();
    const int32_t* rp = staged ? s_rp : rpg;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    int4* piv = ws.piv + p * ws.piv_stride;
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        const unsigned long long key = s_key[k];
        const int e = (int)(key & 0x3fffffffu);
        int lo = 0, hi = n;  // row of edge e: rp[lo] <= e < rp[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (rp[mid] <= e) lo = mid; else hi = mid;
        }
        piv[k] = make_int4(lo, (int)(edges[e] >> 16), 0x7fff - (int)(key >> 30), 0);
    }
    if (threadIdx.x == 0) st->npiv = P;
}

__global__ void __launch_bounds__(256) k_select_count(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    PairState* st = ws.st + p;
    if (!st->cand_overflow) return;  // the candidate sort selected the pivots
    const int alpha = st->alpha;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    const int row0 = blockIdx.x * SEL_ROWS_PER_BLOCK, row1 = min(row0 + SEL_ROWS_PER_BLOCK, n);
    for (int i = row0 + warp; i < row1; i += SEL_WARPS) {
        const int dg = ws.deg[p * ws.row_stride + i];
        const uint32_t* e = edges + ws.rowptr[p * ws.rp_stride + i];
        int gt = 0, eq = 0;
        for (int k = lane; k < dg; k += 32) {
            const int w = (int)(e[k] & 0xffffu);
            gt += (w > alpha);
            eq += (w == alpha);
        }
        gt = __reduce_add_sync(FULL, (unsigned)gt);
        eq = __reduce_add_sync(FULL, (unsigned)eq);
        if (lane == 0) {
            ws.row_gt[p * ws.row_stride + i] = gt;
            ws.row_eq[p * ws.row_stride + i] = eq;
        }
    }
}

// One block per pair: exclusive scans over rows → how many weight-α edges each row contributes
// (lexicographic tie order) and each row's output offset.
__global__ void __launch_bounds__(1024) k_select_scan(WS ws) {
    __shared__ int s_w[32];
    __shared__ int s_carry[2];
    const int p = blockIdx.x;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    PairState* st = ws.st + p;
    if (!st->cand_overflow) return;
    const int need = st->need;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) { s_carry[0] = 0; s_carry[1] = 0; }
    __syncthreads();
    for (int r0 = 0; r0 < n; r0 += 1024) {
        const int i = r0 + t;
        const int eq = (i < n) ? ws.row_eq[p * ws.row_stride + i] : 0;
        const int gt = (i < n) ? ws.row_gt[p * ws.row_stride + i] : 0;
        // scan eq
        int x = warp_incl_scan(eq);
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int y = s_w[lane];
            int yi = warp_incl_scan(y);
            s_w[lane] = yi - y;
        }
        __syncthreads();
        const int ex_eq = s_carry[0] + x - eq + s_w[warp];
        int take = need - ex_eq;
        take = take < 0 ? 0 : (take > eq ? eq : take);
        const int cnt = gt + take;
        __syncthreads();
        // scan cnt
        int c = warp_incl_scan(cnt);
        __shared__ int s_w2[32];
        if (lane == 31) s_w2[warp] = c;
        __syncthreads();
        if (warp == 0) {
            int y = s_w2[lane];
            int yi = warp_incl_scan(y);
            s_w2[lane] = yi - y;
        }
        __syncthreads();
        const int off = s_carry[1] + c - cnt + s_w2[warp];
        if (i < n) {
            ws.row_take[p * ws.row_stride + i] = take;
            ws.row_off[p * ws.row_stride + i] = off;
        }
        __syncthreads();
        if (t == 1023) {
            s_carry[0] = ex_eq + eq;
            s_carry[1] = off + cnt;
        }
        __syncthreads();
    }
    if (t == 0) st->npiv = s_carry[1];
}

__global__ void __launch_bounds__(256) k_select_emit(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const PairState* st = ws.st + p;
    if (!st->cand_overflow) return;
    const int alpha = st->alpha;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    int4* piv = ws.piv + p * ws.piv_stride;
    const int row0 = blockIdx.x * SEL_ROWS_PER_BLOCK, row1 = min(row0 + SEL_ROWS_PER_BLOCK, n);
    for (int i = row0 + warp; i < row1; i += SEL_WARPS) {
        const int64_t ro = p * ws.row_stride + i;
        const int take = ws.row_take[ro];
        if (ws.row_gt[ro] + take == 0) continue;
        const int dg = ws.deg[ro];
        int pos = ws.row_off[ro];
        int eqseen = 0;
        const uint32_t* e = edges + ws.rowptr[p * ws.rp_stride + i];
        for (int k0 = 0; k0 < dg; k0 += 32) {
            const int k = k0 + lane;
            const uint32_t v = (k < dg) ? e[k] : 0u;
            const int w = (int)(v & 0xffffu);
            const bool iseq = (k < dg) && (w == alpha);
            const unsigned eqb = __ballot_sync(FULL, iseq);
            const bool sel = (k < dg) && (w > alpha || (iseq && eqseen + __popc(eqb & lt) < take));
            const unsigned sb = __ballot_sync(FULL, sel);
            if (sel) piv[pos + __popc(sb & lt)] = make_int4(i, (int)(v >> 16), w, 0);
            pos += __popc(sb);
            eqseen += __popc(eqb);
        }
    }
}

}  // namespace trk
