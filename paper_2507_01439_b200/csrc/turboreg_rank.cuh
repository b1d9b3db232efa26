// Optional outputs beside the hot path: per-row SC^2 sums r_i (App. B) and the ranked hypothesis list
// (App. F.1; SPEC RegistrationResult.ranked_hypotheses).  Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_model.cuh"

namespace trk {

// ------------------------------------------------------------------------------------------ r_i
// r_i = Σ_j Ĝ_ij over the full symmetric Ĝ (Eq. 2), which App. B identifies with 2·t_i, t_i the
// number of triangles through node i.  The O2 rows hold each edge once (i < j), so an edge adds its weight
// to both endpoints: one warp per row sums its upper edges (coalesced) into r_i and adds each weight to
// r_j.  Integer atomics: the result is exact and order-independent.
__global__ void __launch_bounds__(256) k_rowsum(WS ws, int32_t* rsum, int64_t rstride) {
    const int p = blockIdx.y;
    const int n = ws.desc[p].n;
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    const int32_t* rowptr = ws.rowptr + p * ws.rp_stride;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    int32_t* r = rsum + p * rstride;
    for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += gridDim.x * 8) {
        const int e0 = rowptr[i], e1 = rowptr[i + 1];
        int own = 0;
        for (int e = e0 + lane; e < e1; e += 32) {
            const uint32_t v = __ldg(edges + e);
            const int w = (int)(v & 0xffffu);
            own += w;
            if (w) atomicAdd(r + (v >> 16), w);
        }
        own = (int)__reduce_add_sync(FULL, (unsigned)own);
        if (lane == 0 && own) atomicAdd(r + i, own);
    }
}

// ------------------------------------------------------------------------------------------ ranking
// The valid hypotheses of one pair ranked by a metric (App. F.1: IN descending, MAE / MSE
// ascending; ties S desc, then (i,j,z) asc — the argmax order of readings r14 / r20, so rank 0 is T*).
// Off the hot path: a bitonic network over slot indices in global memory, one launch per stage, with a
// comparator that reads each slot's precomputed key.
struct RankKey {
    unsigned long long primary;  // IN: 2^32-1-count; MAE/MSE: the error's bits (non-negative double); invalid: ~0
    unsigned long long ijz;      // i << 30 | j << 15 | z
    int32_t nS;                  // -S
    int32_t slot;
};

__device__ __forceinline__ bool rank_less(const RankKey& a, const RankKey& b) {
    if (a.primary != b.primary) return a.primary < b.primary;
    if (a.nS != b.nS) return a.nS < b.nS;
    return a.ijz < b.ijz;
}

__global__ void k_rank_prep(WS ws, int pair, int metric, RankKey* keys, int32_t* idx, int m2) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m2) return;
    const int K = ws.k1 * ws.k2;
    RankKey k{~0ull, ~0ull, 0, s};
    if (s < K) {
        const int4 h = *reinterpret_cast<const int4*>(ws.hyp + (pair * ws.cl_stride + s) * 16 + 12);  // count, flag, S
        const int4 c = ws.cliq[pair * ws.cl_stride + s];
        if (h.y == 0 && c.x >= 0) {
            if (metric == 0) {
                k.primary = 0xffffffffull - (unsigned)h.x;
            } else {
                const double2 e = ws.herr[(pair * ws.cl_stride + s) * SCORE_SEGS_MAX];  // ordered sum (k_finalize)
                k.primary = (unsigned long long)__double_as_longlong(metric == 1 ? e.x : e.y);
            }
            k.nS = -h.z;
            k.ijz = ((unsigned long long)c.x << 30) | ((unsigned long long)c.y << 15) | (unsigned long long)c.z;
        }
    }
    keys[s] = k;
    idx[s] = s;
}

__global__ void k_rank_step(const RankKey* keys, int32_t* idx, int m2, int size, int stride) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m2 / 2) return;
    const int lo = 2 * k - (k & (stride - 1));
    const int hi = lo + stride;
    const bool up = (lo & size) == 0;
    const int a = idx[lo], b = idx[hi];
    if (rank_less(keys[b], keys[a]) == up) { idx[lo] = b; idx[hi] = a; }
}

struct DevHypothesis {  // mirrors turboreg_hypothesis
    int32_t clique[3];
    int32_t clique_weight;
    float R[9];
    float t[3];
    int32_t inlier_count;
    int32_t slot;
    double mae, mse;
};

__global__ void k_rank_emit(WS ws, int pair, const RankKey* keys, const int32_t* idx, int top, int n,
                            DevHypothesis* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= top) return;
    const int s = idx[r];
    DevHypothesis o;
    const float* h = ws.hyp + (pair * ws.cl_stride + s) * 16;
    const int4 c = ws.cliq[pair * ws.cl_stride + s];
    o.clique[0] = c.x; o.clique[1] = c.y; o.clique[2] = c.z;
    o.clique_weight = c.w;
    for (int k = 0; k < 9; ++k) o.R[k] = h[k];
    for (int k = 0; k < 3; ++k) o.t[k] = h[9 + k];
    o.inlier_count = __float_as_int(h[12]);
    o.slot = s;
    if (ws.herr) {
        const double2 e = ws.herr[(pair * ws.cl_stride + s) * SCORE_SEGS_MAX];
        o.mae = e.x / n;
        o.mse = e.y / n;
    } else {
        o.mae = o.mse = __longlong_as_double(0x7ff8000000000000ll);  // NaN: errors not accumulated
    }
    out[r] = o;
}

// number of valid entries (primary != ~0) among the first m2 sorted indices
__global__ void k_rank_count(const RankKey* keys, const int32_t* idx, int m2, int* count) {
    int c = 0;
    for (int k = threadIdx.x; k < m2; k += blockDim.x) c += keys[idx[k]].primary != ~0ull;
    c = (int)__reduce_add_sync(FULL, (unsigned)c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// ------------------------------------------------------------------------------------------ NEXT(1) merge
// A pair split over `world` ranks: each rank's record holds the argmax over its own pivots' TurboCliques
// (k_finalize).  T* is the maximum of those by the same key (count desc, S desc, (i,j,z) asc, reading r14);
// clique and hypothesis counts add up; |P|, E and the per-pair status are the same on every rank.
__global__ void k_split_merge(const DevResult* parts, int world, DevResult* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int best = -1, ncl = 0, nev = 0;
    for (int r = 0; r < world; ++r) {
        const DevResult& a = parts[r];
        ncl += a.num_cliques;
        nev += a.hypotheses_evaluated;
        if (a.status != 0) continue;
        if (best < 0) { best = r; continue; }
        const DevResult& b = parts[best];
        const unsigned long long ka = ((unsigned long long)(unsigned)a.inlier_count << 17) | (unsigned)a.clique_weight;
        const unsigned long long kb = ((unsigned long long)(unsigned)b.inlier_count << 17) | (unsigned)b.clique_weight;
        const unsigned long long ta = ((unsigned long long)a.clique[0] << 30) | ((unsigned long long)a.clique[1] << 15) | a.clique[2];
        const unsigned long long tb = ((unsigned long long)b.clique[0] << 30) | ((unsigned long long)b.clique[1] << 15) | b.clique[2];
        if (ka > kb || (ka == kb && ta < tb)) best = r;
    }
    DevResult o = parts[best >= 0 ? best : 0];
    if (best < 0) {  // no rank has a hypothesis: the shared status (2/3/4/8), else NO_HYPOTHESIS
        int st = 5;
        for (int r = 0; r < world; ++r)
            if (parts[r].status != 5 && parts[r].status != 0) st = parts[r].status;
        o.status = st;
    }
    o.num_cliques = ncl;
    o.hypotheses_evaluated = nev;
    *out = o;
}

// ------------------------------------------------------------------------------------------ checked build
// TRK_CHECKS (libturboreg_checked.so, tests only; compute-sanitizer is closed on the GPU pool): structural
// invariants of the assembled graph and of the TurboCliques, verified on the device after each stage;
// any violation traps, so the call fails with a CUDA error.
#ifdef TRK_CHECKS
__device__ __forceinline__ void trk_fail(const char* what, int p, int a, int b, int c) {
    printf("TRK_CHECKS: %s (pair %d: %d %d %d)\n", what, p, a, b, c);
    __trap();
}
__device__ __forceinline__ bool bit_of(const uint32_t* row, int j) { return (row[j >> 5] >> (j & 31)) & 1u; }
// Every O2 edge slot written exactly once with the right neighbour and weight: row i's words are the
// increasing j > i with C_ij = 1, and Ĝ_ij = popcount(row_i AND row_j) (Eq. 2).  One warp per row.
__global__ void k_check_edges(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n, W = d.W;
    if (n == 0 || ws.st[p].edge_overflow) return;
    const int lane = threadIdx.x & 31;
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    const int32_t* rp = ws.rowptr + p * ws.rp_stride;
    for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += gridDim.x * 8) {
        const uint32_t* ri = bits + (int64_t)i * W;
        int prev = i;
        for (int e = rp[i]; e < rp[i + 1]; ++e) {
            const uint32_t v = edges[e];
            const int j = (int)(v >> 16), w = (int)(v & 0xffffu);
            if (lane == 0 && (j <= prev || j >= n || !bit_of(ri, j))) trk_fail("edge neighbour", p, i, e, j);
            uint32_t c = 0;
            const uint32_t* rj = bits + (int64_t)j * W;
            for (int k = lane; k < W; k += 32) c += __popc(ri[k] & rj[k]);
            c = __reduce_add_sync(0xffffffffu, c);
            if (lane == 0 && (int)c != w) trk_fail("edge weight", p, i, j, w);
            prev = j;
        }
        // the count of upper neighbours equals the row's slot count
        int u = 0;
        for (int k = lane; k < W; k += 32) u += __popc(upper_mask(ri[k], k, i));
        u = (int)__reduce_add_sync(0xffffffffu, (unsigned)u);
        if (lane == 0 && u != rp[i + 1] - rp[i]) trk_fail("row slot count", p, i, u, rp[i + 1] - rp[i]);
    }
}
// Every emitted TurboClique is a 3-clique of C with i < j < z, its pivot's pair, and S = the sum of its three
// O2 weights (Eq. 6); pivots are positive O2 edges.
__global__ void k_check_cliques(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n, W = d.W;
    if (n == 0) return;
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    const uint32_t* edges = ws.edges + p * ws.edges_stride;
    const int32_t* rp = ws.rowptr + p * ws.rp_stride;
    auto weight = [&](int a, int b) -> int {  // a < b: binary search of row a's slots
        int lo = rp[a], hi = rp[a + 1] - 1;
        while (lo <= hi) {
            const int m = (lo + hi) >> 1;
            const int j = (int)(edges[m] >> 16);
            if (j == b) return (int)(edges[m] & 0xffffu);
            if (j < b) lo = m + 1; else hi = m - 1;
        }
        return -1;
    };
    const int K = ws.k1 * ws.k2;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < K; s += gridDim.x * blockDim.x) {
        const int4 c = ws.cliq[p * ws.cl_stride + s];
        if (c.x < 0) continue;
        if (!(c.x < c.y && c.y < c.z && c.z < n)) trk_fail("clique order", p, c.x, c.y, c.z);
        const uint32_t* ri = bits + (int64_t)c.x * W;
        const uint32_t* rj = bits + (int64_t)c.y * W;
        if (!bit_of(ri, c.y) || !bit_of(ri, c.z) || !bit_of(rj, c.z)) trk_fail("clique not a 3-clique", p, c.x, c.y, c.z);
        if (weight(c.x, c.y) + weight(c.x, c.z) + weight(c.y, c.z) != c.w) trk_fail("clique weight", p, c.x, c.y, c.w);
    }
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < ws.st[p].npiv; k += blockDim.x) {
            const int4 v = ws.piv[p * ws.piv_stride + k];
            if (!(v.x < v.y) || v.z <= 0 || weight(v.x, v.y) != v.z) trk_fail("pivot", p, v.x, v.y, v.z);
        }
}
#endif

}  // namespace trk
