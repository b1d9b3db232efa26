// Shared device-side types of the hot path: per-pair descriptor and state, the workspace (WS) with
// its per-pair views, and warp-level helpers.  Part of turboreg_kernels.cuh.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace trk {


constexpr unsigned FULL = 0xffffffffu;

struct PairDesc {
    const float* src;     // N×3 float32 (device), already offset to this pair
    const float* dst;
    int32_t n;            // 0 ⇒ pair skipped (host_status says why)
    int32_t W;            // words per bit row
    int32_t host_status;  // turboreg_status decided on the host (0, 2 or 3)
    int32_t pad;
};

struct PairState {
    int32_t nonfinite;  // set by k_ingest
    int32_t edges;      // E, undirected edges of C(τ)
    int32_t epos;       // E+, edges with Ĝ > 0
    int32_t b1;         // radix-select high digit of α
    int32_t above;      // #weights with high digit > b1
    int32_t alpha;      // α_K1 (Eq. 4)
    int32_t c_gt;       // #weights > α
    int32_t need;       // K1 - c_gt: how many weight-α edges are taken (lexicographically first)
    int32_t npiv;       // |P|
    int32_t edges_base; // edges of C(τ_base)
    int32_t heavy_h;    // |H|, rows whose SC^2 block runs on the tensor cores (0 = none)
    int32_t heavy_thr;  // degree threshold that defined H
    unsigned long long deg_sum;  // Σ_i deg(i) = 2E
    int32_t deg_max;             // max_i deg(i)
    int32_t n_light;             // rows with a list and not heavy (k_sc2_light)
    int32_t n_dense;             // the other rows (k_sc2)
    int32_t ncand;               // pivot candidates (weight >= α) collected
    int32_t cand_overflow;       // ncand > PIV_CAP: the ordered count/scan/emit path selects instead
    int32_t edge_overflow;       // E > the context's per-pair edge capacity: pair skipped (status 8)
    int32_t pad2[4];
    uint32_t bbox[12];     // order keys of max src xyz, -min src xyz, max dst xyz, -min dst xyz (k_ingest)
    int32_t hist_hi[256];  // histogram of Ĝ_ij >> 7 over positive O2 edges
    int32_t hist_lo[128];  // histogram of Ĝ_ij & 127 within bin b1
};

constexpr int PIV_CAP = 8192;  // pivot candidates sorted in shared memory per pair
constexpr int SCORE_SEGS_MAX = 16;  // correspondence segments of a scoring launch (partial sums per segment)

struct WS {
    const PairDesc* desc;
    PairState* st;
    float4* src4;
    float4* dst4;
    int64_t pts_stride;
    uint32_t* bits;
    uint32_t* bits_base;
    int64_t bits_stride;
    int32_t* deg;
    int32_t* row_gt;
    int32_t* row_eq;
    int32_t* row_take;
    int32_t* row_off;
    int64_t row_stride;
    uint32_t* edges;
    int64_t edges_stride;  // per-pair edge capacity (words, multiple of 4): a pair with more O2 edges overflows
    int32_t* rowptr;      // [n+1] per pair, stride rp_stride
    int64_t rp_stride;
    int4* piv;
    int64_t piv_stride;  // K1
    unsigned long long* cand;  // [PIV_CAP] pivot candidate keys per pair
    int4* cliq;
    float* hyp;
    int64_t cl_stride;  // K1*K2
    void* res;          // turboreg_result[batch]
    // heavy/light SC^2 split (turboreg_sc2_mma.cuh)
    int32_t* deg_full;    // [n] full degree
    int32_t* hpos;        // [n] position in H or -1
    int32_t* heavy_list;  // [cap] H in index order
    int32_t* tile_tab;    // [2·batch + 1]: tensor-core tile-count prefix over the batch's pairs, then |H| per pair
    int32_t* tile_ctr;    // tensor-core tile counter (dynamic tile scheduling), zeroed before every launch
    uint16_t* lists;      // [n][LIST_MAX] sorted neighbour lists of rows with degree <= LIST_MAX
    int32_t* light_list;  // [n] sparse non-heavy rows, index order
    int32_t* dense_list;  // [n] all other rows, index order
    int64_t lists_stride;
    int32_t list_max;     // sparse-row degree bound and list row stride of this launch (64, or 256 if W > 256)
    uint32_t* heavy_mask; // [W] bitset of H
    uint32_t* light_mask; // [W] bitset of the sparse rows (k_sc2_light's rows)
    uint2* heavy_UP;      // [cap][W] per heavy row a: (U_{H_a} word, exclusive prefix popcount of U_{H_a})
    int64_t heavy_UP_stride;
    uint8_t* heavy_X;     // [cap][heavy_Kcap] rows of C restricted to H (uint8 0/1, or packed e2m1 when x_fp4)
    int64_t heavy_X_stride;
    int32_t heavy_Kcap;   // bytes per X row: 32 W (uint8) or round_up(16 W, 128) (packed e2m1)
    int32_t heavy_cap;    // max |H| (multiple of 256)
    uint16_t* heavy_D;    // [cap][cap] X X^T (+ sparse-column correction)
    int64_t heavy_D_stride;
    int32_t heavy_min_rows, heavy_min_deg, sc2_path;
    float tau, tau_base, thr;
    int32_t k1, k2, mode;
    int32_t pair_base;    // index of pair 0 of this view in the batch (TMA coordinates address the whole batch)
    uint16_t* uprefix;    // SC^2 mode only: [n][W] exclusive prefix popcount of U_i per word (stride bits_stride)
    double2* herr;        // [K1*K2][SCORE_SEGS_MAX] per hypothesis and correspondence segment (Σ sqrtf(s), Σ s)
                          // (r20); k_finalize adds the segments in order into slot [h][0] (deterministic)
    int32_t x_fp4;        // heavy_X holds packed e2m1 (block-scaled fp4 tensor-core path) instead of uint8
    int32_t mma_l2;       // L2 policy of the X tile loads: 0 evict_normal, 1 evict_last, 2 evict_first
    int32_t heavy_widen;  // 1: H takes every non-sparse row that fits the cap (else only at no extra block)
    int32_t err_mode;     // bit 0: accumulate herr; rank = err_mode >> 1: 0 inlier number, 1 MAE, 2 MSE
    // NEXT(1), one pair split over split_world ranks (1 = not split): this rank's share of every split work
    // list (compat block-row pairs from compat_b0, tensor-core tiles, dense-row items, sparse-row groups,
    // pivots) is the contiguous range split_range(count) below
    int32_t split_rank, split_world, compat_b0;
};

// [lo, hi) of `count` work units owned by this rank: the contiguous partition of sharding.shard_range.
__device__ __forceinline__ void split_range(const WS& ws, int count, int* lo, int* hi) {
    *lo = (int)((long long)ws.split_rank * count / ws.split_world);
    *hi = (int)((long long)(ws.split_rank + 1) * count / ws.split_world);
}

// The workspace restricted to pairs [p0, p0 + count): every per-pair array advanced by p0 strides.
inline WS ws_view(const WS& w, int p0, size_t result_bytes) {
    WS v = w;
    v.desc = w.desc + p0;
    v.st = w.st + p0;
    v.src4 = w.src4 + p0 * w.pts_stride;
    v.dst4 = w.dst4 + p0 * w.pts_stride;
    v.bits = w.bits + p0 * w.bits_stride;
    if (w.bits_base) v.bits_base = w.bits_base + p0 * w.bits_stride;
    v.deg = w.deg + p0 * w.row_stride;
    v.row_gt = w.row_gt + p0 * w.row_stride;
    v.row_eq = w.row_eq + p0 * w.row_stride;
    v.row_take = w.row_take + p0 * w.row_stride;
    v.row_off = w.row_off + p0 * w.row_stride;
    v.edges = w.edges + p0 * w.edges_stride;
    v.rowptr = w.rowptr + p0 * w.rp_stride;
    v.piv = w.piv + p0 * w.piv_stride;
    v.cand = w.cand + (int64_t)p0 * PIV_CAP;
    v.cliq = w.cliq + p0 * w.cl_stride;
    v.hyp = w.hyp + p0 * w.cl_stride * 16;
    v.res = static_cast<char*>(w.res) + p0 * result_bytes;
    v.deg_full = w.deg_full + p0 * w.row_stride;
    v.hpos = w.hpos + p0 * w.row_stride;
    v.heavy_list = w.heavy_list + (int64_t)p0 * w.heavy_cap;
    v.lists = w.lists + p0 * w.lists_stride;
    v.light_list = w.light_list + p0 * w.row_stride;
    v.dense_list = w.dense_list + p0 * w.row_stride;
    v.heavy_mask = w.heavy_mask + p0 * (w.bits_stride / w.row_stride);
    v.light_mask = w.light_mask + p0 * (w.bits_stride / w.row_stride);
    v.heavy_UP = w.heavy_UP + p0 * w.heavy_UP_stride;
    v.heavy_X = w.heavy_X + p0 * w.heavy_X_stride;
    if (w.heavy_D) v.heavy_D = w.heavy_D + p0 * w.heavy_D_stride;
    v.pair_base = w.pair_base + p0;
    if (w.uprefix) v.uprefix = w.uprefix + p0 * w.bits_stride;
    if (w.herr) v.herr = w.herr + p0 * w.cl_stride * SCORE_SEGS_MAX;
    return v;
}


// Row i restricted to its upper part U_i = {c > i} (the O2 out-neighbourhood, Def. 2).
__device__ __forceinline__ uint32_t upper_mask(uint32_t v, int w, int i) {
    int lo = w * 32;
    if (lo + 31 <= i) return 0u;
    if (lo > i) return v;
    int s = i - lo;  // clear bits 0..s
    return v & ~((2u << s) - 1u);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(FULL, v, o);
        v = u > v ? u : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(FULL, v, o);
        v = u < v ? u : v;
    }
    return v;
}
__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

}  // namespace trk
