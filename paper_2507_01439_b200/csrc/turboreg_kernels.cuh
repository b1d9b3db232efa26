// =====================================================================================================
// TurboReg hot-path kernels for sm_100a (B200).  Included once, by turboreg_runtime.cu.
//
// Every kernel takes a batch of independent registration pairs (grid.y / grid.z = pair) and reads its
// pair's geometry from a PairDesc.  Data layout per pair:
//   src4/dst4  float4[n]          correspondences (x, y, z, 0)
//   bits       uint32[n][W]       rows of C(τ); bit c of word c/32 = C_rc; W = ceil(n/32) rounded up to 4
//   edges      uint32[E]          compact CSR of the O2 rows: row i's upper edges (j > i) in increasing j at
//                                 rowptr[i]: (j << 16) | Ĝ_ij   ("rank-indexed" O2 weights, Def. 2)
//   rowptr     int32[n+1]         exclusive scan of the upper degrees
//   deg        int32[n]           upper degree of row i
//   piv        int4[K1]           (i, j, Ĝ_ij, 0) in lexicographic order
//   cliq       int4[K1*K2]        (i, j, z, S) per slot pivot*K2 + r; empty (-1,-1,-1,0)
//   hyp        float[K1*K2][16]   R[9], t[3], count, flag, S, 0
// Float32 arithmetic that decides an integer (Eq. 1 edges, inlier tests) uses explicit _rn intrinsics
// in exactly the oracle's expression tree (readings r1, r13) so no contraction can change a bit.
// =====================================================================================================
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
    int32_t pad[1];
    uint32_t bbox[12];     // order keys of max src xyz, -min src xyz, max dst xyz, -min dst xyz (k_ingest)
    int32_t hist_hi[256];  // histogram of Ĝ_ij >> 7 over positive O2 edges
    int32_t hist_lo[128];  // histogram of Ĝ_ij & 127 within bin b1
};

constexpr int PIV_CAP = 8192;  // pivot candidates sorted in shared memory per pair

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
    int64_t edges_stride;
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
    uint16_t* lists;      // [n][LIST_MAX] sorted neighbour lists of rows with degree <= LIST_MAX
    int32_t* light_list;  // [n] sparse non-heavy rows, index order
    int32_t* dense_list;  // [n] all other rows, index order
    int64_t lists_stride;
    uint32_t* heavy_mask; // [W] bitset of H
    uint32_t* light_mask; // [W] bitset of the sparse rows (k_sc2_light's rows)
    uint2* heavy_UP;      // [cap][W] per heavy row a: (U_{H_a} word, exclusive prefix popcount of U_{H_a})
    int64_t heavy_UP_stride;
    uint8_t* heavy_X;     // [cap][Kcap] uint8 rows of C restricted to H
    int64_t heavy_X_stride;
    int32_t heavy_Kcap;
    int32_t heavy_cap;    // max |H| (multiple of 256)
    uint16_t* heavy_D;    // [cap][cap] X X^T (+ sparse-column correction)
    int64_t heavy_D_stride;
    int32_t heavy_min_rows, heavy_min_deg, sc2_path;
    float tau, tau_base, thr;
    int32_t k1, k2, mode;
    int32_t pair_base;    // index of pair 0 of this view in the batch (TMA coordinates address the whole batch)
    uint16_t* uprefix;    // SC^2 mode only: [n][W] exclusive prefix popcount of U_i per word (stride bits_stride)
    double2* herr;        // [K1*K2] per hypothesis (Σ sqrtf(s), Σ s) over the pair's correspondences (r20)
    int32_t err_mode;     // bit 0: accumulate herr; rank = err_mode >> 1: 0 inlier number, 1 MAE, 2 MSE
};

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
    v.heavy_D = w.heavy_D + p0 * w.heavy_D_stride;
    v.pair_base = w.pair_base + p0;
    if (w.uprefix) v.uprefix = w.uprefix + p0 * w.bits_stride;
    v.herr = w.herr + p0 * w.cl_stride;
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

// ------------------------------------------------------------------------------------------ a1 ingest
// Monotone map float -> uint32 (larger float, larger key; keys of finite floats are > 0).
__device__ __forceinline__ uint32_t float_order_key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float float_from_order_key(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// κ = τ² + 2^-21 S_max (1 + 2^-20), rounded up, with S_max = diam²(src) + diam²(dst) from the bounding boxes
// (an upper bound of |Δs|² + |Δd|² for every pair): the S-dependent term of the compat filter's margin Tq
// bounded once per pair.
__device__ __forceinline__ float compat_kappa(const PairState* st, float t2) {
    double smax = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double es = (double)float_from_order_key(st->bbox[c]) + (double)float_from_order_key(st->bbox[3 + c]);
        const double ed = (double)float_from_order_key(st->bbox[6 + c]) + (double)float_from_order_key(st->bbox[9 + c]);
        smax += es * es + ed * ed;
    }
    return __double2float_ru((double)t2 + ldexp(smax * (1.0 + 0x1p-20), -21));
}

// Repack the caller's N×3 float32 rows into float4 (x, y, z, 0) and flag non-finite input.
__global__ void __launch_bounds__(256) k_ingest(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (k < d.n) {
        float sx = d.src[3 * k], sy = d.src[3 * k + 1], sz = d.src[3 * k + 2];
        float tx = d.dst[3 * k], ty = d.dst[3 * k + 1], tz = d.dst[3 * k + 2];
        bad = !(isfinite(sx) && isfinite(sy) && isfinite(sz) && isfinite(tx) && isfinite(ty) && isfinite(tz));
        ws.src4[p * ws.pts_stride + k] = make_float4(sx, sy, sz, 0.f);
        ws.dst4[p * ws.pts_stride + k] = make_float4(tx, ty, tz, 0.f);
    }
    // bounding boxes (order-preserving float keys, atomicMax; 0 = empty): the compat filter's S bound
    float v[12];
    if (k < d.n && !bad) {
        const float4 a = ws.src4[p * ws.pts_stride + k], b = ws.dst4[p * ws.pts_stride + k];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = -a.x; v[4] = -a.y; v[5] = -a.z;
        v[6] = b.x; v[7] = b.y; v[8] = b.z; v[9] = -b.x; v[10] = -b.y; v[11] = -b.z;
    }
#pragma unroll
    for (int c = 0; c < 12; ++c) {
        const uint32_t key = (k < d.n && !bad) ? float_order_key(v[c]) : 0u;
        const uint32_t m = __reduce_max_sync(FULL, key);
        if ((threadIdx.x & 31) == 0 && m) atomicMax(&ws.st[p].bbox[c], m);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ws.st[p].nonfinite, 1);
}

// ------------------------------------------------------------------------------------------ a2 compat
// Eq. 1 on 32×32 tiles of the upper block triangle.  One warp per pair of adjacent tiles
// (I, J), (I, J+1), J >= I: lane l owns column points J*32+l and J*32+32+l; the 32 row points I*32+r are
// staged in shared memory and read as broadcasts.  Each test is evaluated once: the lane's own bit
// accumulation is the column word (c, I), its warp transpose the row word (I*32+r, J) — exact because
// IEEE subtraction is antisymmetric.
//
// The decision must equal the oracle's float32 tree bit for bit: a = sqrt.rn((dx*dx + dy*dy) + dz*dz),
// b likewise, edge ⇔ |a - b| <= τ (readings r1, r2).  Two correctly rounded square roots per test are
// the expensive part, so a certified filter decides first, without square roots.  With A = a², B = b²,
// S = A + B:
//   S < τ²  ⇒ edge;   S > τ²  ⇒ ( edge ⇔ q := (A − B)² − τ²(2S − τ²) <= 0 )     (q = (S−τ²)² − 4AB)
// In float32 (ε = 2^-24, FMAs) the error of q is below 8ε|A−B|S + 15ετ²S and the filter decides only when
// S > τ²(1 + 2^-16) and |q| > Tq = 2^-19 (|A−B| + κ) S, κ = τ² + 2^-21 S_max (1 + 2^-20) >= τ² + 2^-21 S,
// S_max = diam²(src) + diam²(dst) from the pair's bounding boxes.  These margins also exceed the oracle's
// own float32 rounding band around τ (|Δ − τ| <= 2^-22 (a + b)), so wherever the filter decides it
// provably agrees with the exact tree.  The rest — pairs with |Δ − τ| ≲ 2^-20 (a + b), a
// few per million, and pairs whose points nearly coincide in both clouds (S <= τ²(1 + 2^-16)) — are
// re-evaluated with the exact tree after the tile loop (lanes that met one redo their tests), so the common
// path carries no branch.
__device__ __forceinline__ float f32_dist(float ax, float ay, float az, float bx, float by, float bz) {
    float dx = __fsub_rn(ax, bx), dy = __fsub_rn(ay, by), dz = __fsub_rn(az, bz);
    return __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz)));
}

// Packed float32 pairs (sm_100 f32x2 ALU ops: two IEEE round-to-nearest results per instruction).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    return (f2_t)__float_as_uint(lo) | ((f2_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint32_t f2_lo(f2_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t f2_hi(f2_t v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ float lo_f(f2_t v) { return __uint_as_float(f2_lo(v)); }
__device__ __forceinline__ float hi_f(f2_t v) { return __uint_as_float(f2_hi(v)); }

// Warp-level 32×32 bit-matrix transpose: lane l holds row l (bit b = column b); returns column l.
__device__ __forceinline__ uint32_t transpose32(uint32_t x) {
    const int lane = threadIdx.x & 31;
    const uint32_t masks[5] = {0xffff0000u, 0xff00ff00u, 0xf0f0f0f0u, 0xccccccccu, 0xaaaaaaaau};
#pragma unroll
    for (int st = 0; st < 5; ++st) {
        const int sft = 16 >> st;
        const uint32_t m = masks[st];
        const uint32_t y = __shfl_xor_sync(FULL, x, sft);
        x = (lane & sft) ? ((x & m) | ((y >> sft) & ~m)) : ((x & ~m) | ((y << sft) & m));
    }
    return x;
}

// One 32×32 tile (I, J >= I) by one warp, with the optional τ_base plane (r19): both planes need the exact
// tree value of |a − b|, so this path evaluates it directly (lane = column, rows broadcast from shared memory).
__device__ __forceinline__ void compat_tile_base(const WS& ws, int p, int n, int W, int T, int I, int J,
                                                 const float4* s_rs, const float4* s_rd) {
    const int lane = threadIdx.x & 31;
    const float4* s4 = ws.src4 + p * ws.pts_stride;
    const float4* d4 = ws.dst4 + p * ws.pts_stride;
    const int c = J * 32 + lane;
    const bool cv = c < n;
    const float4 cs = cv ? s4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 cd = cv ? d4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int r0 = I * 32 + lane;
    const bool rv = r0 < n;
    const float tau = ws.tau, taub = ws.tau_base;
    const int rmax = min(32, n - I * 32);
    // validity masks: column word bit r ⇔ row I*32+r exists (and is not this lane's own point);
    // row word bit l ⇔ column J*32+l exists (and is not this lane's own point)
    uint32_t okc = cv ? (rmax >= 32 ? 0xffffffffu : ((1u << rmax) - 1u)) : 0u;
    const uint32_t cvb = __ballot_sync(FULL, cv);
    uint32_t okr = rv ? cvb : 0u;
    if (I == J) { okc &= ~(1u << lane); okr &= ~(1u << lane); }
    uint32_t colw = 0, roww = 0, colb = 0, rowb = 0;
    for (int r = 0; r < 32; ++r) {
        const float4 ps = s_rs[r];
        const float4 pd = s_rd[r];
        const float a = f32_dist(ps.x, ps.y, ps.z, cs.x, cs.y, cs.z);
        const float b = f32_dist(pd.x, pd.y, pd.z, cd.x, cd.y, cd.z);
        const float delta = fabsf(__fsub_rn(a, b));
        const bool e = delta <= tau, eb = delta <= taub;
        colw |= e ? (1u << r) : 0u;
        colb |= eb ? (1u << r) : 0u;
        const uint32_t bal = __ballot_sync(FULL, e), balb = __ballot_sync(FULL, eb);
        roww = (lane == r) ? bal : roww;
        rowb = (lane == r) ? balb : rowb;
    }
    colw &= okc;
    roww &= okr;
    uint32_t* bits = ws.bits + p * ws.bits_stride;
    if (rv) bits[(int64_t)r0 * W + J] = roww;
    if (cv) bits[(int64_t)c * W + I] = colw;
    if (I == J && rv)
        for (int w = T; w < W; ++w) bits[(int64_t)r0 * W + w] = 0u;
    {
        colb &= okc;
        rowb &= okr;
        uint32_t* bb = ws.bits_base + p * ws.bits_stride;
        if (rv) bb[(int64_t)r0 * W + J] = rowb;
        if (cv) bb[(int64_t)c * W + I] = colb;
        if (I == J && rv)
            for (int w = T; w < W; ++w) bb[(int64_t)r0 * W + w] = 0u;
        // edge count of the τ_base plane (upper triangle only)
        int cntb = (I == J) ? __popc(colb & ((lane == 0) ? 0u : (0xffffffffu >> (32 - lane)))) : __popc(colb);
        cntb = __reduce_add_sync(FULL, (unsigned)cntb);
        if (lane == 0 && cntb) atomicAdd(&ws.st[p].edges_base, cntb);
    }
}

// Block b of a pair owns block-rows I = b and I = T-1-b (equal work: T+1 tiles); its 8 warps sweep J.
// Two adjacent 32×32 tiles (I, J) and (I, J+1) by one warp, J >= I: lane l owns column points
// c0 = J*32+l and c1 = c0+32, packed as one f32x2 lane pair, so each row point (a shared-memory broadcast,
// stored negated) serves two tests per f32x2 op and the row loads are amortised over 64 columns.  The
// arithmetic per test is the same op for op in every tiling (same FMAs, same rounding): only the packing
// differs, so DESIGN.md §6.1's proof covers all of them.
template <int NP, int UNR>
__device__ __forceinline__ void compat_tiles(const WS& ws, int p, int n, int W, int T, int I, int J,
                                             const float4* s_rs, const float4* s_rd, const float4* s_nr,
                                             const float4* s_nd, f2_t* s_col, float kap) {
    constexpr int NT = 2 * NP;  // tiles (I, J) .. (I, J+NT-1); lane column k: (J+k)*32 + lane
    const int lane = threadIdx.x & 31;
    const float4* s4 = ws.src4 + p * ws.pts_stride;
    const float4* d4 = ws.dst4 + p * ws.pts_stride;
    const int r0 = I * 32 + lane;
    const bool rv = r0 < n;
    const float tau = ws.tau;
    const int rmax = min(32, n - I * 32);
    const uint32_t rmask = rmax >= 32 ? 0xffffffffu : ((1u << rmax) - 1u);
    // the column pairs (k = 2m, 2m+1) go through the warp's shared-memory slot so each arrives as one
    // 64-bit load and stays an aligned register pair for the whole loop (ptxas re-packs scalar-built pairs
    // on every use)
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NT; ++k) {
        const int c = (J + k) * 32 + lane;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 cs = c < n ? s4[c] : z4, cd = c < n ? d4[c] : z4;
        float* sc = reinterpret_cast<float*>(s_col) + (k & 1);
        sc[2 * ((0 * NP + (k >> 1)) * 32 + lane)] = cs.x;
        sc[2 * ((1 * NP + (k >> 1)) * 32 + lane)] = cs.y;
        sc[2 * ((2 * NP + (k >> 1)) * 32 + lane)] = cs.z;
        sc[2 * ((3 * NP + (k >> 1)) * 32 + lane)] = cd.x;
        sc[2 * ((4 * NP + (k >> 1)) * 32 + lane)] = cd.y;
        sc[2 * ((5 * NP + (k >> 1)) * 32 + lane)] = cd.z;
    }
    __syncwarp();
    f2_t CX[NP], CY[NP], CZ[NP], DX[NP], DY[NP], DZ[NP];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
        CX[m] = s_col[(0 * NP + m) * 32 + lane];
        CY[m] = s_col[(1 * NP + m) * 32 + lane];
        CZ[m] = s_col[(2 * NP + m) * 32 + lane];
        DX[m] = s_col[(3 * NP + m) * 32 + lane];
        DY[m] = s_col[(4 * NP + m) * 32 + lane];
        DZ[m] = s_col[(5 * NP + m) * 32 + lane];
    }
    const float t2 = __fmul_rn(tau, tau);
    const float t4 = __fmul_rn(t2, t2);
    const f2_t t2x2 = f2_pack(t2, t2), m2t2x2 = f2_pack(-2.0f * t2, -2.0f * t2), t4x2 = f2_pack(t4, t4);
    const f2_t nc19 = f2_pack(-0x1p-19f, -0x1p-19f);
    const f2_t mone = f2_pack(-1.0f, -1.0f);
    const float s_hi = __fmul_rn(t2, 1.0f + 0x1p-16f);
    const f2_t s_hi2 = f2_pack(s_hi, s_hi);
    const f2_t kap2 = f2_pack(kap, kap);
    // per test, in bit 31:  cc: S > s_hi (q decides);  b: |q| < Tq (q unsure);  q: q < 0.
    // decided x = ~b & cc;  edge e = x & q;  sacc keeps bit 31 while all decided.
    uint32_t colw[NT], sacc = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < NT; ++k) colw[k] = 0u;
#pragma unroll UNR
    for (int r = 0; r < 32; ++r) {
        const float4 R = s_nr[r];
        const float4 Q = s_nd[r];
#pragma unroll
        for (int m = 0; m < NP; ++m) {
            const f2_t dx = f2_add(CX[m], f2_pack(R.x, R.x)), dy = f2_add(CY[m], f2_pack(R.y, R.y));
            const f2_t dz = f2_add(CZ[m], f2_pack(R.z, R.z));
            const f2_t ex = f2_add(DX[m], f2_pack(Q.x, Q.x)), ey = f2_add(DY[m], f2_pack(Q.y, Q.y));
            const f2_t ez = f2_add(DZ[m], f2_pack(Q.z, Q.z));
            const f2_t A = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
            const f2_t B = f2_fma(ez, ez, f2_fma(ey, ey, f2_mul(ex, ex)));
            const f2_t S = f2_add(A, B);
            const f2_t D = f2_fma(B, mone, A);
            const f2_t q = f2_fma(D, D, f2_fma(S, m2t2x2, t4x2));
            const f2_t absD = D & 0x7fffffff7fffffffull;
            const f2_t nTq = f2_mul(f2_add(absD, kap2), f2_mul(S, nc19));
            const f2_t b = f2_add(nTq, q & 0x7fffffff7fffffffull);  // |q| − Tq
            const f2_t cc = f2_fma(S, mone, s_hi2);
            const uint32_t k0 = f2_lo(cc), k1 = f2_hi(cc);
            const uint32_t x0 = ~f2_lo(b) & k0, x1 = ~f2_hi(b) & k1;
            colw[2 * m] = __funnelshift_l(x0 & f2_lo(q), colw[2 * m], 1);
            colw[2 * m + 1] = __funnelshift_l(x1 & f2_hi(q), colw[2 * m + 1], 1);
            sacc &= x0 & x1;
        }
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) colw[k] = __brev(colw[k]);
    const bool unsure_any = (int32_t)sacc >= 0;
    if (__any_sync(FULL, unsure_any)) {  // rare: redo this lane's tests with the exact tree
        if (unsure_any) {
#pragma unroll
            for (int m = 0; m < NP; ++m) {
                uint32_t w0 = 0u, w1 = 0u;
                for (int r = 0; r < 32; ++r) {
                    const float4 ps = s_rs[r];
                    const float4 pd = s_rd[r];
                    const float a0 = f32_dist(ps.x, ps.y, ps.z, lo_f(CX[m]), lo_f(CY[m]), lo_f(CZ[m]));
                    const float b0 = f32_dist(pd.x, pd.y, pd.z, lo_f(DX[m]), lo_f(DY[m]), lo_f(DZ[m]));
                    const float a1 = f32_dist(ps.x, ps.y, ps.z, hi_f(CX[m]), hi_f(CY[m]), hi_f(CZ[m]));
                    const float b1 = f32_dist(pd.x, pd.y, pd.z, hi_f(DX[m]), hi_f(DY[m]), hi_f(DZ[m]));
                    w0 |= (fabsf(__fsub_rn(a0, b0)) <= tau) ? (1u << r) : 0u;
                    w1 |= (fabsf(__fsub_rn(a1, b1)) <= tau) ? (1u << r) : 0u;
                }
                colw[2 * m] = w0;
                colw[2 * m + 1] = w1;
            }
        }
    }
    uint32_t* bits = ws.bits + p * ws.bits_stride;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
        const int c = (J + k) * 32 + lane;
        const bool cv = c < n;
        uint32_t okc = cv ? rmask : 0u;
        const uint32_t cvb = __ballot_sync(FULL, cv);  // every lane votes (never inside a conditional)
        uint32_t okr = rv ? cvb : 0u;
        if (I == J + k) { okc &= ~(1u << lane); okr &= ~(1u << lane); }
        const uint32_t cw = colw[k] & okc;
        const uint32_t rw = transpose32(cw) & okr;
        if (rv && J + k < T) bits[(int64_t)r0 * W + J + k] = rw;
        if (cv) bits[(int64_t)c * W + I] = cw;
    }
    if (I == J && rv)
        for (int w = T; w < W; ++w) bits[(int64_t)r0 * W + w] = 0u;
}

// Row-pair packing: the f32x2 lanes hold two row points (2k, 2k+1) of tile row I (negated, from shared
// memory, one LDS.128 + one LDS.64 per coordinate triple), each lane's NC column points are scalar
// broadcast operands held in registers.  Same per-test arithmetic as compat_tiles.
template <int NC, int UNR>
__device__ __forceinline__ void compat_tiles_rp(const WS& ws, int p, int n, int W, int T, int I, int J,
                                                const float4* s_rs, const float4* s_rd, const float4* s_pxy,
                                                const float2* s_pz, const float4* s_qxy, const float2* s_qz,
                                                float kap) {
    const int lane = threadIdx.x & 31;
    const float4* s4 = ws.src4 + p * ws.pts_stride;
    const float4* d4 = ws.dst4 + p * ws.pts_stride;
    const int r0 = I * 32 + lane;
    const bool rv = r0 < n;
    const float tau = ws.tau;
    const int rmax = min(32, n - I * 32);
    const uint32_t rmask = rmax >= 32 ? 0xffffffffu : ((1u << rmax) - 1u);
    float4 cs[NC], cd[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const int c = (J + k) * 32 + lane;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        cs[k] = c < n ? s4[c] : z4;
        cd[k] = c < n ? d4[c] : z4;
    }
    const float t2 = __fmul_rn(tau, tau);
    const float t4 = __fmul_rn(t2, t2);
    const f2_t t2x2 = f2_pack(t2, t2), m2t2x2 = f2_pack(-2.0f * t2, -2.0f * t2), t4x2 = f2_pack(t4, t4);
    const f2_t nc19 = f2_pack(-0x1p-19f, -0x1p-19f);
    const f2_t mone = f2_pack(-1.0f, -1.0f);
    const float s_hi = __fmul_rn(t2, 1.0f + 0x1p-16f);
    const f2_t s_hi2 = f2_pack(s_hi, s_hi);
    const f2_t kap2 = f2_pack(kap, kap);
    uint32_t colw[NC], sacc = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < NC; ++k) colw[k] = 0u;
#pragma unroll UNR
    for (int kk = 0; kk < 16; ++kk) {
        const float4 P = s_pxy[kk];
        const float2 Pz = s_pz[kk];
        const float4 Q = s_qxy[kk];
        const float2 Qz = s_qz[kk];
        const f2_t px = f2_pack(P.x, P.y), py = f2_pack(P.z, P.w), pz = f2_pack(Pz.x, Pz.y);
        const f2_t qx = f2_pack(Q.x, Q.y), qy = f2_pack(Q.z, Q.w), qz = f2_pack(Qz.x, Qz.y);
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const f2_t dx = f2_add(px, f2_pack(cs[k].x, cs[k].x)), dy = f2_add(py, f2_pack(cs[k].y, cs[k].y));
            const f2_t dz = f2_add(pz, f2_pack(cs[k].z, cs[k].z));
            const f2_t ex = f2_add(qx, f2_pack(cd[k].x, cd[k].x)), ey = f2_add(qy, f2_pack(cd[k].y, cd[k].y));
            const f2_t ez = f2_add(qz, f2_pack(cd[k].z, cd[k].z));
            const f2_t A = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
            const f2_t B = f2_fma(ez, ez, f2_fma(ey, ey, f2_mul(ex, ex)));
            const f2_t S = f2_add(A, B);
            const f2_t D = f2_fma(B, mone, A);
            const f2_t q = f2_fma(D, D, f2_fma(S, m2t2x2, t4x2));
            const f2_t absD = D & 0x7fffffff7fffffffull;
            const f2_t nTq = f2_mul(f2_add(absD, kap2), f2_mul(S, nc19));
            const f2_t b = f2_add(nTq, q & 0x7fffffff7fffffffull);  // |q| − Tq
            const f2_t cc = f2_fma(S, mone, s_hi2);
            const uint32_t k0 = f2_lo(cc), k1 = f2_hi(cc);
            const uint32_t x0 = ~f2_lo(b) & k0, x1 = ~f2_hi(b) & k1;
            colw[k] = __funnelshift_l(x0 & f2_lo(q), colw[k], 1);
            colw[k] = __funnelshift_l(x1 & f2_hi(q), colw[k], 1);
            sacc &= x0 & x1;
        }
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) colw[k] = __brev(colw[k]);
    const bool unsure_any = (int32_t)sacc >= 0;
    if (__any_sync(FULL, unsure_any)) {  // rare: redo this lane's tests with the exact tree
        if (unsure_any) {
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                uint32_t w0 = 0u;
                for (int r = 0; r < 32; ++r) {
                    const float4 ps = s_rs[r];
                    const float4 pd = s_rd[r];
                    const float a0 = f32_dist(ps.x, ps.y, ps.z, cs[k].x, cs[k].y, cs[k].z);
                    const float b0 = f32_dist(pd.x, pd.y, pd.z, cd[k].x, cd[k].y, cd[k].z);
                    w0 |= (fabsf(__fsub_rn(a0, b0)) <= tau) ? (1u << r) : 0u;
                }
                colw[k] = w0;
            }
        }
    }
    uint32_t* bits = ws.bits + p * ws.bits_stride;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const int c = (J + k) * 32 + lane;
        const bool cv = c < n;
        uint32_t okc = cv ? rmask : 0u;
        const uint32_t cvb = __ballot_sync(FULL, cv);  // every lane votes (never inside a conditional)
        uint32_t okr = rv ? cvb : 0u;
        if (I == J + k) { okc &= ~(1u << lane); okr &= ~(1u << lane); }
        const uint32_t cw = colw[k] & okc;
        const uint32_t rw = transpose32(cw) & okr;
        if (rv && J + k < T) bits[(int64_t)r0 * W + J + k] = rw;
        if (cv) bits[(int64_t)c * W + I] = cw;
    }
    if (I == J && rv)
        for (int w = T; w < W; ++w) bits[(int64_t)r0 * W + w] = 0u;
}

template <bool BASE, int MINB = 4, int UNR = 8, int NP = 1>
__global__ void __launch_bounds__(256, MINB) k_compat(WS ws, int split) {
    __shared__ float4 s_rs[64];
    __shared__ float4 s_rd[64];
    __shared__ float4 s_pxy[2][16];
    __shared__ float2 s_pz[2][16];
    __shared__ float4 s_qxy[2][16];
    __shared__ float2 s_qz[2][16];
    __shared__ float4 s_nr[64];
    __shared__ float4 s_nd[64];
    __shared__ f2_t s_col[8][6 * 32 * (NP > 0 ? NP : 1)];
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int W = d.W;
    const int T = (n + 31) >> 5;
    // `split` blocks share a block-row pair (small batches: enough blocks to fill the GPU); block part sp
    // takes every split-th item of the pair's work list
    const int b = blockIdx.x / split, sp = blockIdx.x % split;
    if (2 * b >= T) return;
    const int warp = threadIdx.x >> 5;
    const float4* s4 = ws.src4 + p * ws.pts_stride;
    const float4* d4 = ws.dst4 + p * ws.pts_stride;
    if constexpr (BASE) {
        for (int half = 0; half < 2; ++half) {
            const int I = half == 0 ? b : T - 1 - b;
            if (half == 1 && I == b) break;
            __syncthreads();
            if (threadIdx.x < 32) {
                const int t = threadIdx.x, r0 = I * 32 + t;
                const float4 a = r0 < n ? s4[r0] : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 q = r0 < n ? d4[r0] : make_float4(0.f, 0.f, 0.f, 0.f);
                s_rs[t] = a;
                s_rd[t] = q;
            }
            __syncthreads();
            for (int J = I + warp + 8 * sp; J < T; J += 8 * split)
                compat_tile_base(ws, p, n, W, T, I, J, s_rs, s_rd);
        }
    } else {
        // block-rows I0 = b and I1 = T-1-b (T+1 tiles together, so every block has the same work) are
        // staged at once and their tile pairs dealt to the 8 warps as one list: no barrier between them
        const int I0 = b, I1 = T - 1 - b;
        __shared__ float s_kap;
        if (threadIdx.x == 0) s_kap = compat_kappa(ws.st + p, __fmul_rn(ws.tau, ws.tau));
        if (threadIdx.x < 64) {
            const int t = threadIdx.x, I = t < 32 ? I0 : I1, r0 = I * 32 + (t & 31);
            const float4 a = r0 < n ? s4[r0] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 q = r0 < n ? d4[r0] : make_float4(0.f, 0.f, 0.f, 0.f);
            s_rs[t] = a;
            s_rd[t] = q;
            s_nr[t] = make_float4(-a.x, -a.y, -a.z, 0.f);
            s_nd[t] = make_float4(-q.x, -q.y, -q.z, 0.f);
            const int h = t >> 5, u = t & 31;
            float* pxy = reinterpret_cast<float*>(s_pxy[h]) + 4 * (u >> 1) + (u & 1);
            float* qxy = reinterpret_cast<float*>(s_qxy[h]) + 4 * (u >> 1) + (u & 1);
            pxy[0] = -a.x; pxy[2] = -a.y;
            qxy[0] = -q.x; qxy[2] = -q.y;
            reinterpret_cast<float*>(s_pz[h])[u] = -a.z;
            reinterpret_cast<float*>(s_qz[h])[u] = -q.z;
        }
        __syncthreads();
        const float kap = s_kap;
        if constexpr (NP < 0) {
            constexpr int NC = -NP;
            const int P0 = (T - I0 + NC - 1) / NC, P1 = (I1 != I0) ? (T - I1 + NC - 1) / NC : 0;
            for (int t = warp + 8 * sp; t < P0 + P1; t += 8 * split) {
                const bool second = t >= P0;
                const int I = second ? I1 : I0, J = I + NC * (second ? t - P0 : t), o = second ? 32 : 0, h = second;
                compat_tiles_rp<NC, UNR>(ws, p, n, W, T, I, J, s_rs + o, s_rd + o, s_pxy[h], s_pz[h], s_qxy[h],
                                         s_qz[h], kap);
            }
            return;
        }
        constexpr int NT = 2 * (NP > 0 ? NP : 1);
        const int P0 = (T - I0 + NT - 1) / NT, P1 = (I1 != I0) ? (T - I1 + NT - 1) / NT : 0;
        for (int t = warp + 8 * sp; t < P0 + P1; t += 8 * split) {
            const bool second = t >= P0;
            const int I = second ? I1 : I0, J = I + NT * (second ? t - P0 : t), o = second ? 32 : 0;
            compat_tiles<(NP > 0 ? NP : 1), UNR>(ws, p, n, W, T, I, J, s_rs + o, s_rd + o, s_nr + o, s_nd + o, s_col[warp], kap);
        }
    }
}

// ------------------------------------------------------------------------------------------ a3 SC^2
// Eq. 2 for every O2 edge (i < j), assembled in row i's rank order.  One warp per row i;
// U_i's words are enumerated lane-parallel (lane = word, rank = warp prefix of popcounts), one edge per
// lane per round:
//   * both endpoints heavy → Ĝ_ij was computed on the tensor cores: gather D[hpos i][hpos j];
//   * otherwise (the sparse remainder) → popcount(row_i AND row_j): row_i in registers (lane-strided),
//     G light edges at a time so G·WPL row_j loads are in flight, REDUX per edge.
// The result (j << 16 | Ĝ_ij) goes to edges[rowptr(i) + rank]; positive weights feed a 256-bin histogram
// of Ĝ >> 7 (the high digit of the pivot radix select, Eq. 4).
constexpr int SC2_WARPS = 8;
constexpr int SC2_ROWS_PER_BLOCK = 64;
constexpr int SEL_WARPS = 8;
constexpr int SEL_ROWS_PER_BLOCK = 64;
constexpr int LIST_MAX = 64;  // rows with degree <= LIST_MAX keep a sorted uint16 neighbour list
constexpr int MMA_BK_ = 128;  // K granularity of the tensor-core block (= MMA_BK)
// Row i as a byte map (one byte per column) trades the per-row expansion (~40 instructions per word) for
// cheaper list lookups; with a few dozen sparse neighbours per dense row it does not pay, so it is off.
constexpr bool SC2_BYTEMAP = false;
template <int WPL>
constexpr int sc2_warp_words() {  // U_i, rank prefix, row i, queue (+ row i as a byte map if enabled)
    return 96 * WPL + 32 * WPL + ((SC2_BYTEMAP && WPL <= 8) ? 32 * WPL * 32 / 4 : 0);
}
template <int WPL>
constexpr int sc2_smem_bytes() { return (SC2_WARPS * sc2_warp_words<WPL>() + 2 * 32 * WPL) * 4; }

// Dense rows (not sparse: heavy, or degree > LIST_MAX), one warp per row i, SC2_BLOCKS_PER_PAIR blocks of
// warps striding over the pair's dense rows.  Row i's edges come from three sources:
//   (1) i, j both heavy: written by the tensor-core epilogue (k_sc2_mma) or k_emit_hh, not here;
//   (2) j sparse (degree <= LIST_MAX, sorted neighbour list L_j), on EITHER side of i:
//       Ĝ_ij = |L_j ∩ N(i)|, one edge per lane, list entries tested against row i's bitmap in shared
//       memory.  For j > i the result goes to row i's slot; for j < i to row j's slot, whose rank
//       (entries of L_j below i, minus those up to j) falls out of the same pass over L_j;
//   (3) both dense but not both heavy (rare): warp-cooperative popcount(row_i AND row_j).
// Sparse-sparse edges are k_sc2_light's.  Every O2 edge is therefore written exactly once.
constexpr int SC2_PERSIST_BLOCKS_PER_SM = 6;
constexpr int SC2_BLOCKS_PER_PAIR = 32;  // 256 warps stride over a pair's dense rows
constexpr int SC2_CLAIM = 4;

// |L ∩ N(i)| for a sorted list L of <= LIST_MAX uint16 entries (16-byte aligned, zero padded) against row
// i's bitmap in shared memory.  Entries past len are zeros, so a chunk is processed whole and the pad's
// bit 0 tests are subtracted once (row i's own bit 0 is read once).
__device__ __forceinline__ uint32_t list_bitmap_count(const uint16_t* L, int len, const uint32_t* sr) {
    const int nch = (len + 7) >> 3;
    uint4 v[LIST_MAX / 8];
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c)
        v[c] = (c < nch) ? __ldg(reinterpret_cast<const uint4*>(L) + c) : make_uint4(0, 0, 0, 0);
    uint32_t cnt = 0;
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c) {
        if (c < nch) {
            const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t k0 = wv[e] & 0xffffu, k1 = wv[e] >> 16;
                cnt += ((sr[k0 >> 5] >> (k0 & 31)) & 1u) + ((sr[k1 >> 5] >> (k1 & 31)) & 1u);
            }
        }
    }
    return cnt - (uint32_t)(nch * 8 - len) * (sr[0] & 1u);
}


// As list_bitmap_count, for an edge (j, i) with j < i stored in row j: also returns the rank of i among
// the entries of L_j above j (= #{x in L_j : j < x < i}).
__device__ __forceinline__ uint32_t list_bitmap_count_rank(const uint16_t* L, int len, const uint32_t* sr, int i,
                                                           int j, int* rank) {
    const int nch = (len + 7) >> 3;
    uint4 v[LIST_MAX / 8];
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c)
        v[c] = (c < nch) ? __ldg(reinterpret_cast<const uint4*>(L) + c) : make_uint4(0, 0, 0, 0);
    uint32_t cnt = 0;
    int r = 0;
    const unsigned span = (unsigned)(i - j - 1);
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c) {
        if (c < nch) {
            const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k0 = (int)(wv[e] & 0xffffu), k1 = (int)(wv[e] >> 16);
                cnt += ((sr[k0 >> 5] >> (k0 & 31)) & 1u) + ((sr[k1 >> 5] >> (k1 & 31)) & 1u);
                // j < k < i as one unsigned range test; pads are 0 <= j: never counted
                r += ((unsigned)(k0 - j - 1) < span) + ((unsigned)(k1 - j - 1) < span);
            }
        }
    }
    *rank = r;
    return cnt - (uint32_t)(nch * 8 - len) * (sr[0] & 1u);
}

// As list_bitmap_count_rank, against row i as a byte map (one byte per column, 0/1) in shared memory:
// one byte load per list entry instead of word load + shift + mask.
__device__ __forceinline__ uint32_t list_bytemap_count_rank(const uint16_t* L, int len, const uint8_t* sb, int i, int j,
                                                            int* rank) {
    const int nch = (len + 7) >> 3;
    uint4 v[LIST_MAX / 8];
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c)
        v[c] = (c < nch) ? __ldg(reinterpret_cast<const uint4*>(L) + c) : make_uint4(0, 0, 0, 0);
    uint32_t cnt = 0;
    int r = 0;
    const unsigned span = (unsigned)(i - j - 1);
#pragma unroll
    for (int c = 0; c < LIST_MAX / 8; ++c) {
        if (c < nch) {
            const uint32_t wv[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k0 = (int)(wv[e] & 0xffffu), k1 = (int)(wv[e] >> 16);
                cnt += (uint32_t)sb[k0] + (uint32_t)sb[k1];
                // j < k < i as one unsigned range test; pads are 0 <= j: never counted
                r += ((unsigned)(k0 - j - 1) < span) + ((unsigned)(k1 - j - 1) < span);
            }
        }
    }
    *rank = r;
    return cnt - (uint32_t)(nch * 8 - len) * (uint32_t)sb[0];
}

// Edge between dense row i (bitmap sr — or byte map sb when non-null —, U_i words su, rank prefix sp in
// shared memory) and sparse row j, on either side of i: one code path for both sides (no divergence).
__device__ __forceinline__ void sc2_sparse_edge(const WS& ws, const uint16_t* lists, const int32_t* deg_full,
                                                const int32_t* rowptr, uint32_t* edges, uint32_t* erow,
                                                const uint32_t* su, const int32_t* sp, const uint32_t* sr,
                                                const uint8_t* sb, int i, int j) {
    const uint16_t* L = lists + (int64_t)j * LIST_MAX;
    int rank;
    const uint32_t c = sb ? list_bytemap_count_rank(L, deg_full[j], sb, i, j, &rank)
                          : list_bitmap_count_rank(L, deg_full[j], sr, i, j, &rank);
    const int wj = j >> 5;
    uint32_t* dst = (j > i) ? erow + sp[wj] + __popc(su[wj] & ((1u << (j & 31)) - 1u)) : edges + rowptr[j] + rank;
    *dst = ((uint32_t)((j > i) ? j : i) << 16) | c;
}

template <int WPL>
__global__ void __launch_bounds__(SC2_WARPS * 32, 3) k_sc2(WS ws) {
    constexpr int G = 4;
    constexpr int QCAP = 32 * WPL;  // sparse-neighbour queue (a round adds at most 32 entries)
    extern __shared__ uint32_t s_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // block: heavy mask, sparse mask; per warp: U_i, rank prefix, row i, queue
    uint32_t* hm = s_dyn;
    uint32_t* lm = s_dyn + 32 * WPL;
    uint32_t* su = s_dyn + 64 * WPL + warp * sc2_warp_words<WPL>();
    int32_t* sp = reinterpret_cast<int32_t*>(su + 32 * WPL);
    uint32_t* sr = su + 64 * WPL;
    uint32_t* sq = su + 96 * WPL;
    uint8_t* sbm = (SC2_BYTEMAP && WPL <= 8) ? reinterpret_cast<uint8_t*>(su + 128 * WPL) : nullptr;
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
    for (int kq = blockIdx.x * SC2_WARPS + warp; kq < nd; kq += nw) {
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
                if (sbm) {  // bits of word w -> bytes 32w .. 32w+31 (two 16-byte stores)
                    uint32_t b[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const uint32_t nib = (reg[k] >> (4 * q)) & 0xfu;
                        b[q] = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
                    }
                    uint4* d = reinterpret_cast<uint4*>(sbm + 32 * w);
                    d[0] = make_uint4(b[0], b[1], b[2], b[3]);
                    d[1] = make_uint4(b[4], b[5], b[6], b[7]);
                }
                su[w] = u;
                sp[w] = carry + incl - cnt;
                carry += __shfl_sync(FULL, incl, 31);
            }
        }
        __syncwarp();
        // (2) sparse neighbours on both sides (queued, one edge per lane) and (3) dense-dense upper
        // neighbours that are not both heavy (warp-cooperative popcount)
        int nq = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int w = c * 32 + lane;
            const uint32_t lmw = (w < W) ? lm[w] : 0u;
            uint32_t ul = ((w < W) ? sr[w] : 0u) & lmw;
            uint32_t ud = ((w < W) ? su[w] : 0u) & ~lmw;
            if (hi >= 0 && w < W) ud &= ~hm[w];
            while (__any_sync(FULL, (ul | ud) != 0u)) {
                int jl = -1, jd = -1;
                if (ul) {
                    jl = w * 32 + __ffs(ul) - 1;
                    ul &= ul - 1u;
                } else if (ud) {
                    jd = w * 32 + __ffs(ud) - 1;
                    ud &= ud - 1u;
                }
                const unsigned sb = __ballot_sync(FULL, jl >= 0);
                if (jl >= 0) sq[nq + __popc(sb & ((1u << lane) - 1u))] = (uint32_t)jl;
                nq += __popc(sb);
                if (nq > QCAP - 32) {
                    __syncwarp();
                    for (int t = lane; t < nq; t += 32) sc2_sparse_edge(ws, lists, deg_full, rowptr, edges, erow, su, sp, sr, sbm, i, (int)sq[t]);
                    __syncwarp();
                    nq = 0;
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
                            erow[sp[wj] + __popc(su[wj] & ((1u << (j & 31)) - 1u))] = ((uint32_t)j << 16) | tot;
                        }
                    }
                }
            }
        }
        __syncwarp();
        for (int t = lane; t < nq; t += 32) sc2_sparse_edge(ws, lists, deg_full, rowptr, edges, erow, su, sp, sr, sbm, i, (int)sq[t]);
        __syncwarp();
    }
}

// Row classes for the SC^2 assembly: sparse rows (a list, not heavy) go to k_sc2_light, the rest to k_sc2.
__global__ void __launch_bounds__(1024) k_rowclass(WS ws) {
    __shared__ int s_w[32];
    __shared__ int s_carry;
    const int p = blockIdx.x;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int32_t* deg = ws.deg_full + p * ws.row_stride;
    const int32_t* hpos = ws.hpos + p * ws.row_stride;
    int32_t* L = ws.light_list + p * ws.row_stride;
    int32_t* Dn = ws.dense_list + p * ws.row_stride;
    if (t == 0) s_carry = 0;
    __syncthreads();
    for (int r0 = 0; r0 < n; r0 += 1024) {
        const int i = r0 + t;
        const int f = (i < n && hpos[i] < 0 && deg[i] <= LIST_MAX) ? 1 : 0;
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
        if (i < n) {
            if (f) L[pos] = i;
            else Dn[i - pos] = i;
        }
        const unsigned fb = __ballot_sync(FULL, f);
        if (lane == 0 && ((r0 + warp * 32) >> 5) < d.W)
            ws.light_mask[p * (ws.bits_stride / ws.row_stride) + ((r0 + warp * 32) >> 5)] = fb;
        __syncthreads();
        if (t == 1023) s_carry = pos + f;
        __syncthreads();
    }
    if (t == 0) { ws.st[p].n_light = s_carry; ws.st[p].n_dense = n - s_carry; }
    // compact CSR row pointers of the O2 edge lists: exclusive scan of the upper degrees
    __syncthreads();
    if (t == 0) s_carry = 0;
    __syncthreads();
    const int32_t* udeg = ws.deg + p * ws.row_stride;
    int32_t* rp = ws.rowptr + p * ws.rp_stride;
    for (int r0 = 0; r0 < n; r0 += 1024) {
        const int i = r0 + t;
        const int f = (i < n) ? udeg[i] : 0;
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
        if (i < n) rp[i] = pos;
        __syncthreads();
        if (t == 1023) s_carry = pos + f;
        __syncthreads();
    }
    if (t == 0) { rp[n] = s_carry; ws.st[p].edges = s_carry; }
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
constexpr int light_rows() { return WPL >= 16 ? 2 : 8; }  // LG: sparse rows per warp group
template <int WPL>
constexpr int light_warp_words() {
    return light_rows<WPL>() * 32 * WPL + light_rows<WPL>() * (LIST_MAX / 2) + 64 + 64 + 4 * light_rows<WPL>();
}
template <int WPL>
constexpr int light_smem_bytes() { return 8 * light_warp_words<WPL>() * 4; }

template <int WPL>
__device__ __forceinline__ void light_flush(const WS& ws, int p, const uint32_t* bm, const int32_t* meta,
                                            const uint32_t* q, int cnt) {
    const int lane = threadIdx.x & 31;
    const uint16_t* lists = ws.lists + p * ws.lists_stride;
    const int32_t* deg_full = ws.deg_full + p * ws.row_stride;
    if (lane < cnt) {
        const uint32_t e = q[lane];
        const int j = (int)(e & 0xffffu), t = (int)((e >> 16) & 63), r = (int)(e >> 22);
        const int i = meta[4 * r], lo = meta[4 * r + 2];
        const uint32_t c = list_bitmap_count(lists + (int64_t)j * LIST_MAX, deg_full[j], bm + r * 32 * WPL);
        ws.edges[p * ws.edges_stride + ws.rowptr[p * ws.rp_stride + i] + (t - lo)] = ((uint32_t)j << 16) | c;
    }
}

template <int WPL>
__global__ void __launch_bounds__(256) k_sc2_light(WS ws) {
    constexpr int LG = light_rows<WPL>();
    extern __shared__ uint32_t s_dyn[];
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    const int n = d.n;
    if (n == 0) return;
    const int W = d.W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nl = ws.st[p].n_light;
    const int g0 = (blockIdx.x * 8 + warp) * LG;
    if (g0 >= nl) return;
    const int nr = min(LG, nl - g0);
    uint32_t* bm = s_dyn + warp * light_warp_words<WPL>();
    uint16_t* ls = reinterpret_cast<uint16_t*>(bm + LG * 32 * WPL);
    uint32_t* qL = bm + LG * 32 * WPL + LG * (LIST_MAX / 2);
    uint32_t* qD = qL + 64;
    int32_t* meta = reinterpret_cast<int32_t*>(qD + 64);
    const uint32_t* bits = ws.bits + p * ws.bits_stride;
    const uint16_t* lists = ws.lists + p * ws.lists_stride;
    const int32_t* deg_full = ws.deg_full + p * ws.row_stride;
    const int32_t* light = ws.light_list + p * ws.row_stride;
    // stage the group's bitmaps and lists with asynchronous 16-byte copies (all rows in flight at once);
    // per-row meta (i, d, lo)
    int my_i = 0, my_d = 0;
    if (lane < nr) {
        my_i = light[g0 + lane];
        my_d = deg_full[my_i];
        meta[4 * lane] = my_i;
        meta[4 * lane + 1] = my_d;
    }
    __syncwarp();
    const int W4 = W >> 2;  // 16-byte chunks of a bit row (W is a multiple of 4)
    for (int idx = lane; idx < nr * W4; idx += 32) {
        const int r = idx / W4, c = idx - r * W4;
        cp_async16(bm + r * 32 * WPL + 4 * c, bits + (int64_t)meta[4 * r] * W + 4 * c);
    }
    for (int idx = lane; idx < nr * (LIST_MAX / 8); idx += 32) {
        const int r = idx / (LIST_MAX / 8), c = idx - r * (LIST_MAX / 8);
        uint16_t* dst = ls + r * LIST_MAX + 8 * c;
        if (c * 8 < meta[4 * r + 1]) cp_async16(dst, lists + (int64_t)meta[4 * r] * LIST_MAX + 8 * c);
        else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    int my_lo = 0;
    for (int r = 0; r < nr; ++r) {
        const int i = __shfl_sync(FULL, my_i, r), di = __shfl_sync(FULL, my_d, r);
        int c = 0;
        for (int t = lane; t < di; t += 32) c += (int)ls[r * LIST_MAX + t] <= i;
        c = __reduce_add_sync(FULL, (unsigned)c);
        if (lane == r) my_lo = c;
    }
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
    const int mstride = ws.bits_stride / ws.row_stride;
    const uint32_t* lmask = ws.light_mask + p * mstride;
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
            const int j = ls[r * LIST_MAX + t];
            packed = (uint32_t)j | ((uint32_t)t << 16) | ((uint32_t)r << 22);
            isL = (__ldg(lmask + (j >> 5)) >> (j & 31)) & 1u;  // sparse j; dense j is k_sc2's edge
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
constexpr int SEL_BLOCKS_PER_PAIR = 32;

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
    __shared__ int s_hist[256];
    const int p = blockIdx.y;
    if (ws.desc[p].n == 0) return;
    PairState* st = ws.st + p;
    const int E = st->edges;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) s_hist[b] = 0;
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
                if (run_bin >= 0) atomicAdd(&s_hist[run_bin], run);
                run_bin = bin;
                run = 0;
            }
            ++run;
        }
        if (run_bin >= 0) atomicAdd(&s_hist[run_bin], run);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (s_hist[b]) atomicAdd(&st->hist_hi[b], s_hist[b]);
}

// ------------------------------------------------------------------------------------------ a3 heavy split
// Full degrees (popcount of each bit row), their sum and maximum, and the sorted uint16 neighbour list of
// every row with degree <= LIST_MAX (zero-padded to a 16-byte chunk); one warp per row.
// Degrees and the sorted lists of sparse rows.  Lane l owns 8 consecutive words [g + 8l, g + 8l + 8) of a
// 256-word group (two 16-byte loads), so lane order is column order and one warp scan of the per-lane
// counts places every lane's entries; only rows with degree <= LIST_MAX extract their set bits.
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
__global__ void __launch_bounds__(256) k_degree(WS ws) {
    __shared__ unsigned long long s_sum;
    __shared__ int s_max;
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
    const int row0 = blockIdx.x * SEL_ROWS_PER_BLOCK, row1 = min(row0 + SEL_ROWS_PER_BLOCK, n);
    uint16_t* lists = ws.lists + p * ws.lists_stride;
    auto finish_row = [&](int i, int deg, int ucnt) {
        uint16_t* L = lists + (int64_t)i * LIST_MAX;
        if (deg <= LIST_MAX)
            for (int t = deg + lane; t < ((deg + 7) & ~7); t += 32) L[t] = 0;  // pad to a 16-byte chunk
        ucnt = (int)__reduce_add_sync(FULL, (unsigned)ucnt);
        if (lane == 0) { ws.deg_full[p * ws.row_stride + i] = deg; ws.deg[p * ws.row_stride + i] = ucnt; }
        mine += deg;
        mx = max(mx, deg);
    };
    if (W <= 256) {  // the whole row in registers; the next row's words are in flight meanwhile
        const int w0 = 8 * lane;
        uint32_t vn[8];
        if (row0 + warp < row1) deg_load8(bits + (int64_t)(row0 + warp) * W, w0, W, vn);
        for (int i = row0 + warp; i < row1; i += SEL_WARPS) {
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = vn[k];
            if (i + SEL_WARPS < row1) deg_load8(bits + (int64_t)(i + SEL_WARPS) * W, w0, W, vn);
            int cnt = 0, ucnt = 0, uc[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                cnt += __popc(v[k]);
                uc[k] = __popc(upper_mask(v[k], w0 + k, i));
                ucnt += uc[k];
            }
            const int incl = warp_incl_scan(cnt);
            const int deg = __shfl_sync(FULL, incl, 31);
            if (deg <= LIST_MAX) deg_extract8(v, w0, incl - cnt, lists + (int64_t)i * LIST_MAX);
            if (ws.uprefix) {  // SC^2 mode: rank of any j in U_i = uprefix[i][j>>5] + popc(U_i word below j)
                int run = warp_incl_scan(ucnt) - ucnt;
                uint32_t pk[4];
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    pk[k >> 1] = (uint32_t)run | ((uint32_t)(run + uc[k]) << 16);
                    run += uc[k] + uc[k + 1];
                }
                uint16_t* up = ws.uprefix + p * ws.bits_stride + (int64_t)i * W + w0;
                if (w0 < W) *reinterpret_cast<uint2*>(up) = make_uint2(pk[0], pk[1]);
                if (w0 + 4 < W) *reinterpret_cast<uint2*>(up + 4) = make_uint2(pk[2], pk[3]);
            }
            finish_row(i, deg, ucnt);
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
            if (deg <= LIST_MAX) {
                int carry = 0;
                for (int g = 0; g < W; g += 256) {
                    uint32_t v[8];
                    const int w0 = g + 8 * lane;
                    deg_load8(ri, w0, W, v);
                    int cnt = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) cnt += __popc(v[k]);
                    const int incl = warp_incl_scan(cnt);
                    deg_extract8(v, w0, carry + incl - cnt, lists + (int64_t)i * LIST_MAX);
                    carry += __shfl_sync(FULL, incl, 31);
                }
            }
            finish_row(i, deg, ucnt);
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
    int thr = max(ws.heavy_min_deg, (st->deg_max + 2) / 3);
    int cnt = 0;
    for (int it = 0; it < 64; ++it) {
        if (t == 0) s_cnt = 0;
        __syncthreads();
        int c = 0;
        for (int i = t; i < n; i += 1024) c += deg[i] >= thr;
        c = __reduce_add_sync(FULL, (unsigned)c);
        if (lane == 0 && c) atomicAdd(&s_cnt, c);
        __syncthreads();
        cnt = s_cnt;
        __syncthreads();
        if (cnt <= ws.heavy_cap) break;
        thr += max(1, thr / 4);
    }
    // widen H to every non-sparse row (degree > LIST_MAX) when that costs no extra 256-row block of the
    // tensor-core contraction: those rows' dense-dense edges then come from the tensor cores instead of the
    // latency-bound popcount path
    {
        const int thr2 = max(ws.heavy_min_deg, LIST_MAX + 1);
        if (thr2 < thr) {
            if (t == 0) s_cnt = 0;
            __syncthreads();
            int c = 0;
            for (int i = t; i < n; i += 1024) c += deg[i] >= thr2;
            c = __reduce_add_sync(FULL, (unsigned)c);
            if (lane == 0 && c) atomicAdd(&s_cnt, c);
            __syncthreads();
            const int cnt2 = s_cnt;
            __syncthreads();
            if (cnt2 <= ws.heavy_cap && (cnt2 + 255) / 256 <= (cnt + 255) / 256) { thr = thr2; cnt = cnt2; }
        }
    }
    const bool use = ws.sc2_path != 1 && cnt >= ws.heavy_min_rows && cnt <= ws.heavy_cap;
    if (t == 0) { s_carry = 0; st->heavy_h = use ? cnt : 0; st->heavy_thr = thr; }
    __syncthreads();
    for (int r0 = 0; r0 < n; r0 += 1024) {
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
        if (f) ws.heavy_list[p * ws.heavy_cap + pos] = i;
        const unsigned fb = __ballot_sync(FULL, f);
        if (lane == 0) {
            const int wi = (r0 + warp * 32) >> 5;
            if (wi < d.W) ws.heavy_mask[p * (ws.bits_stride / ws.row_stride) + wi] = fb;
        }
        __syncthreads();
        if (t == 1023) s_carry = pos + f;
        __syncthreads();
    }
}

// X[a][k] = C[H_a][k] as uint8 0/1 over all columns (rows a in [|H|, round_up(|H|, 256)) are zero), and
// for a < |H| the upper words of row H_a with their exclusive prefix popcounts (UP), from which the
// tensor-core epilogue reads the O2 test and the edge-list rank of every (H_a, H_b).  One warp per X row.
__global__ void __launch_bounds__(256) k_expand(WS ws) {
    const int p = blockIdx.y;
    const PairDesc d = ws.desc[p];
    if (d.n == 0) return;
    const int h = ws.st[p].heavy_h;
    if (h == 0) return;
    const int hp = (h + 255) / 256 * 256;
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a >= hp) return;
    const int W = d.W;
    const int ia = (a < h) ? ws.heavy_list[p * ws.heavy_cap + a] : -1;
    const uint32_t* row = (a < h) ? ws.bits + p * ws.bits_stride + (int64_t)ia * W : nullptr;
    uint8_t* X = ws.heavy_X + p * ws.heavy_X_stride + (int64_t)a * ws.heavy_Kcap;
    uint2* up = ws.heavy_UP + p * ws.heavy_UP_stride + (int64_t)a * W;
    int carry = 0;
    for (int w0 = 0; w0 < W; w0 += 32) {  // 32 bytes per bit word (two 16-byte stores)
        const int w = w0 + lane;
        const uint32_t v = (row && w < W) ? row[w] : 0u;
        if (w < W) {
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
        if (row) {
            const uint32_t u = (w < W) ? upper_mask(v, w, ia) : 0u;
            const int cnt = __popc(u);
            const int incl = warp_incl_scan(cnt);
            if (w < W) up[w] = make_uint2(u, (uint32_t)(carry + incl - cnt));
            carry += __shfl_sync(FULL, incl, 31);
        }
    }
}


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
    const int32_t* rp = ws.rowptr + p * ws.rp_stride;
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
            const int e = e0 + k;
            int lo = 0, hi = n;  // row of edge e: rp[lo] <= e < rp[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(rp + mid) <= e) lo = mid; else hi = mid;
            }
            const int slot = base++;
            if (slot < PIV_CAP)
                cand[slot] = ((unsigned long long)(0x7fff - (int)(v[k] & 0xffffu)) << 30) |
                             ((unsigned long long)lo << 15) | (v[k] >> 16);
        }
    }
}

// One block per pair: bitonic sort of the candidates, the first min(K1, #candidates) become the pivots.
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
    int m2 = 1;
    while (m2 < m) m2 <<= 1;
    const unsigned long long* cand = ws.cand + (int64_t)p * PIV_CAP;
    for (int k = threadIdx.x; k < m2; k += blockDim.x) s_key[k] = (k < m) ? cand[k] : ~0ull;
    __syncthreads();
    for (int size = 2; size <= m2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = threadIdx.x; k < m2 / 2; k += blockDim.x) {
                const int lo = 2 * k - (k & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s_key[lo], b = s_key[hi];
                if ((a > b) == up) { s_key[lo] = b; s_key[hi] = a; }
            }
            __syncthreads();
        }
    }
    const int P = min(ws.k1, m);
    int4* piv = ws.piv + p * ws.piv_stride;
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        const unsigned long long key = s_key[k];
        piv[k] = make_int4((int)((key >> 15) & 0x7fff), (int)(key & 0x7fff), 0x7fff - (int)(key >> 30), 0);
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

// ------------------------------------------------------------------------------------------ a5 PGS
// Alg. 1 L5-13, Eqs. 5-7.  One warp per pivot (i, j): the O2 common neighbours are
// M = U_i ∧ U_j (z > j > i; for a pivot C_ij = 1, so Ĝ_iz > 0 ⇔ C_iz, reading r10), scanned word-parallel;
// Ĝ_iz and Ĝ_jz are gathered from the rank-indexed edge lists (rank = prefix popcount of U_i / U_j below
// z, from a warp scan).  S = Ĝ_ij + Ĝ_iz + Ĝ_jz; the top-K2 by (S desc, z asc) are kept (readings r7, r8):
// per-lane register lists (K2 <= KL) merged by K2 warp argmax rounds, or K2 threshold rounds otherwise.
constexpr int PGS_WARPS = 8;
constexpr int PGS_KL = 8;

template <typename F>
__device__ __forceinline__ void pgs_scan_candidates(const uint32_t* ri, const uint32_t* rj, int W, int i, int j,
                                                    const uint32_t* ei, const uint32_t* ej, int wij, F&& f) {
    const int lane = threadIdx.x & 31;
    int carry_i = 0, carry_j = 0;
    const int nchunks = (W + 31) >> 5;
    for (int c = (i + 1) >> 10; c < nchunks; ++c) {  // chunks holding no bit > i contribute nothing
        const int w = c * 32 + lane;
        const uint32_t ui = (w < W) ? upper_mask(ri[w], w, i) : 0u;
        const uint32_t uj = (w < W) ? upper_mask(rj[w], w, j) : 0u;
        const int pi = __popc(ui), pj = __popc(uj);
        const int si = warp_incl_scan(pi), sj = warp_incl_scan(pj);
        const int exi = carry_i + si - pi, exj = carry_j + sj - pj;
        carry_i += __shfl_sync(FULL, si, 31);
        carry_j += __shfl_sync(FULL, sj, 31);
        uint32_t m = ui & uj;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1u;
            const uint32_t below = (1u << b) - 1u;
            const int rk_i = exi + __popc(ui & below);
            const int rk_j = exj + __popc(uj & below);
            const int wiz = (int)(__ldg(ei + rk_i) & 0xffffu);
            const int wjz = (int)(__ldg(ej + rk_j) & 0xffffu);
            const int z = w * 32 + b;
            const int S = wij + wiz + wjz;
            f(((unsigned long long)(unsigned)S << 32) | (unsigned long long)(0xffffffffu - (unsigned)z));
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
            const int S = wij + (int)wiz + (int)wjz;
            f(((unsigned long long)(unsigned)S << 32) | (unsigned long long)(0xffffffffu - (unsigned)z));
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
                                             int j, const uint32_t* ei, const uint32_t* ej, int wij, int K2, int4* out) {
    const int lane = threadIdx.x & 31;
    unsigned long long top[KL];
#pragma unroll
    for (int r = 0; r < KL; ++r) top[r] = 0ull;
    auto insert = [&](unsigned long long key) {
        if (key > top[KL - 1]) {  // sorted insertion, descending
            unsigned long long k = key;
#pragma unroll
            for (int r = 0; r < KL; ++r) {
                if (k > top[r]) { unsigned long long tmp = top[r]; top[r] = k; k = tmp; }
            }
        }
    };
    if constexpr (MODE == 1) pgs_scan_candidates_sc2(ws, q, ri, rj, W, i, j, ei, ej, wij, insert);
    else pgs_scan_candidates(ri, rj, W, i, j, ei, ej, wij, insert);
    int emitted = 0;
    for (int r = 0; r < K2; ++r) {
        const unsigned long long head = top[0];
        const unsigned long long best = warp_max_u64(head);
        if (best == 0ull) break;
        if (head == best) {  // keys are unique (distinct z), exactly one lane pops
#pragma unroll
            for (int s2 = 0; s2 < KL - 1; ++s2) top[s2] = top[s2 + 1];
            top[KL - 1] = 0ull;
        }
        if (lane == 0) {
            const int z = (int)(0xffffffffu - (unsigned)(best & 0xffffffffull));
            out[r] = sorted_clique(i, j, z, (int)(best >> 32));
        }
        ++emitted;
    }
    return emitted;
}

template <int MODE>
__global__ void __launch_bounds__(PGS_WARPS * 32) k_pgs(WS ws) {
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
    const int P = ws.st[q].npiv;
    if (pv >= P) {
        for (int r = lane; r < K2; r += 32) out[r] = make_int4(-1, -1, -1, 0);
        return;
    }
    const int4 pvt = ws.piv[q * ws.piv_stride + pv];
    const int i = pvt.x, j = pvt.y, wij = pvt.z;
    const uint32_t* bits = ws.bits + q * ws.bits_stride;
    const uint32_t* ri = bits + (int64_t)i * W;
    const uint32_t* rj = bits + (int64_t)j * W;
    const uint32_t* edges = ws.edges + q * ws.edges_stride;
    const uint32_t* ei = edges + ws.rowptr[q * ws.rp_stride + i];
    const uint32_t* ej = edges + ws.rowptr[q * ws.rp_stride + j];
    int emitted = 0;
    if (K2 <= 2) {
        emitted = pgs_topk_list<2, MODE>(ws, q, ri, rj, W, i, j, ei, ej, wij, K2, out);
    } else if (K2 <= 4) {
        emitted = pgs_topk_list<4, MODE>(ws, q, ri, rj, W, i, j, ei, ej, wij, K2, out);
    } else if (K2 <= PGS_KL) {
        emitted = pgs_topk_list<PGS_KL, MODE>(ws, q, ri, rj, W, i, j, ei, ej, wij, K2, out);
    } else {
        unsigned long long thr = ~0ull;
        for (int r = 0; r < K2; ++r) {
            unsigned long long mine = 0ull;
            auto take = [&](unsigned long long key) {
                if (key < thr && key > mine) mine = key;
            };
            if constexpr (MODE == 1) pgs_scan_candidates_sc2(ws, q, ri, rj, W, i, j, ei, ej, wij, take);
            else pgs_scan_candidates(ri, rj, W, i, j, ei, ej, wij, take);
            const unsigned long long best = warp_max_u64(mine);
            if (best == 0ull) break;
            if (lane == 0) {
                const int z = (int)(0xffffffffu - (unsigned)(best & 0xffffffffull));
                out[r] = sorted_clique(i, j, z, (int)(best >> 32));
            }
            thr = best;
            ++emitted;
        }
    }
    for (int r = emitted + lane; r < K2; r += 32) out[r] = make_int4(-1, -1, -1, 0);
}

// ------------------------------------------------------------------------------------------ a6 Kabsch
// P:283.  One thread per TurboClique slot, FP64.  Degenerate predicate (reading r11) in the oracle's
// exact expression tree; then a closed form of the least-squares fit: three points are coplanar, so H
// has σ3 = 0 and the optimal rotation maps the source plane onto the target plane.  With orthonormal
// in-plane bases (e1, e2, n_x), (f1, f2, n_y) and the 2×2 cross-covariance M of the in-plane coordinates,
// the optimum is the better of the rotation family (c, s) ∝ (M00 + M11, M01 - M10) and the reflection
// family (c, s) ∝ (M00 - M11, M01 + M10), the normal mapped with sign det(Q) so det R = +1.
__device__ __forceinline__ bool tri_degenerate(double p0x, double p0y, double p0z, double p1x, double p1y,
                                               double p1z, double p2x, double p2y, double p2z) {
    const double ax = __dsub_rn(p1x, p0x), ay = __dsub_rn(p1y, p0y), az = __dsub_rn(p1z, p0z);
    const double bx = __dsub_rn(p2x, p0x), by = __dsub_rn(p2y, p0y), bz = __dsub_rn(p2z, p0z);
    const double cx = __dsub_rn(__dmul_rn(ay, bz), __dmul_rn(az, by));
    const double cy = __dsub_rn(__dmul_rn(az, bx), __dmul_rn(ax, bz));
    const double cz = __dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx));
    const double c2 = __dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz));
    const double a2 = __dadd_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)), __dmul_rn(az, az));
    const double b2 = __dadd_rn(__dadd_rn(__dmul_rn(bx, bx), __dmul_rn(by, by)), __dmul_rn(bz, bz));
    return c2 <= __dmul_rn(1e-12, __dmul_rn(a2, b2));
}

struct d3 { double x, y, z; };
__device__ __forceinline__ d3 mk(const float4& v) { return {(double)v.x, (double)v.y, (double)v.z}; }
__device__ __forceinline__ d3 sub(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 cross(d3 a, d3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
__device__ __forceinline__ d3 scale(d3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ d3 unit(d3 a) { return scale(a, rsqrt(dot(a, a))); }

// Returns false if the fit is degenerate (σ2 <= 1e-12 σ1 of the in-plane covariance, as the oracle's SVD).
__device__ bool kabsch3(const float4& x0f, const float4& x1f, const float4& x2f, const float4& y0f, const float4& y1f,
                        const float4& y2f, double R[9], double t[3]) {
    const d3 x0 = mk(x0f), x1 = mk(x1f), x2 = mk(x2f), y0 = mk(y0f), y1 = mk(y1f), y2 = mk(y2f);
    const d3 cx = {(x0.x + x1.x + x2.x) / 3.0, (x0.y + x1.y + x2.y) / 3.0, (x0.z + x1.z + x2.z) / 3.0};
    const d3 cy = {(y0.x + y1.x + y2.x) / 3.0, (y0.y + y1.y + y2.y) / 3.0, (y0.z + y1.z + y2.z) / 3.0};
    const d3 nx = unit(cross(sub(x1, x0), sub(x2, x0)));
    const d3 e1 = unit(sub(x1, x0));
    const d3 e2 = cross(nx, e1);
    const d3 ny = unit(cross(sub(y1, y0), sub(y2, y0)));
    const d3 f1 = unit(sub(y1, y0));
    const d3 f2 = cross(ny, f1);
    const d3 a[3] = {sub(x0, cx), sub(x1, cx), sub(x2, cx)};
    const d3 b[3] = {sub(y0, cy), sub(y1, cy), sub(y2, cy)};
    double M00 = 0, M01 = 0, M10 = 0, M11 = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double A0 = dot(a[k], e1), A1 = dot(a[k], e2);
        const double B0 = dot(b[k], f1), B1 = dot(b[k], f2);
        M00 += A0 * B0; M01 += A0 * B1; M10 += A1 * B0; M11 += A1 * B1;
    }
    const double pr = M00 + M11, qr = M01 - M10, pf = M00 - M11, qf = M01 + M10;
    const double vr = sqrt(pr * pr + qr * qr), vf = sqrt(pf * pf + qf * qf);
    const double s1 = 0.5 * (vr + vf), s2 = 0.5 * fabs(vr - vf);
    if (!(s1 > 0.0) || s2 <= 1e-12 * s1) return false;
    double Q00, Q01, Q10, Q11, dsign;
    if (vr >= vf) {
        const double c = pr / vr, s = qr / vr;
        Q00 = c; Q01 = -s; Q10 = s; Q11 = c; dsign = 1.0;
    } else {
        const double c = pf / vf, s = qf / vf;
        Q00 = c; Q01 = s; Q10 = s; Q11 = -c; dsign = -1.0;
    }
    // R = F Q E^T + det(Q) n_y n_x^T, F = [f1 f2], E = [e1 e2]
    const double F[3][2] = {{f1.x, f2.x}, {f1.y, f2.y}, {f1.z, f2.z}};
    const double E[3][2] = {{e1.x, e2.x}, {e1.y, e2.y}, {e1.z, e2.z}};
    const double NY[3] = {ny.x, ny.y, ny.z}, NX[3] = {nx.x, nx.y, nx.z};
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const double g0 = F[r][0] * Q00 + F[r][1] * Q10;
        const double g1 = F[r][0] * Q01 + F[r][1] * Q11;
#pragma unroll
        for (int c = 0; c < 3; ++c) R[3 * r + c] = g0 * E[c][0] + g1 * E[c][1] + dsign * NY[r] * NX[c];
    }
    t[0] = cy.x - (R[0] * cx.x + R[1] * cx.y + R[2] * cx.z);
    t[1] = cy.y - (R[3] * cx.x + R[4] * cx.y + R[5] * cx.z);
    t[2] = cy.z - (R[6] * cx.x + R[7] * cx.y + R[8] * cx.z);
    return true;
}

// SC^2 mode only (reading r9): the K1·K2 clique slots of a pair in canonical order (S desc, (i,j,z) asc)
// with duplicate triples (found from several pivots) dropped, compacted to the front; the rest invalid.
// One block per pair, bitonic sort of 64-bit keys ((2^18-1-S) << 45 | i << 30 | j << 15 | z) in shared
// memory (K1·K2 <= CANON_CAP).
constexpr int CANON_CAP = 16384;
__global__ void __launch_bounds__(1024) k_canon(WS ws) {
    extern __shared__ unsigned long long s_key[];
    __shared__ int s_warp[32];
    const int q = blockIdx.x;
    if (ws.desc[q].n == 0) return;
    const int K = ws.k1 * ws.k2;
    int4* cl = ws.cliq + q * ws.cl_stride;
    int m2 = 1;
    while (m2 < K) m2 <<= 1;
    for (int k = threadIdx.x; k < m2; k += blockDim.x) {
        unsigned long long key = ~0ull;
        if (k < K) {
            const int4 c = cl[k];
            if (c.x >= 0)
                key = ((unsigned long long)(0x3ffff - c.w) << 45) | ((unsigned long long)c.x << 30) |
                      ((unsigned long long)c.y << 15) | (unsigned long long)c.z;
        }
        s_key[k] = key;
    }
    __syncthreads();
    for (int size = 2; size <= m2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int k = threadIdx.x; k < m2 / 2; k += blockDim.x) {
                const int lo = 2 * k - (k & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s_key[lo], b = s_key[hi];
                if ((a > b) == up) { s_key[lo] = b; s_key[hi] = a; }
            }
            __syncthreads();
        }
    }
    // keep the first of each run of equal triples (equal triples have equal S: S is the triangle's weight)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int base = 0;
    for (int k0 = 0; k0 < K; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        const unsigned long long key = (k < K) ? s_key[k] : ~0ull;
        const bool keep = key != ~0ull && (k == 0 || s_key[k - 1] != key);
        const unsigned b = __ballot_sync(FULL, keep);
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { before += (w < warp) ? s_warp[w] : 0; total += s_warp[w]; }
        __syncthreads();
        if (keep) {
            const int slot = base + before + __popc(b & ((1u << lane) - 1u));
            cl[slot] = make_int4((int)((key >> 30) & 0x7fff), (int)((key >> 15) & 0x7fff), (int)(key & 0x7fff),
                                 0x3ffff - (int)(key >> 45));
        }
        base += total;
    }
    __syncthreads();
    for (int k = base + threadIdx.x; k < K; k += blockDim.x) cl[k] = make_int4(-1, -1, -1, 0);
}

__global__ void __launch_bounds__(128) k_kabsch(WS ws) {
    const int q = blockIdx.y;
    const PairDesc d = ws.desc[q];
    if (d.n == 0) return;
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int K = ws.k1 * ws.k2;
    if (s >= K) return;
    const int4 c = ws.cliq[q * ws.cl_stride + s];
    float* h = ws.hyp + (q * ws.cl_stride + s) * 16;
    float out[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) out[k] = 0.f;
    int flag = 2;
    if (c.x >= 0) {
        const float4* s4 = ws.src4 + q * ws.pts_stride;
        const float4* d4 = ws.dst4 + q * ws.pts_stride;
        const float4 x0 = s4[c.x], x1 = s4[c.y], x2 = s4[c.z];
        const float4 y0 = d4[c.x], y1 = d4[c.y], y2 = d4[c.z];
        flag = 1;
        if (!tri_degenerate(x0.x, x0.y, x0.z, x1.x, x1.y, x1.z, x2.x, x2.y, x2.z) &&
            !tri_degenerate(y0.x, y0.y, y0.z, y1.x, y1.y, y1.z, y2.x, y2.y, y2.z)) {
            double R[9], t[3];
            if (kabsch3(x0, x1, x2, y0, y1, y2, R, t)) {
                flag = 0;
#pragma unroll
                for (int k = 0; k < 9; ++k) out[k] = __double2float_rn(R[k]);
#pragma unroll
                for (int k = 0; k < 3; ++k) out[9 + k] = __double2float_rn(t[k]);
            }
        }
    }
    out[13] = __int_as_float(flag);
    out[14] = __int_as_float(c.w);
    float4* h4 = reinterpret_cast<float4*>(h);
#pragma unroll
    for (int k = 0; k < 4; ++k) h4[k] = make_float4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
}

// ------------------------------------------------------------------------------------------ a7 scoring
// g(T) = inlier number.  Block = 128 hypotheses × a chunk of SCORE_PC correspondences that
// one thread stages into shared memory with two bulk async copies (cp.async.bulk, the TMA engine)
// completing on an mbarrier; every thread then streams the chunk (broadcast LDS.128) through its own
// (R, t) in the oracle's fixed fp32 FMA tree (reading r13) and adds its count atomically.
constexpr int SCORE_THREADS = 128;               // each thread scores two hypotheses
constexpr int SCORE_HT = 2 * SCORE_THREADS;      // hypotheses per block (one packed pair per thread)
constexpr int SCORE_PC = 512;                    // correspondences per pipeline stage

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// g(T) = inlier number.  A block owns 256·NP hypotheses of one pair (2·NP per thread, packed
// in pairs as f32x2 lanes: one fma.rn.f32x2 evaluates the same correspondence under two transforms) and one of
// `segs` contiguous segments of the N correspondences (partial counts meet in one atomicAdd per
// hypothesis; the finer grid leaves no half-empty last wave), streamed through a 2-stage shared-memory ring filled by bulk async copies (cp.async.bulk, the TMA
// engine) completing on per-stage mbarriers; the copy of chunk c+1 overlaps the arithmetic on chunk c.
// Each lane is exactly the oracle's float32 FMA tree (reading r13), so counts are bit-identical.
template <bool ERR, int NP>
__global__ void __launch_bounds__(SCORE_THREADS, (NP == 1 ? 8 : 4)) k_score(WS ws, int segs) {
    // NP packed hypothesis pairs per thread: hypotheses h = base + threadIdx.x + SCORE_THREADS * u, u < 2 NP
    constexpr int NH = 2 * NP;
    __shared__ __align__(16) float4 s_src[2][SCORE_PC];
    __shared__ __align__(16) float4 s_dst[2][SCORE_PC];
    __shared__ __align__(8) unsigned long long s_bar[2];
    const int q = blockIdx.y;
    const PairDesc d = ws.desc[q];
    const int n = d.n;
    if (n == 0) return;
    const int K = ws.k1 * ws.k2;
    const int seg = blockIdx.x % segs;
    const int hbase = (blockIdx.x / segs) * (SCORE_THREADS * NH) + threadIdx.x;
    const int pseg = (n + segs - 1) / segs;
    const int pbeg = min(n, seg * pseg), np = min(n, pbeg + pseg) - pbeg;  // this block's points
    float Rh[NH][12];
    bool vh[NH];
    bool any = false;
#pragma unroll
    for (int u = 0; u < NH; ++u) {
        const int h = hbase + SCORE_THREADS * u;
#pragma unroll
        for (int k = 0; k < 12; ++k) Rh[u][k] = 0.f;
        vh[u] = false;
        if (h < K) {
            const float4* h4 = reinterpret_cast<const float4*>(ws.hyp + (q * ws.cl_stride + h) * 16);
            const float4 a = h4[0], b = h4[1], c = h4[2], e = h4[3];
            vh[u] = __float_as_int(e.y) == 0;
            Rh[u][0] = a.x; Rh[u][1] = a.y; Rh[u][2] = a.z; Rh[u][3] = a.w; Rh[u][4] = b.x; Rh[u][5] = b.y;
            Rh[u][6] = b.z; Rh[u][7] = b.w; Rh[u][8] = c.x; Rh[u][9] = c.y; Rh[u][10] = c.z; Rh[u][11] = c.w;
        }
        any |= vh[u];
    }
    if (!__syncthreads_or(any && np > 0)) return;
    const uint32_t bar0 = smem_u32(&s_bar[0]), bar1 = smem_u32(&s_bar[1]);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nchunks = (np + SCORE_PC - 1) / SCORE_PC;
    const float4* gs = ws.src4 + q * ws.pts_stride + pbeg;
    const float4* gd = ws.dst4 + q * ws.pts_stride + pbeg;
    auto issue = [&](int c) {  // thread 0: stage chunk c into buffer c & 1
        const int st = c & 1;
        const int kc = min(SCORE_PC, np - c * SCORE_PC);
        const uint32_t bytes = (uint32_t)kc * 16u;
        const uint32_t bar = st ? bar1 : bar0;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2u * bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(s_src[st])),
                     "l"(gs + c * SCORE_PC), "r"(bytes), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(s_dst[st])),
                     "l"(gd + c * SCORE_PC), "r"(bytes), "r"(bar)
                     : "memory");
    };
    if (threadIdx.x == 0) issue(0);
    const uint32_t thr2b = __float_as_uint(__fmul_rn(ws.thr, ws.thr));
    f2_t Rp[NP][9], tp[NP][3];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
#pragma unroll
        for (int k = 0; k < 9; ++k) Rp[m][k] = f2_pack(Rh[2 * m][k], Rh[2 * m + 1][k]);
#pragma unroll
        for (int k = 0; k < 3; ++k) tp[m][k] = f2_pack(Rh[2 * m][9 + k], Rh[2 * m + 1][9 + k]);
    }
    const f2_t mone = f2_pack(-1.0f, -1.0f);
    int cnt[NH];
    double ea[NH], es[NH];  // ERR: Σ sqrtf(s), Σ s per hypothesis (r20)
#pragma unroll
    for (int u = 0; u < NH; ++u) { cnt[u] = 0; ea[u] = es[u] = 0.0; }
    for (int c = 0; c < nchunks; ++c) {
        const int st = c & 1;
        if (threadIdx.x == 0 && c + 1 < nchunks) issue(c + 1);  // buffer st^1 was released by the barrier below
        {
            const uint32_t bar = st ? bar1 : bar0, parity = (uint32_t)((c >> 1) & 1);
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                    : "=r"(done)
                    : "r"(bar), "r"(parity)
                    : "memory");
            }
        }
        const int kc = min(SCORE_PC, np - c * SCORE_PC);
        const float4* xs = s_src[st];
        const float4* ys = s_dst[st];
#pragma unroll 4
        for (int k = 0; k < kc; ++k) {
            const float4 x = xs[k];
            const float4 y = ys[k];
            const f2_t X = f2_pack(x.x, x.x), Y = f2_pack(x.y, x.y), Z = f2_pack(x.z, x.z);
#pragma unroll
            for (int m = 0; m < NP; ++m) {
                const f2_t p0 = f2_fma(Rp[m][2], Z, f2_fma(Rp[m][1], Y, f2_fma(Rp[m][0], X, tp[m][0])));
                const f2_t p1 = f2_fma(Rp[m][5], Z, f2_fma(Rp[m][4], Y, f2_fma(Rp[m][3], X, tp[m][1])));
                const f2_t p2 = f2_fma(Rp[m][8], Z, f2_fma(Rp[m][7], Y, f2_fma(Rp[m][6], X, tp[m][2])));
                const f2_t e0 = f2_fma(f2_pack(y.x, y.x), mone, p0);  // p − y: exact negation, one rounding
                const f2_t e1 = f2_fma(f2_pack(y.y, y.y), mone, p1);
                const f2_t e2 = f2_fma(f2_pack(y.z, y.z), mone, p2);
                const f2_t sq = f2_fma(e2, e2, f2_fma(e1, e1, f2_mul(e0, e0)));
                // s >= 0, so integer order of the bit patterns is float order
                cnt[2 * m] += f2_lo(sq) <= thr2b;
                cnt[2 * m + 1] += f2_hi(sq) <= thr2b;
                if constexpr (ERR) {
                    const float s0 = __uint_as_float(f2_lo(sq)), s1 = __uint_as_float(f2_hi(sq));
                    ea[2 * m] += (double)__fsqrt_rn(s0);
                    ea[2 * m + 1] += (double)__fsqrt_rn(s1);
                    es[2 * m] += (double)s0;
                    es[2 * m + 1] += (double)s1;
                }
            }
        }
        __syncthreads();  // every thread is done with buffer st before it is refilled
    }
#pragma unroll
    for (int u = 0; u < NH; ++u) {
        const int h = hbase + SCORE_THREADS * u;
        if (!vh[u]) continue;
        if (cnt[u]) atomicAdd(reinterpret_cast<int*>(ws.hyp + (q * ws.cl_stride + h) * 16 + 12), cnt[u]);
        if constexpr (ERR) {
            double2* he = ws.herr + q * ws.cl_stride;
            atomicAdd(&he[h].x, ea[u]);
            atomicAdd(&he[h].y, es[u]);
        }
    }
}

// ------------------------------------------------------------------------------------------ a8 argmax
// Eq. 9 with reading r14: key (count desc, S desc, (i,j,z) asc), as a max over
// (count << 17 | S) and then a min over the packed triple among the maxima.  Writes the result record.
struct DevResult {  // mirrors turboreg_result
    float R[9];
    float t[3];
    int32_t inlier_count;
    int32_t clique[3];
    int32_t clique_weight;
    int32_t num_pivots, num_cliques, hypotheses_evaluated;
    int32_t status;
    float stage_ms[3];
    int64_t num_edges;
};

__global__ void __launch_bounds__(256) k_finalize(WS ws) {
    __shared__ unsigned long long s_red[8];
    __shared__ int s_cnt[2][8];
    const int q = blockIdx.x;
    const PairDesc d = ws.desc[q];
    const PairState* st = ws.st + q;
    DevResult* res = reinterpret_cast<DevResult*>(ws.res) + q;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int K = ws.k1 * ws.k2;
    const float* hyp = ws.hyp + q * ws.cl_stride * 16;
    const int4* cl = ws.cliq + q * ws.cl_stride;
    // key of a valid hypothesis, maximised: inlier mode (count << 17 | S); error modes (reading r20) the
    // complement of the error's bit pattern (non-negative doubles order like their bits) — S and ijz break
    // ties below, as in the oracle's scan of the canonical list
    const int rank = ws.err_mode >> 1;
    const double2* he = ws.herr + q * ws.cl_stride;
    auto key_of = [&](int s, const float* h) -> unsigned long long {
        if (rank == 0)
            return ((unsigned long long)(unsigned)__float_as_int(h[12]) << 17) | (unsigned)__float_as_int(h[14]);
        const double e = rank == 1 ? he[s].x : he[s].y;
        return ~(unsigned long long)__double_as_longlong(e);
    };
    unsigned long long best1 = 0ull;
    int ncl = 0, nev = 0;
    if (d.n > 0) {
        for (int s = t; s < K; s += blockDim.x) {
            const float* h = hyp + (int64_t)s * 16;
            const int flag = __float_as_int(h[13]);
            if (flag != 2) ++ncl;
            if (flag == 0) {
                ++nev;
                const unsigned long long key = key_of(s, h);
                best1 = key > best1 ? key : best1;
            }
        }
    }
    best1 = warp_max_u64(best1);
    ncl = __reduce_add_sync(FULL, (unsigned)ncl);
    nev = __reduce_add_sync(FULL, (unsigned)nev);
    if (lane == 0) { s_red[warp] = best1; s_cnt[0][warp] = ncl; s_cnt[1][warp] = nev; }
    __syncthreads();
    if (t == 0) {
        unsigned long long b = 0ull;
        int a = 0, e = 0;
        for (int w = 0; w < 8; ++w) { b = s_red[w] > b ? s_red[w] : b; a += s_cnt[0][w]; e += s_cnt[1][w]; }
        s_red[0] = b; s_cnt[0][0] = a; s_cnt[1][0] = e;
    }
    __syncthreads();
    best1 = s_red[0];
    ncl = s_cnt[0][0];
    nev = s_cnt[1][0];
    __syncthreads();
    int bestS = -1;  // error modes: the largest S among the minimum-error hypotheses
    if (rank != 0) {
        int ms = -1;
        if (d.n > 0 && nev > 0)
            for (int s = t; s < K; s += blockDim.x) {
                const float* h = hyp + (int64_t)s * 16;
                if (__float_as_int(h[13]) == 0 && key_of(s, h) == best1) ms = max(ms, __float_as_int(h[14]));
            }
        ms = (int)__reduce_max_sync(FULL, (unsigned)(ms + 1)) - 1;
        if (lane == 0) s_cnt[0][warp] = ms;
        __syncthreads();
        if (t == 0) {
            int m = -1;
            for (int w = 0; w < 8; ++w) m = max(m, s_cnt[0][w]);
            s_cnt[0][0] = m;
        }
        __syncthreads();
        bestS = s_cnt[0][0];
        __syncthreads();
    }
    unsigned long long bestt = ~0ull;
    if (d.n > 0 && nev > 0) {
        for (int s = t; s < K; s += blockDim.x) {
            const float* h = hyp + (int64_t)s * 16;
            if (__float_as_int(h[13]) != 0) continue;
            const unsigned long long key = key_of(s, h);
            if (key != best1) continue;
            if (rank != 0 && __float_as_int(h[14]) != bestS) continue;
            const int4 c = cl[s];
            const unsigned long long tk = ((unsigned long long)c.x << 30) | ((unsigned long long)c.y << 15) | c.z;
            if (tk < bestt) bestt = tk;
        }
    }
    bestt = warp_min_u64(bestt);
    __shared__ int s_slot;
    if (lane == 0) s_red[warp] = bestt;
    if (t == 0) s_slot = 0x7fffffff;
    __syncthreads();
    if (t == 0) {
        unsigned long long b = ~0ull;
        for (int w = 0; w < 8; ++w) b = s_red[w] < b ? s_red[w] : b;
        s_red[0] = b;
    }
    __syncthreads();
    bestt = s_red[0];
    if (bestt != ~0ull) {  // the slot holding the winning triple (duplicates carry identical values)
        for (int s = t; s < K; s += blockDim.x) {
            if (__float_as_int(hyp[(int64_t)s * 16 + 13]) != 0) continue;
            if (key_of(s, hyp + (int64_t)s * 16) != best1) continue;
            const int4 c = cl[s];
            const unsigned long long tk = ((unsigned long long)c.x << 30) | ((unsigned long long)c.y << 15) | c.z;
            if (tk == bestt) atomicMin(&s_slot, s);
        }
    }
    __syncthreads();
    if (t == 0) {
        const int bests = (bestt == ~0ull) ? -1 : s_slot;
        int status = d.host_status;
        if (status == 0 && st->nonfinite) status = 4;
        if (status == 0 && bests < 0) status = 5;
        DevResult r;
        for (int k = 0; k < 9; ++k) r.R[k] = 0.f;
        for (int k = 0; k < 3; ++k) r.t[k] = 0.f;
        r.inlier_count = 0;
        r.clique[0] = r.clique[1] = r.clique[2] = -1;
        r.clique_weight = 0;
        r.num_pivots = (d.n > 0) ? st->npiv : 0;
        r.num_cliques = (d.n > 0) ? ncl : 0;
        r.hypotheses_evaluated = (d.n > 0) ? nev : 0;
        r.status = status;
        r.stage_ms[0] = r.stage_ms[1] = r.stage_ms[2] = 0.f;
        r.num_edges = (d.n > 0) ? st->edges : 0;
        if (status == 0) {
            const float* h = hyp + (int64_t)bests * 16;
            for (int k = 0; k < 9; ++k) r.R[k] = h[k];
            for (int k = 0; k < 3; ++k) r.t[k] = h[9 + k];
            r.inlier_count = __float_as_int(h[12]);
            const int4 c = cl[bests];
            r.clique[0] = c.x; r.clique[1] = c.y; r.clique[2] = c.z;
            r.clique_weight = c.w;
        }
        *res = r;
    }
}

}  // namespace trk
