// a1 ingest and a2 compatibility graph (Eq. 1).  Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_common.cuh"

namespace trk {

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
    const float k = __double2float_ru((double)t2 + ldexp(smax * (1.0 + 0x1p-20), -21));
    return k >= 0x1p-100f ? k : __int_as_float(0x7f800000);  // absurdly small τ: κ = +inf, every test exact
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
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
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

// The same transpose in 13 instructions: the two byte-level stages are one PRMT each (a per-lane byte
// selector), the three bit-level stages a funnel rotate by a per-lane amount and one bitwise select
// (per-lane keep mask) — every stage free of predicated pairs.  The lane constants are built once per work
// item (Transpose32 below) and shared by its tiles.
struct Transpose32 {
    uint32_t sel16, sel8, keep4, keep2, keep1, rot4, rot2, rot1;
    __device__ __forceinline__ Transpose32() {
        const int lane = threadIdx.x & 31;
        sel16 = (lane & 16) ? 0x3276u : 0x5410u;  // hi lanes: (x & 0xffff0000) | (y >> 16); lo: (x & 0xffff) | (y << 16)
        sel8 = (lane & 8) ? 0x3715u : 0x6240u;
        keep4 = (lane & 4) ? 0xf0f0f0f0u : 0x0f0f0f0fu;
        keep2 = (lane & 2) ? 0xccccccccu : 0x33333333u;
        keep1 = (lane & 1) ? 0xaaaaaaaau : 0x55555555u;
        rot4 = (lane & 4) ? 28u : 4u;
        rot2 = (lane & 2) ? 30u : 2u;
        rot1 = (lane & 1) ? 31u : 1u;
    }
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
        x = __byte_perm(x, __shfl_xor_sync(FULL, x, 16), sel16);
        x = __byte_perm(x, __shfl_xor_sync(FULL, x, 8), sel8);
        uint32_t y = __shfl_xor_sync(FULL, x, 4);
        x = (x & keep4) | (__funnelshift_l(y, y, rot4) & ~keep4);
        y = __shfl_xor_sync(FULL, x, 2);
        x = (x & keep2) | (__funnelshift_l(y, y, rot2) & ~keep2);
        y = __shfl_xor_sync(FULL, x, 1);
        x = (x & keep1) | (__funnelshift_l(y, y, rot1) & ~keep1);
        return x;
    }
};

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
    // −2^-19 (|D| + κ) in one rounding: fma(|D|, −2^-19, −2^-19 κ) = −2^-19 fl(|D| + κ) exactly (power-of-two
    // scaling; κ ≥ 2^-100 keeps it normal, see compat_kappa), so b below is bit-identical to
    // fma(fl(|D| + κ), −2^-19 S, |q|) of DESIGN §6.1 with one operation fewer
    const f2_t nkap19 = f2_pack(-0x1p-19f * kap, -0x1p-19f * kap);
    // per test, in bit 31:  cc: S > s_hi (q decides);  b: |q| < Tq (q unsure);  q: q < 0.
    // decided = ~b & cc (bit 31);  edge = sign(q);  sacc keeps bit 31 while all decided.
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
            // |q| − Tq with one rounding: the sign is exactly that of |q| − fl(|D| + κ)·S·2^-19
            const f2_t b = f2_fma(f2_fma(absD, nc19, nkap19), S, q & 0x7fffffff7fffffffull);
            const f2_t cc = f2_fma(S, mone, s_hi2);
            const uint32_t k0 = f2_lo(cc), k1 = f2_hi(cc);
            // edge bit = sign(q): only read when every test of the lane is decided (else the lane redoes all)
            colw[2 * m] = __funnelshift_l(f2_lo(q), colw[2 * m], 1);
            colw[2 * m + 1] = __funnelshift_l(f2_hi(q), colw[2 * m + 1], 1);
            sacc &= ~f2_lo(b) & k0;
            sacc &= ~f2_hi(b) & k1;
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
// DIAG: tile k = 0 is the diagonal tile (J == I).  Its self tests (row r = lane) have S = 0, which the
// filter cannot certify (S <= τ²(1 + 2^-16)); they are excluded from the decided mask (C_ii = 0 is masked
// off below anyway), so a diagonal item no longer sends every lane through the exact tree.
template <int NC, int UNR, bool DIAG = false>
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
    // −2^-19 (|D| + κ) in one rounding: fma(|D|, −2^-19, −2^-19 κ) = −2^-19 fl(|D| + κ) exactly (power-of-two
    // scaling; κ ≥ 2^-100 keeps it normal, see compat_kappa), so b below is bit-identical to
    // fma(fl(|D| + κ), −2^-19 S, |q|) of DESIGN §6.1 with one operation fewer
    const f2_t nkap19 = f2_pack(-0x1p-19f * kap, -0x1p-19f * kap);
    uint32_t colw[NC], sacc = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < NC; ++k) colw[k] = 0u;
    const uint32_t selfw = DIAG ? (1u << lane) : 0u;  // the lane's own row (DIAG)
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
            // |q| − Tq with one rounding: the sign is exactly that of |q| − fl(|D| + κ)·S·2^-19
            const f2_t b = f2_fma(f2_fma(absD, nc19, nkap19), S, q & 0x7fffffff7fffffffull);
            const f2_t cc = f2_fma(S, mone, s_hi2);
            uint32_t k0 = f2_lo(cc), k1 = f2_hi(cc);
            if (DIAG && k == 0) {  // rows 2kk, 2kk+1 of the diagonal tile: the self test is not a test
                k0 |= (selfw << (31 - 2 * kk)) & 0x80000000u;
                k1 |= (selfw << (30 - 2 * kk)) & 0x80000000u;
            }
            // edge bit = sign(q): only read when every test of the lane is decided (else the lane redoes all)
            colw[k] = __funnelshift_l(f2_lo(q), colw[k], 1);
            colw[k] = __funnelshift_l(f2_hi(q), colw[k], 1);
            sacc &= ~f2_lo(b) & k0;
            sacc &= ~f2_hi(b) & k1;
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
    const Transpose32 tp32;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const int c = (J + k) * 32 + lane;
        const bool cv = c < n;
        uint32_t okc = cv ? rmask : 0u;
        const uint32_t cvb = __ballot_sync(FULL, cv);  // every lane votes (never inside a conditional)
        uint32_t okr = rv ? cvb : 0u;
        if (I == J + k) { okc &= ~(1u << lane); okr &= ~(1u << lane); }
        const uint32_t cw = colw[k] & okc;
        const uint32_t rw = tp32(cw) & okr;
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
    const int b = ws.compat_b0 + blockIdx.x / split, sp = blockIdx.x % split;
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
            // per block-row: item 0 is the diagonal tile alone (its self tests are excluded from the filter's
            // decided mask, DIAG), then the tiles right of it NC at a time
            const int P0 = 1 + (T - I0 - 1 + NC - 1) / NC, P1 = (I1 != I0) ? 1 + (T - I1 - 1 + NC - 1) / NC : 0;
            for (int t = warp + 8 * sp; t < P0 + P1; t += 8 * split) {
                const bool second = t >= P0;
                const int u = second ? t - P0 : t;
                const int I = second ? I1 : I0, o = second ? 32 : 0, h = second;
                if (u == 0)
                    compat_tiles_rp<1, UNR, true>(ws, p, n, W, T, I, I, s_rs + o, s_rd + o, s_pxy[h], s_pz[h],
                                                  s_qxy[h], s_qz[h], kap);
                else
                    compat_tiles_rp<NC, UNR>(ws, p, n, W, T, I, I + 1 + NC * (u - 1), s_rs + o, s_rd + o, s_pxy[h],
                                             s_pz[h], s_qxy[h], s_qz[h], kap);
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

}  // namespace trk
