// a6 Kabsch, a7 hypothesis scoring, a8 argmax (Eq. 9).  Part of turboreg_kernels.cuh.
#pragma once
#include "turboreg_pgs.cuh"

namespace trk {

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

// ------------------------------------------------------------------------------------------ NEXT(3)
// Point-cloud resolution pr for the τ initialisation τ = 0.25·pr: nn[i] = distance from
// point i to its nearest other point in the float32 tree of reading r1 (the minimum is taken on the squared
// distance — correctly rounded sqrt is monotone, so sqrt(min) = min(sqrt) and sqrt(k-th) = k-th(sqrt)), then
// the lower median (reading r22) by a 4-pass radix select on the (non-negative) float bit patterns.
constexpr int NN_TILE = 1024;
// grid (point blocks, j splits): split y scans candidates [y·span, (y+1)·span) and folds its minimum squared
// distance into nn2[i] (float bits; non-negative floats order like their bit patterns, so an integer
// atomicMin is the float minimum).  nn2 must start at +inf.
__global__ void __launch_bounds__(256) k_nn_dist(const float* xyz, int n, int span, int* nn2, int* nonfinite) {
    __shared__ float4 s_p[NN_TILE];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float xi = 0.f, yi = 0.f, zi = 0.f;
    if (i < n) {
        xi = xyz[3 * (int64_t)i];
        yi = xyz[3 * (int64_t)i + 1];
        zi = xyz[3 * (int64_t)i + 2];
        if (blockIdx.y == 0 && (!isfinite(xi) || !isfinite(yi) || !isfinite(zi))) atomicOr(nonfinite, 1);
    }
    float best = __int_as_float(0x7f800000);  // +inf
    const int jb = blockIdx.y * span, je = min(n, jb + span);
    for (int j0 = jb; j0 < je; j0 += NN_TILE) {
        __syncthreads();
        for (int t = threadIdx.x; t < NN_TILE; t += blockDim.x) {
            const int j = j0 + t;
            s_p[t] = j < je ? make_float4(xyz[3 * (int64_t)j], xyz[3 * (int64_t)j + 1], xyz[3 * (int64_t)j + 2], 0.f)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        const int m = min(NN_TILE, je - j0);
        // two candidates per f32x2 op (each lane half is the same IEEE op as the scalar tree); the point's own
        // slot is masked after the arithmetic
        const f2_t X = f2_pack(xi, xi), Y = f2_pack(yi, yi), Z = f2_pack(zi, zi);
        const int self = i - j0;
        int t = 0;
#pragma unroll 8
        for (; t + 1 < m; t += 2) {
            const float4 qa = s_p[t], qb = s_p[t + 1];
            const f2_t dx = f2_sub(X, f2_pack(qa.x, qb.x)), dy = f2_sub(Y, f2_pack(qa.y, qb.y)),
                       dz = f2_sub(Z, f2_pack(qa.z, qb.z));
            const f2_t d2 = f2_add(f2_add(f2_mul(dx, dx), f2_mul(dy, dy)), f2_mul(dz, dz));
            const float lo = (t == self) ? best : lo_f(d2), hi = (t + 1 == self) ? best : hi_f(d2);
            best = fminf(best, fminf(lo, hi));
        }
        if (t < m && t != self) {
            const float4 q = s_p[t];
            const float dx = __fsub_rn(xi, q.x), dy = __fsub_rn(yi, q.y), dz = __fsub_rn(zi, q.z);
            best = fminf(best, __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz)));
        }
    }
    if (i < n) atomicMin(nn2 + i, __float_as_int(best));
}
__global__ void k_fill_inf(int* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = 0x7f800000;
}
// k-th smallest (0-based) of n non-negative float bit patterns; *out = sqrt of it (the distance)
__global__ void __launch_bounds__(1024) k_select_kth(const int* v, int n, int k, float* out) {
    __shared__ unsigned s_h[256];
    __shared__ unsigned s_prefix, s_mask, s_k;
    if (threadIdx.x == 0) { s_prefix = 0u; s_mask = 0u; s_k = (unsigned)k; }
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) s_h[b] = 0u;
        __syncthreads();
        const unsigned prefix = s_prefix, mask = s_mask;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned u = (unsigned)v[i];
            if ((u & mask) == prefix) atomicAdd(&s_h[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned kk = s_k, b = 0;
            while (s_h[b] <= kk) { kk -= s_h[b]; ++b; }
            s_k = kk;
            s_prefix = prefix | (b << shift);
            s_mask = mask | (255u << shift);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = __fsqrt_rn(__uint_as_float(s_prefix));
}

// ------------------------------------------------------------------------------------------ NEXT(4)
// Equal-budget 3-point RANSAC baseline: slot k of the clique list gets the sorted
// distinct triple drawn from the counter-based SplitMix64 stream (x_m = mix(seed + (m+1)·γ), draws 3k..3k+2:
// a = x mod n, b = x' mod (n-1) skipping a, c = x'' mod (n-2) skipping a and b), S = 0; k_kabsch, k_score
// and k_finalize then run unchanged on ws.k1 = iters, ws.k2 = 1.
__device__ __forceinline__ uint64_t sm64_draw(uint64_t seed, uint64_t m) {
    uint64_t x = seed + (m + 1ull) * 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__global__ void __launch_bounds__(256) k_ransac_sample(WS ws, unsigned long long seed) {
    const int q = blockIdx.y;
    const PairDesc d = ws.desc[q];
    const int K = ws.k1 * ws.k2;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0) { ws.st[q].npiv = 0; ws.st[q].edges = 0; }
    if (k >= K) return;
    int4 c = make_int4(-1, -1, -1, 0);
    const int n = d.n;
    if (n >= 3) {
        const uint64_t m = 3ull * (uint64_t)k;
        long long a = (long long)(sm64_draw(seed, m) % (uint64_t)n);
        long long b = (long long)(sm64_draw(seed, m + 1) % (uint64_t)(n - 1));
        b += (b >= a);
        long long e = (long long)(sm64_draw(seed, m + 2) % (uint64_t)(n - 2));
        e += (e >= min(a, b));
        e += (e >= max(a, b));
        const long long lo = min(a, min(b, e)), hi = max(a, max(b, e));
        c = make_int4((int)lo, (int)(a + b + e - lo - hi), (int)hi, 0);
    }
    ws.cliq[q * ws.cl_stride + k] = c;
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
#ifndef TRK_SCORE_MINB
#define TRK_SCORE_MINB 4
#endif
__global__ void __launch_bounds__(SCORE_THREADS, (NP == 1 ? 8 : TRK_SCORE_MINB)) k_score(WS ws, int segs) {
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
    // thr2 = RN(thr·thr) (reading r13); thrn = the next float above it: s <= thr2 ⇔ s < thrn ⇔ the sign bit of
    // fl(s − thrn) (a difference of two floats is 0 only when they are equal, so the sign is exact)
    const float thrn = __uint_as_float(__float_as_uint(__fmul_rn(ws.thr, ws.thr)) + 1u);
    const f2_t thrn2 = f2_pack(thrn, thrn);
    f2_t Rp[NP][9], tp[NP][3];
#pragma unroll
    for (int m = 0; m < NP; ++m) {
#pragma unroll
        for (int k = 0; k < 9; ++k) Rp[m][k] = f2_pack(Rh[2 * m][k], Rh[2 * m + 1][k]);
#pragma unroll
        for (int k = 0; k < 3; ++k) tp[m][k] = f2_pack(Rh[2 * m][9 + k], Rh[2 * m + 1][9 + k]);
    }
    const f2_t mone = f2_pack(-1.0f, -1.0f);
    uint32_t cnt[NH];
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
                // inlier ⇔ s − thrn < 0: one packed subtract for both hypotheses, then the sign bits are added
                // (LEA.HI) — integer ALU instructions take FP32-pipe issue slots on this part, FADD2 halves them
                const f2_t dd = f2_sub(sq, thrn2);
                asm("{ .reg .b32 lo, hi; mov.b64 {lo, hi}, %2; shr.u32 lo, lo, 31; shr.u32 hi, hi, 31; "
                    "add.u32 %0, %0, lo; add.u32 %1, %1, hi; }"  // one LEA.HI per hypothesis
                    : "+r"(cnt[2 * m]), "+r"(cnt[2 * m + 1]) : "l"(dd));
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
        if constexpr (ERR)  // this segment's partial sums in their own slot: no float atomics (deterministic)
            ws.herr[(q * ws.cl_stride + h) * SCORE_SEGS_MAX + seg] = make_double2(ea[u], es[u]);
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

__global__ void __launch_bounds__(1024) k_finalize(WS ws) {
    __shared__ unsigned long long s_red[32];
    __shared__ int s_cnt[2][32];
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
    double2* hes = ws.herr + q * ws.cl_stride * SCORE_SEGS_MAX;
    if ((ws.err_mode & 1) && d.n > 0) {  // MAE/MSE sums: the segments' partials added in segment order
        for (int s = t; s < K; s += blockDim.x) {
            double2 a = hes[(int64_t)s * SCORE_SEGS_MAX];
#pragma unroll
            for (int g = 1; g < SCORE_SEGS_MAX; ++g) {
                const double2 b = hes[(int64_t)s * SCORE_SEGS_MAX + g];
                a.x += b.x;
                a.y += b.y;
            }
            hes[(int64_t)s * SCORE_SEGS_MAX] = a;
        }
        __syncthreads();
    }
    auto he_of = [&](int s) { return hes[(int64_t)s * SCORE_SEGS_MAX]; };
    auto quad = [&](int s) { return *reinterpret_cast<const int4*>(hyp + (int64_t)s * 16 + 12); };  // count, flag, S
    auto key_of = [&](int s, const int4 h) -> unsigned long long {
        if (rank == 0) return ((unsigned long long)(unsigned)h.x << 17) | (unsigned)h.z;
        const double2 hv = he_of(s);
        const double e = rank == 1 ? hv.x : hv.y;
        return ~(unsigned long long)__double_as_longlong(e);
    };
    unsigned long long best1 = 0ull;
    int ncl = 0, nev = 0;
    if (d.n > 0) {
        for (int s = t; s < K; s += blockDim.x) {
            const int4 h = quad(s);
            const int flag = h.y;
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
        for (int w = 0; w < 32; ++w) { b = s_red[w] > b ? s_red[w] : b; a += s_cnt[0][w]; e += s_cnt[1][w]; }
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
                const int4 h = quad(s);
                if (h.y == 0 && key_of(s, h) == best1) ms = max(ms, h.z);
            }
        ms = (int)__reduce_max_sync(FULL, (unsigned)(ms + 1)) - 1;
        if (lane == 0) s_cnt[0][warp] = ms;
        __syncthreads();
        if (t == 0) {
            int m = -1;
            for (int w = 0; w < 32; ++w) m = max(m, s_cnt[0][w]);
            s_cnt[0][0] = m;
        }
        __syncthreads();
        bestS = s_cnt[0][0];
        __syncthreads();
    }
    unsigned long long bestt = ~0ull;
    if (d.n > 0 && nev > 0) {
        for (int s = t; s < K; s += blockDim.x) {
            const int4 h = quad(s);
            if (h.y != 0) continue;
            const unsigned long long key = key_of(s, h);
            if (key != best1) continue;
            if (rank != 0 && h.z != bestS) continue;
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
        for (int w = 0; w < 32; ++w) b = s_red[w] < b ? s_red[w] : b;
        s_red[0] = b;
    }
    __syncthreads();
    bestt = s_red[0];
    if (bestt != ~0ull) {  // the slot holding the winning triple (duplicates carry identical values)
        for (int s = t; s < K; s += blockDim.x) {
            const int4 h = quad(s);
            if (h.y != 0) continue;
            if (key_of(s, h) != best1) continue;
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
        if (status == 0 && st->edge_overflow) status = 8;  // TURBOREG_ERR_EDGE_CAPACITY
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
        r.num_edges = (d.n > 0) ? (st->edge_overflow ? (int64_t)(st->deg_sum >> 1) : st->edges) : 0;
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
