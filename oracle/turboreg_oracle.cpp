// =====================================================================================================
// TurboReg CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded C++17 implementation of what the TurboReg hot path computes
// (arXiv 2507.01439, /root/reference/PAPER.md, cited as P:<line>).  It exists to prove the CUDA path
// right and nothing else: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it.  The product path (paper_2507_01439_b200/) never imports,
// links or executes anything under oracle/, and this file shares no code, headers, tables or helpers
// with it.
//
// Build: g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see oracle/__init__.py).
// -ffp-contract=off guarantees that no multiply-add is fused unless written as std::fma below, so every
// float32 expression is evaluated exactly in the order it is written (x86-64 SSE, FLT_EVAL_METHOD 0).
//
// Steps follow SURVEY.md §8(c) literally, in the paper's order and notation:
//   1 compatibility graph G (Eq. 1)                         oracle_compat
//   2 SC^2 graph Ĝ_ij = G_ij Σ_k G_ik G_jk (Eq. 2)           oracle_sc2
//   3 O2Graph Õ (Def. 2)                                    oracle_o2
//   4 pivots P = top-K1 edges (Eq. 4; Alg. 1 L4 P:261)      oracle_select_pivots
//   5 PGS per pivot: N(i,j), S^(ij)(z), top-K2 (Eqs. 5-7, Alg. 1)      oracle_pgs
//   6 canonical clique order (+ dedup in SC^2 mode)                    oracle_canonical
//   7 Kabsch per clique, one-sided Jacobi SVD in double        oracle_kabsch
//   8 inlier number g(T) in fixed-order float32            oracle_count_inliers
//   8' MAE / MSE of a hypothesis (App. F.1, reading r20)     oracle_hypothesis_errors
//   9 argmax T* (Eq. 9)                                     oracle_estimate
//   NEXT(3) point-cloud resolution for τ = 0.25 pr              oracle_point_resolution
//   NEXT(4) equal-budget 3-point RANSAC baseline          oracle_ransac
// plus a brute-force 3-clique enumerator used only as a test pin (App. B/C).
//
// Every reading of a point where the paper is silent is listed in DESIGN.md §"Readings" (r1..r18) and
// referenced below by its number.  Parity status of every function: pinned (tests/test_oracle_*.py).
// =====================================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

struct oracle_params {
    float tau;               // τ of Eq. 1 (the stringent TurboClique threshold, Def. 1)
    int32_t k1;              // K1, number of pivots (Eq. 4)
    int32_t k2;              // K2, TurboCliques per pivot (Eq. 7)
    float inlier_threshold;  // residual bound of g(·) (reading r12)
    int32_t graph_mode;      // 0 = O2Graph (Def. 2), 1 = undirected SC^2 graph (Table 5 row 10)
    int32_t rank_metric;     // 0 = inlier number (Eq. 9), 1 = MAE, 2 = MSE (App. F.1, reading r20)
};

struct oracle_result {
    float R[9];
    float t[3];
    int32_t inlier_count;
    int32_t clique[3];
    int32_t clique_weight;
    int32_t num_pivots;
    int32_t num_cliques;
    int32_t hypotheses_evaluated;
    int32_t status;             // 0 ok, 5 = no hypothesis
    int64_t num_edges;          // undirected edges of G
    int64_t near_edges;         // pairs within the near-threshold band of τ (reading r1)
    int64_t f64_disagreements;  // pairs whose float64 decision differs from the float32 one
    int64_t neighbor_checks;    // Alg. 1 L8 evaluations = Σ_pivots (N-2)
    int32_t best_count_f64;     // shadow: inliers of the winner's float64 (R,t) in float64
    int32_t near_corr;          // winner: correspondences within the near band of the inlier threshold
    double mae, mse;            // winner's mean absolute / squared residual (reading r20)
};

// ------------------------------------------------------------------------------------------ step 1
// Eq. 1: G_ij = 1 iff | ||x_i - x_j|| - ||y_i - y_j|| | <= τ.  Reading r1: float32,
// round-to-nearest, written order ((dx*dx + dy*dy) + dz*dz), sqrtf, fabsf, closed "<=" (r2), G_ii = 0.
// Every ordered pair (i,j), i != j, is evaluated on its own (no mirroring).
// Diagnostics: near_count counts unordered pairs with |Δ64 - τ| <= 1e-6 + 4 ulp_f32(max(a,b));
// f64_disagree counts unordered pairs whose decision in float64 differs.
static float f32_dist(const float* p, const float* q) {
    float dx = p[0] - q[0];
    float dy = p[1] - q[1];
    float dz = p[2] - q[2];
    float s = (dx * dx + dy * dy) + dz * dz;
    return std::sqrt(s);
}
static double f64_dist(const float* p, const float* q) {
    double dx = (double)p[0] - (double)q[0];
    double dy = (double)p[1] - (double)q[1];
    double dz = (double)p[2] - (double)q[2];
    return std::sqrt((dx * dx + dy * dy) + dz * dz);
}
static double ulp_f32(float v) {
    float a = std::fabs(v);
    return (double)std::nextafter(a, INFINITY) - (double)a;
}

int64_t oracle_compat(const float* src, const float* dst, int32_t n, float tau, uint8_t* C,
                      int64_t* near_count, int64_t* f64_disagree) {
    int64_t edges = 0, near = 0, dis = 0;
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t j = 0; j < n; ++j) {
            if (i == j) { C[(int64_t)i * n + j] = 0; continue; }
            float a = f32_dist(src + 3 * i, src + 3 * j);
            float b = f32_dist(dst + 3 * i, dst + 3 * j);
            float delta = std::fabs(a - b);
            uint8_t e = (delta <= tau) ? 1 : 0;
            C[(int64_t)i * n + j] = e;
            if (i < j) {
                edges += e;
                double a64 = f64_dist(src + 3 * i, src + 3 * j);
                double b64 = f64_dist(dst + 3 * i, dst + 3 * j);
                double d64 = std::fabs(a64 - b64);
                double band = 1e-6 + 4.0 * ulp_f32(std::max(a, b));
                if (std::fabs(d64 - (double)tau) <= band) ++near;
                if ((d64 <= (double)tau) != (e == 1)) ++dis;
            }
        }
    }
    if (near_count) *near_count = near;
    if (f64_disagree) *f64_disagree = dis;
    return edges;
}

// ------------------------------------------------------------------------------------------ step 2
// Eq. 2: Ĝ_ij = G_ij Σ_k G_ik G_jk, exact 32-bit integer count; when G_ij = 0 the product
// is zero and the sum is skipped.  Full N×N, every (i,j) evaluated on its own.
void oracle_sc2(const uint8_t* C, int32_t n, int32_t* G) {
    for (int32_t i = 0; i < n; ++i) {
        const uint8_t* ci = C + (int64_t)i * n;
        for (int32_t j = 0; j < n; ++j) {
            int32_t s = 0;
            if (ci[j]) {
                const uint8_t* cj = C + (int64_t)j * n;
                for (int32_t k = 0; k < n; ++k) s += (int32_t)ci[k] * (int32_t)cj[k];
            }
            G[(int64_t)i * n + j] = s;
        }
    }
}

// ------------------------------------------------------------------------------------------ step 3
// Def. 2: Õ_ij = Ĝ_ij for i < j, 0 for i >= j.
void oracle_o2(const int32_t* G, int32_t n, int32_t* O) {
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < n; ++j)
            O[(int64_t)i * n + j] = (i < j) ? G[(int64_t)i * n + j] : 0;
}

// ------------------------------------------------------------------------------------------ step 4
// Eq. 4, Alg. 1 L4: the K1 highest-weighted edges.  Readings: only i < j (r4),
// only weight > 0 (r5), ties at the cut broken by (i, j) ascending (r5), order (w desc, i asc, j asc).
// Output piv[p] = (i, j, w); returns |P| = min(K1, #positive edges).
int32_t oracle_select_pivots(const int32_t* Gbar, int32_t n, int32_t k1, int32_t* piv) {
    struct E { int32_t w, i, j; };
    std::vector<E> cand;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = i + 1; j < n; ++j) {
            int32_t w = Gbar[(int64_t)i * n + j];
            if (w > 0) cand.push_back({w, i, j});
        }
    std::sort(cand.begin(), cand.end(), [](const E& a, const E& b) {
        if (a.w != b.w) return a.w > b.w;
        if (a.i != b.i) return a.i < b.i;
        return a.j < b.j;
    });
    int32_t m = (int32_t)std::min<int64_t>((int64_t)k1, (int64_t)cand.size());
    for (int32_t p = 0; p < m; ++p) {
        piv[3 * p + 0] = cand[p].i;
        piv[3 * p + 1] = cand[p].j;
        piv[3 * p + 2] = cand[p].w;
    }
    return m;
}

// ------------------------------------------------------------------------------------------ step 5
// Alg. 1 L5-13 with Eqs. 5-7, literally:
//   for each pivot (i,j): S = 0^N; for z in {0..N-1} \ {i,j}: if Ḡ_iz > 0 and Ḡ_jz > 0:
//   S(z) = Ḡ_ij + Ḡ_iz + Ḡ_jz; keep top-K2 of S over N(i,j) by (S desc, z asc) (readings r7, r8).
// No padding when |N(i,j)| < K2 (r7, Eq. 7 restricts z to N(i,j)).  Emits (sorted triple, S) per
// clique, pivot after pivot.  *checks counts the L8 neighbour tests (N-2 per pivot).
int32_t oracle_pgs(const int32_t* Gbar, int32_t n, const int32_t* piv, int32_t npiv, int32_t k2,
                   int32_t* cliques, int64_t* checks) {
    int32_t out = 0;
    int64_t chk = 0;
    std::vector<int32_t> S(n);
    std::vector<int32_t> nbr;
    for (int32_t p = 0; p < npiv; ++p) {
        int32_t i = piv[3 * p + 0], j = piv[3 * p + 1];
        std::fill(S.begin(), S.end(), 0);
        nbr.clear();
        for (int32_t z = 0; z < n; ++z) {
            if (z == i || z == j) continue;
            ++chk;
            int32_t giz = Gbar[(int64_t)i * n + z];
            int32_t gjz = Gbar[(int64_t)j * n + z];
            if (giz > 0 && gjz > 0) {
                S[z] = Gbar[(int64_t)i * n + j] + giz + gjz;
                nbr.push_back(z);
            }
        }
        std::sort(nbr.begin(), nbr.end(), [&](int32_t a, int32_t b) {
            if (S[a] != S[b]) return S[a] > S[b];
            return a < b;
        });
        int32_t take = (int32_t)std::min<int64_t>((int64_t)k2, (int64_t)nbr.size());
        for (int32_t r = 0; r < take; ++r) {
            int32_t z = nbr[r];
            int32_t t3[3] = {i, j, z};
            std::sort(t3, t3 + 3);
            cliques[4 * out + 0] = t3[0];
            cliques[4 * out + 1] = t3[1];
            cliques[4 * out + 2] = t3[2];
            cliques[4 * out + 3] = S[z];
            ++out;
        }
    }
    if (checks) *checks = chk;
    return out;
}

// ------------------------------------------------------------------------------------------ step 6
// Canonical list order (S desc, (i,j,z) ascending); in SC^2 mode duplicates are dropped after sorting
// (reading r9; SPEC design decision on "redundant TurboClique detection").
int32_t oracle_canonical(int32_t* cliques, int32_t k, int32_t dedup) {
    struct Q { int32_t i, j, z, s; };
    std::vector<Q> v(k);
    for (int32_t c = 0; c < k; ++c) v[c] = {cliques[4 * c], cliques[4 * c + 1], cliques[4 * c + 2], cliques[4 * c + 3]};
    std::sort(v.begin(), v.end(), [](const Q& a, const Q& b) {
        if (a.s != b.s) return a.s > b.s;
        if (a.i != b.i) return a.i < b.i;
        if (a.j != b.j) return a.j < b.j;
        return a.z < b.z;
    });
    int32_t m = 0;
    for (int32_t c = 0; c < k; ++c) {
        if (dedup && m > 0 && v[m - 1].i == v[c].i && v[m - 1].j == v[c].j && v[m - 1].z == v[c].z) continue;
        v[m++] = v[c];
    }
    for (int32_t c = 0; c < m; ++c) {
        cliques[4 * c] = v[c].i; cliques[4 * c + 1] = v[c].j; cliques[4 * c + 2] = v[c].z; cliques[4 * c + 3] = v[c].s;
    }
    return m;
}

// ------------------------------------------------------------------------------------------ step 7
// Degenerate triangle predicate (reading r11): with a = p1 - p0, b = p2 - p0 in double,
// degenerate iff ||a × b||^2 <= (1e-6)^2 ||a||^2 ||b||^2.
int32_t oracle_triangle_degenerate(const float* p0, const float* p1, const float* p2) {
    double ax = (double)p1[0] - (double)p0[0], ay = (double)p1[1] - (double)p0[1], az = (double)p1[2] - (double)p0[2];
    double bx = (double)p2[0] - (double)p0[0], by = (double)p2[1] - (double)p0[1], bz = (double)p2[2] - (double)p0[2];
    double cx = ay * bz - az * by;
    double cy = az * bx - ax * bz;
    double cz = ax * by - ay * bx;
    double c2 = (cx * cx + cy * cy) + cz * cz;
    double a2 = (ax * ax + ay * ay) + az * az;
    double b2 = (bx * bx + by * by) + bz * bz;
    return (c2 <= 1e-12 * (a2 * b2)) ? 1 : 0;
}

// Kabsch (reading r11): least-squares rigid fit y ≈ R x + t of m >= 3 pairs,
// unweighted, no scale.  H = Σ (x_k - x̄)(y_k - ȳ)^T; H = U Σ V^T by cyclic one-sided Jacobi;
// R = V diag(1, 1, sign det(V U^T)) U^T; t = ȳ - R x̄.  Returns 1 (degenerate) when σ2 <= 1e-12 σ1.
int32_t oracle_kabsch(const double* P, const double* Q, int32_t m, double* R, double* t) {
    double cp[3] = {0, 0, 0}, cq[3] = {0, 0, 0};
    for (int32_t k = 0; k < m; ++k)
        for (int d = 0; d < 3; ++d) { cp[d] += P[3 * k + d]; cq[d] += Q[3 * k + d]; }
    for (int d = 0; d < 3; ++d) { cp[d] /= m; cq[d] /= m; }
    double A[3][3] = {{0}};  // A = H, H[r][c] = Σ_k (x_k - x̄)_r (y_k - ȳ)_c
    for (int32_t k = 0; k < m; ++k)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                A[r][c] += (P[3 * k + r] - cp[r]) * (Q[3 * k + c] - cq[c]);
    double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    // One-sided Jacobi: orthogonalise the columns of A by plane rotations accumulated into V, so that
    // A V = U Σ with orthogonal columns.
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < 2; ++p) {
            for (int q = p + 1; q < 3; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                for (int r = 0; r < 3; ++r) {
                    alpha += A[r][p] * A[r][p];
                    beta += A[r][q] * A[r][q];
                    gamma += A[r][p] * A[r][q];
                }
                if (gamma == 0.0) continue;
                double rel = std::fabs(gamma) / std::sqrt(alpha * beta);
                if (!(rel > 1e-15)) continue;
                off = std::max(off, rel);
                double zeta = (beta - alpha) / (2.0 * gamma);
                double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                double c = 1.0 / std::sqrt(1.0 + tt * tt);
                double s = c * tt;
                for (int r = 0; r < 3; ++r) {
                    double ap = A[r][p], aq = A[r][q];
                    A[r][p] = c * ap - s * aq;
                    A[r][q] = s * ap + c * aq;
                    double vp = V[r][p], vq = V[r][q];
                    V[r][p] = c * vp - s * vq;
                    V[r][q] = s * vp + c * vq;
                }
            }
        }
        if (off <= 1e-15) break;
    }
    double sig[3];
    for (int c = 0; c < 3; ++c) sig[c] = std::sqrt(A[0][c] * A[0][c] + A[1][c] * A[1][c] + A[2][c] * A[2][c]);
    int ord[3] = {0, 1, 2};
    std::sort(ord, ord + 3, [&](int a, int b) { return sig[a] > sig[b]; });
    if (!(sig[ord[0]] > 0.0) || sig[ord[1]] <= 1e-12 * sig[ord[0]]) return 1;
    double U[3][3], Vs[3][3];
    for (int k = 0; k < 3; ++k)
        for (int r = 0; r < 3; ++r) Vs[r][k] = V[r][ord[k]];
    for (int k = 0; k < 2; ++k)
        for (int r = 0; r < 3; ++r) U[r][k] = A[r][ord[k]] / sig[ord[k]];
    if (sig[ord[2]] > 1e-12 * sig[ord[0]]) {
        for (int r = 0; r < 3; ++r) U[r][2] = A[r][ord[2]] / sig[ord[2]];
    } else {  // σ3 = 0 (always for three points): complete U by u3 = u1 × u2; d below fixes the sign
        U[0][2] = U[1][0] * U[2][1] - U[2][0] * U[1][1];
        U[1][2] = U[2][0] * U[0][1] - U[0][0] * U[2][1];
        U[2][2] = U[0][0] * U[1][1] - U[1][0] * U[0][1];
    }
    double M[3][3];  // V U^T
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            M[r][c] = Vs[r][0] * U[c][0] + Vs[r][1] * U[c][1] + Vs[r][2] * U[c][2];
    double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                 M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    double d = det < 0 ? -1.0 : 1.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            R[3 * r + c] = Vs[r][0] * U[c][0] + Vs[r][1] * U[c][1] + d * Vs[r][2] * U[c][2];
    for (int r = 0; r < 3; ++r) t[r] = cq[r] - (R[3 * r] * cp[0] + R[3 * r + 1] * cp[1] + R[3 * r + 2] * cp[2]);
    return 0;
}

// ------------------------------------------------------------------------------------------ step 8
// g(T) = inlier number.  Reading r13: float32, fixed order with explicit fused multiply-adds:
//   p_r = fma(R[r][2], z, fma(R[r][1], y, fma(R[r][0], x, t_r)));  e_r = p_r - y_r;
//   s = fma(e_2, e_2, fma(e_1, e_1, e_0 * e_0));  inlier iff s <= thr2,  thr2 = RN_f32(thr * thr).
int32_t oracle_count_inliers(const float* src, const float* dst, int32_t n, const float* R, const float* t, float thr) {
    float thr2 = thr * thr;
    int32_t cnt = 0;
    for (int32_t k = 0; k < n; ++k) {
        float x = src[3 * k], y = src[3 * k + 1], z = src[3 * k + 2];
        float e[3];
        for (int r = 0; r < 3; ++r) {
            float p = std::fma(R[3 * r + 2], z, std::fma(R[3 * r + 1], y, std::fma(R[3 * r + 0], x, t[r])));
            e[r] = p - dst[3 * k + r];
        }
        float s = std::fma(e[2], e[2], std::fma(e[1], e[1], e[0] * e[0]));
        if (s <= thr2) ++cnt;
    }
    return cnt;
}

// float64 shadow count and near-band count (diagnostics only; reading r13).
// App. F.1 ranks the K1K2 hypotheses by inlier number, mean absolute error (MAE) and mean
// squared error (MSE) without writing the errors out; SPEC ranks MAE/MSE ascending.  Reading
// r20: over all N correspondences, with the residual of reading r13 (float32 FMA tree, s = |r|^2 in
// float32): MAE = (1/N) Σ_k sqrtf(s_k), MSE = (1/N) Σ_k s_k, the sums in float64 in index order.
void oracle_hypothesis_errors(const float* src, const float* dst, int32_t n, const float* R, const float* t,
                              double* mae, double* mse) {
    double sa = 0.0, ss = 0.0;
    for (int32_t k = 0; k < n; ++k) {
        float x = src[3 * k], y = src[3 * k + 1], z = src[3 * k + 2];
        float e[3];
        for (int r = 0; r < 3; ++r) {
            float p = std::fma(R[3 * r + 2], z, std::fma(R[3 * r + 1], y, std::fma(R[3 * r + 0], x, t[r])));
            e[r] = p - dst[3 * k + r];
        }
        float s2 = std::fma(e[2], e[2], std::fma(e[1], e[1], e[0] * e[0]));
        sa += (double)std::sqrt(s2);
        ss += (double)s2;
    }
    *mae = n > 0 ? sa / n : 0.0;
    *mse = n > 0 ? ss / n : 0.0;
}

static void shadow_count(const float* src, const float* dst, int32_t n, const double* R, const double* t, float thr,
                         int32_t* cnt64, int32_t* near) {
    int32_t c = 0, nb = 0;
    for (int32_t k = 0; k < n; ++k) {
        double e2 = 0.0;
        for (int r = 0; r < 3; ++r) {
            double p = R[3 * r] * src[3 * k] + R[3 * r + 1] * src[3 * k + 1] + R[3 * r + 2] * src[3 * k + 2] + t[r];
            double e = p - (double)dst[3 * k + r];
            e2 += e * e;
        }
        double nrm = std::sqrt(e2);
        if (nrm <= (double)thr) ++c;
        if (std::fabs(nrm - (double)thr) <= 1e-6 + 4.0 * ulp_f32(thr)) ++nb;
    }
    *cnt64 = c;
    *near = nb;
}

// Brute-force 3-clique enumeration (test pin for App. B/C): all i<j<z with all three edges.
int64_t oracle_brute_triangles(const uint8_t* C, int32_t n, int32_t* out, int64_t cap) {
    int64_t m = 0;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = i + 1; j < n; ++j) {
            if (!C[(int64_t)i * n + j]) continue;
            for (int32_t z = j + 1; z < n; ++z) {
                if (C[(int64_t)i * n + z] && C[(int64_t)j * n + z]) {
                    if (out && m < cap) { out[3 * m] = i; out[3 * m + 1] = j; out[3 * m + 2] = z; }
                    ++m;
                }
            }
        }
    return m;
}

// ------------------------------------------------------------------------------------------ step 9
// Full pipeline (Fig. 2 caption P:99-107; SPEC estimate S:314-317).  Optional trace buffers
// (NULL = not wanted): C_out [n*n] u8, G_out [n*n] i32 (Ĝ), piv_out [k1*3], cliques_out [k1*k2*4]
// (canonical order), hyp_out [k1*k2*16] floats: R[9], t[3], count (as float bits of int32 via memcpy),
// degenerate flag, S, pad — in canonical clique order.
int32_t oracle_estimate(const float* src, const float* dst, int32_t n, const oracle_params* prm, oracle_result* res,
                        uint8_t* C_out, int32_t* G_out, int32_t* piv_out, int32_t* cliques_out, float* hyp_out,
                        double* err_out) {
    std::memset(res, 0, sizeof(*res));
    if (n < 3) { res->status = 2; return 2; }
    std::vector<uint8_t> C((size_t)n * n);
    res->num_edges = oracle_compat(src, dst, n, prm->tau, C.data(), &res->near_edges, &res->f64_disagreements);
    std::vector<int32_t> G((size_t)n * n);
    oracle_sc2(C.data(), n, G.data());
    std::vector<int32_t> Gbar;
    if (prm->graph_mode == 0) {
        Gbar.resize((size_t)n * n);
        oracle_o2(G.data(), n, Gbar.data());
    } else {
        Gbar = G;
    }
    std::vector<int32_t> piv((size_t)3 * prm->k1);
    int32_t np = oracle_select_pivots(Gbar.data(), n, prm->k1, piv.data());
    res->num_pivots = np;
    std::vector<int32_t> cl((size_t)4 * np * prm->k2 + 4);
    int32_t nc = oracle_pgs(Gbar.data(), n, piv.data(), np, prm->k2, cl.data(), &res->neighbor_checks);
    nc = oracle_canonical(cl.data(), nc, prm->graph_mode == 1 ? 1 : 0);
    res->num_cliques = nc;
    if (C_out) std::memcpy(C_out, C.data(), C.size());
    if (G_out) std::memcpy(G_out, G.data(), G.size() * sizeof(int32_t));
    if (piv_out) std::memcpy(piv_out, piv.data(), (size_t)3 * np * sizeof(int32_t));
    if (cliques_out) std::memcpy(cliques_out, cl.data(), (size_t)4 * nc * sizeof(int32_t));

    int32_t best = -1, best_cnt = -1, best_s = -1;
    double best_err = 0.0;
    int32_t nvalid = 0;
    std::vector<double> bestR64(9), bestt64(3);
    for (int32_t c = 0; c < nc; ++c) {
        int32_t idx[3] = {cl[4 * c], cl[4 * c + 1], cl[4 * c + 2]};
        int32_t s = cl[4 * c + 3];
        float* h = hyp_out ? hyp_out + 16 * (size_t)c : nullptr;
        if (h) std::memset(h, 0, 16 * sizeof(float));
        bool degen = oracle_triangle_degenerate(src + 3 * idx[0], src + 3 * idx[1], src + 3 * idx[2]) ||
                     oracle_triangle_degenerate(dst + 3 * idx[0], dst + 3 * idx[1], dst + 3 * idx[2]);
        double P[9], Q[9], R64[9], t64[3];
        for (int k = 0; k < 3; ++k)
            for (int d = 0; d < 3; ++d) { P[3 * k + d] = src[3 * idx[k] + d]; Q[3 * k + d] = dst[3 * idx[k] + d]; }
        if (!degen && oracle_kabsch(P, Q, 3, R64, t64) != 0) degen = true;
        if (degen) {
            if (h) { int32_t one = 1; std::memcpy(&h[13], &one, 4); }
            if (err_out) err_out[2 * c] = err_out[2 * c + 1] = std::nan("");
            continue;
        }
        ++nvalid;
        float R32[9], t32[3];
        for (int k = 0; k < 9; ++k) R32[k] = (float)R64[k];
        for (int k = 0; k < 3; ++k) t32[k] = (float)t64[k];
        int32_t cnt = oracle_count_inliers(src, dst, n, R32, t32, prm->inlier_threshold);
        double mae = 0.0, mse = 0.0;
        if (prm->rank_metric != 0 || err_out) oracle_hypothesis_errors(src, dst, n, R32, t32, &mae, &mse);
        if (err_out) { err_out[2 * c] = mae; err_out[2 * c + 1] = mse; }
        if (h) {
            std::memcpy(h, R32, sizeof(R32));
            std::memcpy(h + 9, t32, sizeof(t32));
            std::memcpy(&h[12], &cnt, 4);
            std::memcpy(&h[14], &s, 4);
        }
        // Eq. 9 argmax with reading r14: (count desc, S desc, (i,j,z) asc).  The list is already in
        // (S desc, ijz asc) order, so the first strictly larger count wins.
        // reading r20: with rank_metric MAE / MSE the first strictly smaller error wins (ties keep the list's
        // (S desc, ijz asc) order)
        const double err = prm->rank_metric == 1 ? mae : mse;
        const bool better = prm->rank_metric == 0 ? (cnt > best_cnt || (cnt == best_cnt && s > best_s))
                                                  : (best < 0 || err < best_err);
        if (better) {
            best = c; best_cnt = cnt; best_s = s; best_err = err;
            res->mae = mae; res->mse = mse;
            std::memcpy(res->R, R32, sizeof(R32));
            std::memcpy(res->t, t32, sizeof(t32));
            std::memcpy(bestR64.data(), R64, sizeof(R64));
            std::memcpy(bestt64.data(), t64, sizeof(t64));
        }
    }
    res->hypotheses_evaluated = nvalid;
    if (best < 0) {
        std::memset(res->R, 0, sizeof(res->R));
        std::memset(res->t, 0, sizeof(res->t));
        res->status = 5;  // NoHypothesis: never a fabricated transform
        return 5;
    }
    res->inlier_count = best_cnt;
    res->clique[0] = cl[4 * best]; res->clique[1] = cl[4 * best + 1]; res->clique[2] = cl[4 * best + 2];
    res->clique_weight = best_s;
    shadow_count(src, dst, n, bestR64.data(), bestt64.data(), prm->inlier_threshold, &res->best_count_f64, &res->near_corr);
    res->status = 0;
    return 0;
}

// ------------------------------------------------------------------------------------------ NEXT(3)
// Point-cloud resolution for the τ initialisation τ = 0.25 · pr (SPEC S:163-171
// estimate_resolution): the median over points of the distance to each point's nearest other point,
// brute force in the float32 tree of reading r1, the lower median (element (n-1)/2 of the sorted
// distances, reading r22).  Returns -1 for n < 2.
float oracle_point_resolution(const float* xyz, int32_t n) {
    if (n < 2) return -1.f;
    std::vector<float> nn((size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        float best = INFINITY;
        for (int32_t j = 0; j < n; ++j) {
            if (j == i) continue;
            const float d = f32_dist(xyz + 3 * (size_t)i, xyz + 3 * (size_t)j);
            if (d < best) best = d;
        }
        nn[i] = best;
    }
    std::sort(nn.begin(), nn.end());
    return nn[(size_t)(n - 1) / 2];
}

// ------------------------------------------------------------------------------------------ NEXT(4)
// Equal-budget 3-point RANSAC baseline: `iters` hypotheses from uniformly
// drawn correspondence triples, each fitted and scored exactly as steps 7-8, argmax by (count desc,
// (i,j,z) asc) (reading r14 with S = 0).  The random numbers come from the counter-based SplitMix64
// (Steele, Lea & Flood 2014; x_k = mix(seed + (k+1)·0x9e3779b97f4a7c15)), which the CUDA side implements
// independently: triple k uses draws 3k, 3k+1, 3k+2 — a = r0 mod n, b = r1 mod (n-1) skipping a,
// c = r2 mod (n-2) skipping a and b — sorted ascending.
uint64_t oracle_splitmix64(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

void oracle_ransac_triple(uint64_t seed, int64_t k, int32_t n, int32_t* out3) {
    const uint64_t r0 = oracle_splitmix64(seed, 3 * (uint64_t)k), r1 = oracle_splitmix64(seed, 3 * (uint64_t)k + 1),
                   r2 = oracle_splitmix64(seed, 3 * (uint64_t)k + 2);
    int64_t a = (int64_t)(r0 % (uint64_t)n);
    int64_t b = (int64_t)(r1 % (uint64_t)(n - 1));
    if (b >= a) ++b;  // uniform over the n-1 indices other than a
    int64_t c = (int64_t)(r2 % (uint64_t)(n - 2));
    const int64_t lo = std::min(a, b), hi = std::max(a, b);
    if (c >= lo) ++c;  // uniform over the n-2 indices other than a and b
    if (c >= hi) ++c;
    int64_t v[3] = {a, b, c};
    std::sort(v, v + 3);
    for (int q = 0; q < 3; ++q) out3[q] = (int32_t)v[q];
}

int32_t oracle_ransac(const float* src, const float* dst, int32_t n, int32_t iters, uint64_t seed, float thr,
                      oracle_result* res, int32_t* cliques_out, float* hyp_out) {
    std::memset(res, 0, sizeof(*res));
    if (n < 3) { res->status = 2; return 2; }
    int32_t best = -1, best_cnt = -1;
    int32_t best_ijz[3] = {0, 0, 0};
    int32_t nvalid = 0;
    std::vector<double> bestR64(9), bestt64(3);
    for (int32_t c = 0; c < iters; ++c) {
        int32_t idx[3];
        oracle_ransac_triple(seed, c, n, idx);
        if (cliques_out) { cliques_out[4 * c] = idx[0]; cliques_out[4 * c + 1] = idx[1]; cliques_out[4 * c + 2] = idx[2]; cliques_out[4 * c + 3] = 0; }
        float* h = hyp_out ? hyp_out + 16 * (size_t)c : nullptr;
        if (h) std::memset(h, 0, 16 * sizeof(float));
        bool degen = oracle_triangle_degenerate(src + 3 * idx[0], src + 3 * idx[1], src + 3 * idx[2]) ||
                     oracle_triangle_degenerate(dst + 3 * idx[0], dst + 3 * idx[1], dst + 3 * idx[2]);
        double P[9], Q[9], R64[9], t64[3];
        for (int k = 0; k < 3; ++k)
            for (int d = 0; d < 3; ++d) { P[3 * k + d] = src[3 * idx[k] + d]; Q[3 * k + d] = dst[3 * idx[k] + d]; }
        if (!degen && oracle_kabsch(P, Q, 3, R64, t64) != 0) degen = true;
        if (degen) {
            if (h) { int32_t one = 1; std::memcpy(&h[13], &one, 4); }
            continue;
        }
        ++nvalid;
        float R32[9], t32[3];
        for (int k = 0; k < 9; ++k) R32[k] = (float)R64[k];
        for (int k = 0; k < 3; ++k) t32[k] = (float)t64[k];
        const int32_t cnt = oracle_count_inliers(src, dst, n, R32, t32, thr);
        if (h) {
            std::memcpy(h, R32, sizeof(R32));
            std::memcpy(h + 9, t32, sizeof(t32));
            std::memcpy(&h[12], &cnt, 4);
        }
        const bool ijz_less = std::lexicographical_compare(idx, idx + 3, best_ijz, best_ijz + 3);
        if (best < 0 || cnt > best_cnt || (cnt == best_cnt && ijz_less)) {
            best = c; best_cnt = cnt;
            std::memcpy(best_ijz, idx, sizeof(idx));
            std::memcpy(res->R, R32, sizeof(R32));
            std::memcpy(res->t, t32, sizeof(t32));
            std::memcpy(bestR64.data(), R64, sizeof(R64));
            std::memcpy(bestt64.data(), t64, sizeof(t64));
        }
    }
    res->num_cliques = iters;
    res->hypotheses_evaluated = nvalid;
    if (best < 0) {
        std::memset(res->R, 0, sizeof(res->R));
        std::memset(res->t, 0, sizeof(res->t));
        res->status = 5;
        return 5;
    }
    res->inlier_count = best_cnt;
    std::memcpy(res->clique, best_ijz, sizeof(best_ijz));
    shadow_count(src, dst, n, bestR64.data(), bestt64.data(), thr, &res->best_count_f64, &res->near_corr);
    res->status = 0;
    return 0;
}

}  // extern "C"
