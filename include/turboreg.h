/* =====================================================================================================
 * turboreg.h — C ABI of the B200-native TurboReg hot path (arXiv 2507.01439).
 *
 * The library computes, for each registration pair (a set of N putative correspondences
 * m_i = (x_i, y_i)), the hot path of TurboReg (Fig. 2 caption):
 *
 *   (a2) compatibility graph C at the stringent τ (Eq. 1, Def. 1) as bit rows,
 *        optionally a second plane C(τ_base) (SURVEY §8(c) reading c3);
 *   (a3) SC^2 weights Ĝ = C ⊙ (C·C) (Eq. 2) and the O2Graph view Õ (Def. 2);
 *   (a4) pivots: the K1 highest-weighted O2 edges (Eq. 4, Alg. 1 L4 P:261);
 *   (a5) Pivot-Guided Search: per pivot, the top-K2 TurboCliques by S^(ij)(z) (Eqs. 5-7 P:202-220,
 *        Alg. 1);
 *   (a6) a Kabsch rigid fit per TurboClique;
 *   (a7) the inlier number g(T) of every hypothesis against all N correspondences;
 *   (a8) T* = argmax g (Eq. 9).
 *
 * Conventions: indices 0-based; y ≈ R·x + t; R row-major; float32 inputs.
 * Every tie is broken deterministically: pivots (w desc, i asc, j asc); TurboCliques per pivot
 * (S desc, z asc); the final argmax (g desc, S desc, (i,j,z) asc).
 *
 * All kernels are hand-written CUDA for sm_100a; there is no CPU fallback.  Functions return a
 * turboreg_status; argument and validation failures return before any launch and write nothing.
 * ===================================================================================================*/
#ifndef TURBOREG_H
#define TURBOREG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct turboreg_ctx turboreg_ctx; /* opaque; owns all device workspace and one CUDA stream */

typedef enum {
    TURBOREG_OK = 0,
    TURBOREG_ERR_INVALID_ARGUMENT = 1, /* NULL pointer; tau <= 0; k1 < 1; k2 < 1; inlier_threshold <= 0;
                                          tau_base not 0 and < tau; unknown graph_mode or flags;
                                          graph_mode 1 with k1*k2 > 16384;
                                          batch < 1 or > max_batch; max_n outside [3, 32768]        */
    TURBOREG_ERR_TOO_FEW_POINTS = 2,   /* N < 3: no 3-clique exists          — per pair */
    TURBOREG_ERR_TOO_MANY_POINTS = 3,  /* N > max_n fixed at create                         — per pair */
    TURBOREG_ERR_NONFINITE_INPUT = 4,  /* a NaN/Inf coordinate                       — per pair */
    TURBOREG_ERR_NO_HYPOTHESIS = 5,    /* no pivot, no clique, or every clique degenerate;
                                          R, t are all zeros — never a fabricated transform  — per pair */
    TURBOREG_ERR_CUDA = 6,             /* a CUDA runtime error (whole call)                              */
    TURBOREG_ERR_OUT_OF_MEMORY = 7,    /* workspace allocation failed at create/set_params/set_option
                                          (whole call; the context keeps its previous workspace)        */
    TURBOREG_ERR_EDGE_CAPACITY = 8     /* the pair's compatibility graph has more undirected edges than the
                                          per-pair edge capacity fixed at create (turboreg_create_ex):
                                          nothing after the graph is computed; out.num_edges holds the
                                          pair's true edge count so the caller can size a new context
                                                                                            — per pair */
} turboreg_status;

/* Largest cloud accepted by turboreg_point_resolution (O(n^2) distance evaluations). */
#define TURBOREG_MAX_CLOUD_POINTS (1 << 21)

/* turboreg_params.flags */
#define TURBOREG_F_STAGE_TIMING 0x1u  /* fill turboreg_result.stage_ms (CUDA events; adds ~12 events)  */
#define TURBOREG_F_KERNEL_TIMING 0x2u /* accumulate per-kernel CUDA-event times, see turboreg_profile_* */
#define TURBOREG_F_HYP_ERRORS 0x4u    /* also accumulate MAE / MSE of every hypothesis over all N
                                         correspondences (App. F.1, reading r20; TURBOREG_I_ERRORS)      */
#define TURBOREG_F_RANK_MAE 0x8u      /* select T* by minimum MAE instead of maximum inlier number
                                         (ties: S desc, then (i,j,z) asc); implies HYP_ERRORS           */
#define TURBOREG_F_RANK_MSE 0x10u     /* likewise by minimum MSE; not together with RANK_MAE             */
#define TURBOREG_F_ROW_SUMS 0x20u     /* also compute the per-row SC^2 sums r_i = Σ_j Ĝ_ij (= 2·t_i, App. B
                                         P:755-761) after the SC^2 assembly (TURBOREG_I_ROWSUM)          */

typedef struct {
    float tau;              /* τ of Eq. 1, metres, > 0: the stringent TurboClique threshold (Def. 1); drives
                               SC^2, O2, pivots and cliques                                              */
    float tau_base;         /* optional second compatibility plane C(τ_base), τ_base >= τ; 0 = not built  */
    int32_t k1;             /* K1 pivots (Eq. 4); paper: 1000/2000 indoor, 250/500 outdoor     */
    int32_t k2;             /* K2 TurboCliques per pivot (Eq. 7); paper: 2                       */
    float inlier_threshold; /* residual bound of g(·), metres, > 0 (paper silent; reading r12)          */
    int32_t graph_mode;     /* 0 = O2Graph (Def. 2, the paper's method); 1 = undirected SC^2 graph
                               (Table 5 row 10): cliques from neighbours on both sides of a pivot,
                               listed in canonical order (S desc, i, j, z asc) with duplicates removed
                               (reading r9); requires k1*k2 <= 16384                                    */
    uint32_t flags;         /* TURBOREG_F_*                                                               */
} turboreg_params;

typedef struct {
    float R[9];                   /* T* rotation, row-major; zeros unless status == TURBOREG_OK        */
    float t[3];                   /* T* translation                                                     */
    int32_t inlier_count;         /* g(T*), exact integer                                        */
    int32_t clique[3];            /* the winning TurboClique, i < j < z; -1 when none                   */
    int32_t clique_weight;        /* S^(ij)(z) of the winner (Eq. 6)                                     */
    int32_t num_pivots;           /* |P| = min(K1, #edges with Ĝ > 0)                                    */
    int32_t num_cliques;          /* |C| <= K1*K2 (no padding, reading r7)                               */
    int32_t hypotheses_evaluated; /* num_cliques minus degenerate cliques                        */
    int32_t status;               /* turboreg_status of this pair                                        */
    float stage_ms[3];            /* graph / PGS / model estimation (App. F.3 naming); 0 unless
                                     TURBOREG_F_STAGE_TIMING (per call, not per pair)                   */
    int64_t num_edges;            /* undirected edges of C(τ)                                            */
} turboreg_result;

/* Create a context on CUDA device `device` for the problem of P:116-118 (given the putative correspondences
 * of a pair, estimate T in SE(3)) with the parameters of Eq. 1 (tau), Eq. 4 (k1), Eq. 7 (k2) and g(.) of
 * P:284-287 (inlier_threshold); SPEC S:47-51 (EstimatorParams) for the parameter set.  The context can
 * register up to `max_batch` pairs of up to `max_n` correspondences per call (3 <= max_n <= 32768, the
 * uint16 index range of the O2 edge lists; 1 <= max_batch <= 65535).  All device workspace is allocated
 * here, in one allocation (no allocation on the register path): per pair about max_n²/8 bytes of bit rows
 * (Eq. 1), 4 bytes per O2 edge of capacity (Eq. 2 weights in compact rows, Def. 2), the tensor-core operand
 * block (≈ 2048 × max_n/2 bytes) and O(max_n + k1·k2) more; turboreg_workspace_bytes reports the total.
 * turboreg_create reserves the complete-graph edge capacity max_n(max_n−1)/2 (no pair can overflow);
 * turboreg_create_ex takes `max_edges` per pair instead (0 = complete graph), e.g. a density bound for large
 * batches — pairs with more edges report TURBOREG_ERR_EDGE_CAPACITY.  On success *out receives the context
 * (caller owns it; release with turboreg_destroy); on failure nothing is allocated and *out is NULL.
 * Errors: invalid params / sizes → INVALID_ARGUMENT; no such device → CUDA; allocation → OUT_OF_MEMORY. */
turboreg_status turboreg_create(const turboreg_params* params, int device, int32_t max_n, int32_t max_batch,
                                turboreg_ctx** out);
turboreg_status turboreg_create_ex(const turboreg_params* params, int device, int32_t max_n, int32_t max_batch,
                                   int64_t max_edges, turboreg_ctx** out);

/* Replace the parameters (same meaning and validation as at create; e.g. tau = 0.25 · the point-cloud
 * resolution, after turboreg_point_resolution).  Waits for the context's previous call to finish.
 * A change of k1, k1·k2, graph_mode or whether tau_base is set reallocates the workspace: the new one is
 * allocated before the old one is freed, and on OUT_OF_MEMORY the context keeps its old parameters and
 * workspace (still usable).  Errors: INVALID_ARGUMENT (params rejected, nothing changed), OUT_OF_MEMORY. */
turboreg_status turboreg_set_params(turboreg_ctx* ctx, const turboreg_params* params);

/* Register one pair: the whole hot path (Fig. 2 caption P:99-107; Alg. 1 P:256-278 then Eq. 9),
 * result as in SPEC S:53-58 (RegistrationResult).  src_xyz, dst_xyz: N×3 float32 row-major (x_i and y_i,
 * correspondence order preserved — O2 depends on it), HOST or DEVICE pointers (detected; the caller
 * keeps ownership).  Runs on the context's own stream and blocks: on return *out (host) holds the result.
 * Per-pair failures (2/3/4/5/8) are returned as the function value AND in out->status; a device `out`
 * → INVALID_ARGUMENT. */
turboreg_status turboreg_register(turboreg_ctx* ctx, const float* src_xyz, const float* dst_xyz, int32_t n,
                                  turboreg_result* out);

/* Point-cloud resolution for the τ initialisation τ = 0.25 · pr (
 * SPEC S:163-171 estimate_resolution): *out_pr = the median over the n points of the distance to each
 * point's nearest other point, distances in the float32 tree of reading r1, the lower median (element
 * (n-1)/2 of the sorted distances, reading r22).  xyz: n×3 float32 row-major, HOST or DEVICE (detected);
 * blocking.  Errors: n < 2, n > TURBOREG_MAX_CLOUD_POINTS or a null pointer → TURBOREG_ERR_INVALID_ARGUMENT;
 * a non-finite coordinate → TURBOREG_ERR_NONFINITE_INPUT (*out_pr untouched).  n is independent of max_n: the call uses
 * its own device buffers (grown on demand), after the context's previous call has finished. */
turboreg_status turboreg_point_resolution(turboreg_ctx* ctx, const float* xyz, int32_t n, float* out_pr);

/* Equal-budget 3-point RANSAC baseline (SPEC S:324-332 — not part of TurboReg):
 * `iters` hypotheses from correspondence triples drawn uniformly without replacement by the counter-based
 * SplitMix64 generator (draw m = mix(seed + (m+1)·0x9e3779b97f4a7c15); triple k uses draws 3k..3k+2:
 * a = d0 mod n, b = d1 mod (n-1) skipping a, c = d2 mod (n-2) skipping a and b; sorted ascending), each
 * fitted and scored exactly like a TurboClique (3-point Kabsch, degeneracy test r11, inlier number r13),
 * winner by (count desc, (i,j,z) asc).  Same inputs, blocking behaviour and result record as
 * turboreg_register (clique = winning triple, clique_weight = 0, num_pivots = num_edges = 0,
 * num_cliques = iters); always ranks by inlier number.  Requires 1 <= iters <= the context's K1·K2
 * (else TURBOREG_ERR_INVALID_ARGUMENT).  The per-hypothesis intermediates (TURBOREG_I_CLIQUES /
 * TURBOREG_I_HYPS) of the call hold the sampled triples and their fits. */
turboreg_status turboreg_ransac(turboreg_ctx* ctx, const float* src_xyz, const float* dst_xyz, int32_t n, int32_t iters,
                                uint64_t seed, turboreg_result* out);

/* Register `batch` independent pairs in one pass (the pairs of a sweep such as 3DMatch's 1623, are
 * independent problems of P:116-118).  Pair p uses points [offsets[p], offsets[p] + n[p]) of
 * src_xyz / dst_xyz (N×3 float32, host or device; the caller guarantees those rows exist — the C ABI cannot
 * check buffer extents).  offsets and n are HOST arrays.  out: `batch` results (>= batch·sizeof(result)
 * bytes), HOST or DEVICE pointer.  stream: a cudaStream_t (NULL = the context's own stream).
 * With a host `out` the call blocks until the results are in `out`; with a device `out` and device
 * inputs it is asynchronous on `stream` (the caller must keep inputs alive and unmodified until the stream
 * reaches that point).  Consecutive calls may use different streams: each call's stream first waits for
 * the previous call on this context (the workspace is shared), and host-side descriptor staging is a ring
 * that is never overwritten before its copy has run.  A context is not thread-safe; independent contexts
 * may run concurrently.  Per-pair failures go into out[p].status and the call returns TURBOREG_OK;
 * argument errors (null pointer, batch outside [1, max_batch], negative offset or n) return
 * INVALID_ARGUMENT before anything is launched; CUDA errors are returned for the whole call. */
turboreg_status turboreg_register_batch(turboreg_ctx* ctx, const float* src_xyz, const float* dst_xyz,
                                        const int64_t* offsets, const int32_t* n, int32_t batch,
                                        turboreg_result* out, void* stream);

/* One hypothesis of the ranked list (SPEC RegistrationResult.ranked_hypotheses). */
typedef struct {
    int32_t clique[3];     /* TurboClique i < j < z                                                        */
    int32_t clique_weight; /* S^(ij)(z) (Eq. 6)                                                            */
    float R[9];            /* its Kabsch fit, row-major                                            */
    float t[3];
    int32_t inlier_count;  /* g(T)                                                             */
    int32_t slot;          /* its slot in the clique list (TURBOREG_I_CLIQUES)                              */
    double mae, mse;       /* over all N correspondences (reading r20); NaN unless the context accumulates
                              errors (TURBOREG_F_HYP_ERRORS or a RANK flag)                                 */
} turboreg_hypothesis;

/* The valid (non-degenerate) hypotheses of pair `pair` of the LAST register call, ranked by `metric`
 * (App. F.1: 0 = inlier number IN descending, 1 = MAE ascending, 2 = MSE ascending; ties S desc,
 * then (i,j,z) asc — the argmax order of readings r14/r20, so entry 0 under the context's own ranking is
 * the returned T*).  Writes the first min(top_k, #valid) entries to the HOST array `out` and that number to
 * *count.  The ranking runs on the GPU (a bitonic network over the K1·K2 slots, off the hot path) after the
 * context's last call has finished.  Errors: null ctx/count, top_k < 0, out NULL with top_k > 0, pair not
 * in the last call or not registered, metric outside 0..2, metric 1/2 without error accumulation, or
 * K1·K2 > 2^22 → INVALID_ARGUMENT. */
turboreg_status turboreg_ranked_hypotheses(turboreg_ctx* ctx, int32_t pair, int32_t metric, int32_t top_k,
                                           turboreg_hypothesis* out, int32_t* count);

/* ----------------------------------------------------------------- NEXT(1): one pair split over ranks
 * Pivot-level parallelism across GPUs for large N ("Pivot-level Parallelism"; SPEC S:268-269;
 * SURVEY §8(e)).  Each of `world` ranks (one context per GPU, same parameters) runs the three phases below
 * on the same pair; the caller exchanges device buffers between them (all-reduce SUM, all-gather), e.g. with
 * NCCL — paper_2507_01439_b200/split.py does it over torch.distributed.  Work split: compat block-row pairs,
 * tensor-core tiles, dense-row items, sparse-row groups and pivots are each partitioned into contiguous
 * rank ranges; every bit word of C and every O2 edge word is written by exactly one rank into a zeroed
 * buffer, so a SUM all-reduce rebuilds the full arrays on every rank; pivot selection then runs on identical
 * data everywhere (no candidate exchange needed).  Results are bit-identical to turboreg_register.
 * Requirements: graph_mode 0, inlier-number ranking, no ROW_SUMS, sc2_path != 2 (else INVALID_ARGUMENT).
 *   1. turboreg_split_begin: ingest + this rank's compat tiles into a zeroed bit matrix.
 *        exchange: all-reduce SUM of buffer TURBOREG_SPLIT_BITS (int32 words, n·W of them).
 *   2. turboreg_split_sc2: degrees / heavy split / row classes on the full C, this rank's share of the SC^2
 *        assembly into a zeroed edge array; *num_edges = E (the call synchronises).
 *        exchange: all-reduce SUM of the first E words of buffer TURBOREG_SPLIT_EDGES.
 *   3. turboreg_split_search: pivots (identical on every rank), PGS on this rank's pivot slice, Kabsch and
 *        scoring of its TurboCliques, its local argmax into buffer TURBOREG_SPLIT_RESULT (one record).
 *        exchange: all-gather of the `world` records into a device array (rank order).
 *   4. turboreg_split_merge: T* = the argmax over the gathered records (key of reading r14) on the GPU,
 *        counts summed; `out` host (blocking) or device.
 * src/dst: HOST or DEVICE n×3 float32; phases 1, 3, 4 are asynchronous on `stream` (NULL = context stream).
 * Per-pair statuses 2/3 are returned by turboreg_split_begin; 4/5/8 appear in the merged record. */
#define TURBOREG_SPLIT_BITS 0
#define TURBOREG_SPLIT_EDGES 1
#define TURBOREG_SPLIT_RESULT 2
turboreg_status turboreg_split_begin(turboreg_ctx* ctx, const float* src_xyz, const float* dst_xyz, int32_t n,
                                     int32_t rank, int32_t world, void* cuda_stream);
turboreg_status turboreg_split_buffer(turboreg_ctx* ctx, int32_t which, void** dev_ptr, size_t* bytes);
turboreg_status turboreg_split_sc2(turboreg_ctx* ctx, int64_t* num_edges, void* cuda_stream);
turboreg_status turboreg_split_search(turboreg_ctx* ctx, void* cuda_stream);
turboreg_status turboreg_split_merge(turboreg_ctx* ctx, const void* parts, int32_t world, turboreg_result* out,
                                     void* cuda_stream);

/* Release the context and all its device memory, after its last call has finished.  NULL is ignored. */
void turboreg_destroy(turboreg_ctx* ctx);

/* Static, human-readable name of a status. */
const char* turboreg_status_string(turboreg_status s);

/* ---------------------------------------------------------------------------------- test / profiling */
/* Intermediates of pair `pair` of the LAST register call (kept in the workspace until the next call),
 * copied to host buffer dst (capacity `bytes`).  *needed (may be NULL) receives the byte size.  `what`:
 *   TURBOREG_I_BITS      uint32 [n][W]  rows of C(τ), W = words per row (*needed / (4n))
 *   TURBOREG_I_BITS_BASE uint32 [n][W]  rows of C(τ_base) (only if tau_base > 0)
 *   TURBOREG_I_SC2       int32  [n][n]  Ĝ expanded to a dense symmetric matrix
 *   TURBOREG_I_PIVOTS    int32  [P][3]  (i, j, w) in (w desc, i asc, j asc) order — (i, j) lexicographic
 *                        order when more than 8192 edges reach the cut weight α_K1
 *   TURBOREG_I_CLIQUES   int32  [K1*K2][4] (i, j, z, S), i < j < z: O2 mode per slot p*K2 + r; SC^2 mode
 *                        in canonical order, de-duplicated, compacted; empty slots are (-1,-1,-1,0)
 *   TURBOREG_I_HYPS      float  [K1*K2][16]: R[9], t[3], count (int32 bits), flag (int32 bits:
 *                        0 valid, 1 degenerate, 2 empty slot), S (int32 bits), 0
 *   TURBOREG_I_ERRORS    double [K1*K2][2] (MAE, MSE) per slot, NaN for empty / degenerate slots (needs
 *                        TURBOREG_F_HYP_ERRORS or a RANK flag, else TURBOREG_ERR_INVALID_ARGUMENT)
 *   TURBOREG_I_EDGES     uint32 [n+1 + E] the compact O2 rows: rowptr[0..n], then E words (j << 16) | Ĝ_ij,
 *                        row i's upper edges (j > i) in increasing j at rowptr[i]
 *   TURBOREG_I_STATE     int64  [16] per-pair scalars: n, W, edges, positive edges, alpha, c_gt, need,
 *                        num_pivots, nonfinite, ...
 *   TURBOREG_I_ROWSUM    int32  [n] r_i = Σ_j Ĝ_ij (needs TURBOREG_F_ROW_SUMS, else INVALID_ARGUMENT)   */
#define TURBOREG_I_BITS 1
#define TURBOREG_I_BITS_BASE 2
#define TURBOREG_I_SC2 3
#define TURBOREG_I_PIVOTS 4
#define TURBOREG_I_CLIQUES 5
#define TURBOREG_I_HYPS 6
#define TURBOREG_I_STATE 7
#define TURBOREG_I_ERRORS 8
#define TURBOREG_I_EDGES 9
#define TURBOREG_I_ROWSUM 10
turboreg_status turboreg_get_intermediates(turboreg_ctx* ctx, int32_t pair, int32_t what, void* dst, size_t bytes,
                                           size_t* needed);

/* Run steps a3-a5 (SC^2, pivots, PGS) on a caller-supplied adjacency (HOST uint32 bit rows, row r at
 * bits + r*stride_words, bit c of word c/32 = C_rc; must be symmetric with zero diagonal) for one pair of
 * n nodes, using the context's K1, K2, graph_mode.  Results are read back with
 * turboreg_get_intermediates(pair 0, TURBOREG_I_SC2 / _PIVOTS / _CLIQUES). */
turboreg_status turboreg_pgs_from_adjacency(turboreg_ctx* ctx, const uint32_t* bits, int32_t n, int32_t stride_words);

/* Per-kernel CUDA-event timing over a region (requires TURBOREG_F_KERNEL_TIMING in params.flags).
 * profile_begin resets the accumulators; profile_end synchronises the last call's events and writes,
 * for each of the library's kernels k < cap: names[k] (static string), ms[k] (summed duration) and
 * launches[k]; returns the number of kernels in *count. */
turboreg_status turboreg_profile_begin(turboreg_ctx* ctx);
turboreg_status turboreg_profile_end(turboreg_ctx* ctx, const char** names, float* ms, int64_t* launches,
                                     int32_t cap, int32_t* count);

/* Tuning / test knobs (never change results, only which kernels compute them):
 *   "sc2_path"         0 = auto: dense high-degree block on tcgen05 tensor cores + sparse popcount for the
 *                          rest (default); 1 = popcount only; 2 = dense block on CUDA cores (__dp4a) —
 *                          a cross-check of the tensor-core path
 *   "heavy_min_rows"   minimum |H| for the dense block to be used (default 128)
 *   "heavy_min_degree" minimum degree of a heavy row (default 32)
 *   "heavy_cap"        maximum |H| (multiple of 256, <= the allocated capacity)
 *   "pipeline_host_inputs" 1 = a call with host inputs and >= 16 pairs copies them in 8 sub-batches of
 *                      doubling size, each copy overlapping the previous sub-batch's compatibility pass
 *                      (default); 0 = one copy
 *                      before one launch sequence
 *   "mma_fp4"          1 = run the dense block as kind::mxf4.block_scale on packed e2m1 operands (unit block
 *                      scales, fp32 accumulate; exact below 2^24) with 128x240 tiles (default); 0 = kind::i8
 *                      with 128x256 tiles (same results)
 *   "sc2_chunks"       32-word chunks of a dense row per SC^2 work item: 0 = auto (whole rows for batches
 *                      >= 32 pairs, 4 chunks for rows above 512 words, single chunks otherwise), 1..64 fixed
 *   "heavy_widen"      1 = the dense block takes every non-sparse row (degree > list length) that fits the
 *                      cap (default); 0 = only when that adds no 256-row block of the contraction; d > 1 =
 *                      every row of degree >= d that fits the cap (tuning)
 *   "mma_l2_policy"    L2 policy of the dense block's operand (TMA) loads: 1 = evict_last (default),
 *                      0 = evict_normal, 2 = evict_first
 *   "score_pairs"      hypothesis pairs (f32x2 lanes) per scoring thread: 2 (default) or 1
 *   "concurrent_sc2"   1 = the sparse-row SC^2 kernel runs on a second stream alongside the dense-row kernel
 *                      (default; calls with stage/kernel timing stay on one stream); 0 = one stream
 *   "cuda_graph"       1 = replay the launch sequence from a CUDA graph captured per (batch, max n) shape
 *                      (default; calls with stage/kernel timing always launch directly); 0 = launch directly
 *   "compat_variant"   compat-graph tiling: 0 = row pairs in f32x2 lanes x 2 column tiles per warp
 *                      (default); 1 = column pairs x 2 tiles; 2 = row pairs x 1 column tile
 * Returns TURBOREG_ERR_INVALID_ARGUMENT for unknown names or values. */
turboreg_status turboreg_set_option(turboreg_ctx* ctx, const char* name, int64_t value);

/* Number of kernels this context has launched since creation (all calls). */
int64_t turboreg_launch_count(const turboreg_ctx* ctx);

/* Bytes of device workspace owned by the context. */
size_t turboreg_workspace_bytes(const turboreg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TURBOREG_H */
