// =====================================================================================================
// Host runtime + C ABI of the TurboReg hot path (include/turboreg.h).  Owns the device workspace, the
// stream, per-kernel event timing and the launch sequence of the hand-written sm_100a kernels in
// turboreg_kernels.cuh.  No CPU fallback: every step of the path runs in those kernels.
// =====================================================================================================
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "turboreg.h"
#include "turboreg_kernels.cuh"
#include "turboreg_sc2_mma.cuh"

static_assert(sizeof(trk::DevResult) == sizeof(turboreg_result), "result layout");
static_assert(sizeof(trk::DevHypothesis) == sizeof(turboreg_hypothesis), "hypothesis layout");

namespace {

enum KernelId {
    KID_INGEST = 0,
    KID_COMPAT,
    KID_DEGREE,
    KID_HEAVY,
    KID_ROWCLASS,
    KID_EXPAND,
    KID_SC2_MMA,
    KID_EMIT_HH,
    KID_SC2,
    KID_SC2_LIGHT,
    KID_HIST_HI,
    KID_HIST_LO,
    KID_ALPHA,
    KID_COLLECT,
    KID_PIVOT_SORT,
    KID_SEL_COUNT,
    KID_SEL_SCAN,
    KID_SEL_EMIT,
    KID_PGS,
    KID_CANON,
    KID_KABSCH,
    KID_SCORE,
    KID_FINALIZE,
    KID_RANSAC,
    KID_ROWSUM,
    KID_ZERO_EDGES,
    KID_MERGE,
    KID_COUNT
};
const char* kKernelNames[KID_COUNT] = {"k_ingest",   "k_compat",       "k_degree",      "k_heavy",       "k_rowclass",
                                       "k_expand",   "k_sc2_mma",      "k_emit_hh",     "k_sc2",         "k_sc2_light",   "k_hist_hi",     "k_hist_lo",     "k_alpha",       "k_collect",     "k_pivot_sort",
                                       "k_select_count", "k_select_scan", "k_select_emit", "k_pgs",
                                       "k_canon",    "k_kabsch",   "k_score",        "k_finalize",    "k_ransac_sample", "k_rowsum", "k_zero_edges", "k_split_merge"};
// stage of each kernel for turboreg_result.stage_ms: 0 graph (O2Graph construction), 1 PGS, 2 model
const int kKernelStage[KID_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 1, 0, 0, 2};

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline int words_per_row(int n) { return (int)round_up((n + 31) / 32, 4); }
// sparse-row list length for rows of W words: the SC^2 kernels' WPL = ceil(W/32) templates above 8 use the
// long lists (trk::list_max_of)
inline int list_cap(int64_t W) { return (W + 31) / 32 > 8 ? trk::LIST_MAX_BIG : trk::LIST_MAX; }
constexpr int HEAVY_CAP_MAX = 2048;
constexpr int NCHUNK = 8;  // sub-batches of a pipelined host-input call (sizes doubling: 1, 2, 4, .. 128 / 255)


}  // namespace

struct turboreg_ctx {
    turboreg_params prm{};
    int device = 0;
    int32_t max_n = 0, max_batch = 0, Wmax = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // H2D of pipelined host-input sub-batches
    cudaStream_t side_stream = nullptr;  // the sparse-row SC^2 kernel, concurrent with the dense-row one
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool use_fork = true;
    int32_t ransac_iters = 0;       // > 0 while turboreg_ransac runs: the RUN_RANSAC path
    unsigned long long ransac_seed = 0;
    cudaEvent_t ev_start = nullptr, ev_chunk[NCHUNK] = {};
    bool use_chunks = true;
    // device workspace
    void* d_base = nullptr;
    size_t ws_bytes = 0;
    trk::WS ws{};
    trk::PairDesc* d_desc = nullptr;
    void* d_results = nullptr;
    float* d_inputs = nullptr;  // staging for host inputs: 2 × max_batch × max_n × 3 floats
    int* d_counters = nullptr;  // per-call work-queue counters
    // pinned host staging: a ring of NDESC descriptor slots, each reusable once the event recorded after
    // its H2D copy has completed (an asynchronous call must not see its descriptors overwritten)
    static constexpr int NDESC = 4;
    trk::PairDesc* h_desc = nullptr;  // NDESC × max_batch
    cudaEvent_t ev_desc[NDESC] = {};
    int desc_slot = 0;
    // completion of the last call on whatever stream it ran: the next call's stream waits on it before it
    // touches the shared workspace
    cudaEvent_t ev_done = nullptr;
    // per-pair O2 edge capacity (words) and the layout choices the allocation was made for
    int64_t edge_cap = 0;
    bool alloc_fp4 = true, alloc_D = false;
    // point_resolution's and the ranking's own device buffers (grown on demand; independent of max_n)
    void* pr_buf = nullptr;
    size_t pr_bytes = 0;
    void* rank_buf = nullptr;
    size_t rank_bytes = 0;
    int32_t* d_rowsum = nullptr;  // [max_batch][max_n] r_i (TURBOREG_F_ROW_SUMS)
    int32_t split_rank = 0, split_world = 1;  // NEXT(1): this context's share of a split pair (1 = no split)
    turboreg_result* h_results = nullptr;
    float* h_inputs = nullptr;
    // bookkeeping of the last call
    int32_t last_batch = 0;
    std::vector<int32_t> last_n;
    // timing
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<int> ev_kid;
    double k_ms[KID_COUNT] = {0};
    int64_t k_launches[KID_COUNT] = {0};
    int64_t launches = 0;
    // CUDA graphs of the launch sequence, one per (batch, max n, mode); dropped whenever ws changes
    struct GraphEntry {
        int32_t batch, maxn, mode, p0, phase;
        cudaGraphExec_t exec;
        std::vector<int> kids;
    };
    std::vector<GraphEntry> graphs;
    bool use_graphs = true;
    // SC^2 heavy/light split
    int32_t heavy_cap_alloc = 0;
    CUtensorMap tmX, tmX4;  // X as uint8 rows / as packed e2m1 rows (half the bytes)
    bool tmX_ok = false, tmX4_ok = false;
    int32_t opt_mma_fp4 = 1;  // block-scaled fp4 dense block (default); 0 = kind::i8
    int32_t opt_compat_variant = 0, opt_sc2_path = 0, opt_heavy_min_rows = 128, opt_heavy_min_deg = 32, opt_heavy_cap = 0;
    int num_sms = 148;
    int32_t opt_score_pairs = 2;
    int32_t opt_sc2_chunks = 0;  // 0 = auto
    int32_t opt_mma_l2 = 1;      // L2 policy of the tensor-core block's X loads (WS::mma_l2)
    int32_t opt_heavy_widen = 1;  // WS::heavy_widen
};

namespace {

turboreg_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return TURBOREG_OK;
    if (e == cudaErrorMemoryAllocation) return TURBOREG_ERR_OUT_OF_MEMORY;
    return TURBOREG_ERR_CUDA;
}
#define CK(x)                                                       \
    do {                                                            \
        cudaError_t e__ = (x);                                      \
        if (e__ != cudaSuccess) {                                   \
            if (std::getenv("TURBOREG_DEBUG"))                      \
                std::fprintf(stderr, "turboreg: %s at %s:%d\n",     \
                             cudaGetErrorString(e__), __FILE__, __LINE__); \
            return cuda_status(e__);                                \
        }                                                           \
    } while (0)

bool params_valid(const turboreg_params* p) {
    if (!p) return false;
    if (!(p->tau > 0.f) || !std::isfinite(p->tau)) return false;
    if (!(p->tau_base == 0.f || (p->tau_base >= p->tau && std::isfinite(p->tau_base)))) return false;
    if (p->k1 < 1 || p->k2 < 1) return false;
    if ((int64_t)p->k1 * p->k2 > (int64_t)1 << 30) return false;
    if (!(p->inlier_threshold > 0.f) || !std::isfinite(p->inlier_threshold)) return false;
    if (p->graph_mode != 0 && p->graph_mode != 1) return false;
    if (p->graph_mode == 1 && (int64_t)p->k1 * p->k2 > trk::CANON_CAP) return false;  // canonical sort in smem
    if (p->flags & ~(TURBOREG_F_STAGE_TIMING | TURBOREG_F_KERNEL_TIMING | TURBOREG_F_HYP_ERRORS | TURBOREG_F_RANK_MAE |
                     TURBOREG_F_RANK_MSE | TURBOREG_F_ROW_SUMS))
        return false;
    if ((p->flags & TURBOREG_F_RANK_MAE) && (p->flags & TURBOREG_F_RANK_MSE)) return false;
    return true;
}

void drop_graphs(turboreg_ctx* c) {
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
}

void free_ws(turboreg_ctx* c) {
    drop_graphs(c);
    if (c->d_base) cudaFree(c->d_base);
    c->d_base = nullptr;
    c->ws_bytes = 0;
}

// Layout of X: packed e2m1 rows (16 W bytes, rounded to the 128-byte K block) unless the dense block runs
// as kind::i8 or on the CUDA cores (uint8 rows, 32 W bytes).
bool want_fp4_layout(const turboreg_ctx* c) { return c->opt_sc2_path != 2 && c->opt_mma_fp4; }
bool want_D(const turboreg_ctx* c) { return c->opt_sc2_path == 2; }  // D only on the __dp4a cross-check path
// per-hypothesis error sums only when MAE/MSE are asked for (reading r20)
bool want_err(const turboreg_params& p) {
    return (p.flags & (TURBOREG_F_HYP_ERRORS | TURBOREG_F_RANK_MAE | TURBOREG_F_RANK_MSE)) != 0;
}

// Carve one allocation into the per-pair arrays (sizes by max_n, max_batch, K1*K2, the edge capacity and
// the X layout).  The new allocation is made before the old one is released: on failure the context keeps
// its previous workspace (and parameters) intact.
turboreg_status alloc_ws(turboreg_ctx* c) {
    const int64_t B = c->max_batch, N = c->max_n, W = c->Wmax;
    const int64_t K1 = c->prm.k1, KC = (int64_t)c->prm.k1 * c->prm.k2;
    const bool base = c->prm.tau_base > 0.f;
    const bool fp4 = want_fp4_layout(c), withD = want_D(c);
    struct Item { size_t bytes; void** dst; };
    trk::WS w = c->ws;
    w.pts_stride = round_up(N, 32);  // even, so the paired arrays (stride / 2) stay 16-byte aligned
    w.bits_stride = N * W;
    w.row_stride = N;
    w.edges_stride = round_up(std::max<int64_t>(1, c->edge_cap), 4);  // uint4-aligned per pair
    w.piv_stride = K1;
    w.cl_stride = KC;
    void* p_desc; void* p_st; void* p_src4; void* p_dst4; void* p_bits; void* p_bitsb = nullptr; void* p_deg;
    void* p_gt; void* p_eq; void* p_take; void* p_off; void* p_edges; void* p_piv; void* p_cl; void* p_hyp;
    void* p_res; void* p_in; void* p_degf; void* p_hpos; void* p_X; void* p_D; void* p_hl; void* p_hm; void* p_lm; void* p_up; void* p_upre = nullptr; void* p_herr; void* p_ctr; void* p_lists; void* p_ll; void* p_dl; void* p_cand; void* p_rp; void* p_rs; void* p_tt;
    const int64_t cap = c->heavy_cap_alloc, Kcap = fp4 ? round_up((int64_t)W * 16, trk::MMA_BK) : (int64_t)W * 32;
    std::vector<Item> items = {
        {sizeof(trk::PairDesc) * B, &p_desc},
        {sizeof(trk::PairState) * B, &p_st},
        {sizeof(float4) * w.pts_stride * B, &p_src4},
        {sizeof(float4) * w.pts_stride * B, &p_dst4},
        {sizeof(uint32_t) * N * W * B, &p_bits},
        {sizeof(int32_t) * N * B, &p_deg},
        {sizeof(int32_t) * N * B, &p_gt},
        {sizeof(int32_t) * N * B, &p_eq},
        {sizeof(int32_t) * N * B, &p_take},
        {sizeof(int32_t) * N * B, &p_off},
        {sizeof(uint32_t) * (size_t)w.edges_stride * B, &p_edges},
        {sizeof(int4) * K1 * B, &p_piv},
        {sizeof(int4) * KC * B, &p_cl},
        {sizeof(float) * 16 * KC * B, &p_hyp},
        {sizeof(turboreg_result) * B, &p_res},
        {sizeof(float) * 6 * N * B, &p_in},
        {sizeof(int32_t) * N * B, &p_degf},
        {sizeof(int32_t) * N * B, &p_hpos},
        {(size_t)(cap * Kcap * B), &p_X},
        {withD ? sizeof(uint16_t) * (size_t)(cap * cap * B) : 0, &p_D},
        {sizeof(int32_t) * (size_t)(cap * B), &p_hl},
        {sizeof(uint32_t) * (size_t)(W * B), &p_hm},
        {sizeof(uint32_t) * (size_t)(W * B), &p_lm},
        {want_err(c->prm) ? sizeof(double2) * (size_t)(KC * trk::SCORE_SEGS_MAX * B) : 0, &p_herr},
        {sizeof(uint2) * (size_t)(cap * W * B), &p_up},
        {sizeof(int) * 16, &p_ctr},
        {sizeof(uint16_t) * (size_t)(N * list_cap(W) * B), &p_lists},
        {sizeof(int32_t) * (size_t)(N * B), &p_ll},
        {sizeof(int32_t) * (size_t)(N * B), &p_dl},
        {sizeof(unsigned long long) * (size_t)(trk::PIV_CAP * B), &p_cand},
        {sizeof(int32_t) * (size_t)((N + 1) * B), &p_rp},
        {sizeof(int32_t) * (size_t)(N * B), &p_rs},
        {sizeof(int32_t) * (size_t)(2 * B + 2), &p_tt},
    };
    if (base) items.push_back({sizeof(uint32_t) * N * W * B, &p_bitsb});
    if (c->prm.graph_mode == 1) items.push_back({sizeof(uint16_t) * N * W * B, &p_upre});
    size_t total = 0;
    for (auto& it : items) total += round_up((int64_t)it.bytes, 256);
    void* basep = nullptr;
    CK(cudaSetDevice(c->device));
    CK(cudaMalloc(&basep, total));
    char* cur = static_cast<char*>(basep);
    for (auto& it : items) {
        *it.dst = cur;
        cur += round_up((int64_t)it.bytes, 256);
    }
    free_ws(c);  // the old workspace (if any) goes only now that the new one exists
    c->d_base = basep;
    c->ws_bytes = total;
    c->alloc_fp4 = fp4;
    c->alloc_D = withD;
    c->d_desc = static_cast<trk::PairDesc*>(p_desc);
    w.desc = c->d_desc;
    w.st = static_cast<trk::PairState*>(p_st);
    w.src4 = static_cast<float4*>(p_src4);
    w.dst4 = static_cast<float4*>(p_dst4);
    w.bits = static_cast<uint32_t*>(p_bits);
    w.bits_base = static_cast<uint32_t*>(p_bitsb);
    w.deg = static_cast<int32_t*>(p_deg);
    w.row_gt = static_cast<int32_t*>(p_gt);
    w.row_eq = static_cast<int32_t*>(p_eq);
    w.row_take = static_cast<int32_t*>(p_take);
    w.row_off = static_cast<int32_t*>(p_off);
    w.edges = static_cast<uint32_t*>(p_edges);
    w.piv = static_cast<int4*>(p_piv);
    w.cliq = static_cast<int4*>(p_cl);
    w.hyp = static_cast<float*>(p_hyp);
    w.res = p_res;
    c->d_results = p_res;
    c->d_inputs = static_cast<float*>(p_in);
    w.deg_full = static_cast<int32_t*>(p_degf);
    w.hpos = static_cast<int32_t*>(p_hpos);
    w.heavy_X = static_cast<uint8_t*>(p_X);
    w.heavy_X_stride = cap * Kcap;
    w.heavy_Kcap = (int32_t)Kcap;
    w.heavy_D = withD ? static_cast<uint16_t*>(p_D) : nullptr;
    w.heavy_D_stride = cap * cap;
    w.heavy_list = static_cast<int32_t*>(p_hl);
    w.tile_tab = static_cast<int32_t*>(p_tt);
    w.tile_ctr = w.tile_tab + 2 * B + 1;
    w.heavy_mask = static_cast<uint32_t*>(p_hm);
    w.light_mask = static_cast<uint32_t*>(p_lm);
    w.heavy_UP = static_cast<uint2*>(p_up);
    w.uprefix = static_cast<uint16_t*>(p_upre);
    w.herr = want_err(c->prm) ? static_cast<double2*>(p_herr) : nullptr;
    w.heavy_UP_stride = cap * W;
    c->d_counters = static_cast<int*>(p_ctr);
    c->d_rowsum = static_cast<int32_t*>(p_rs);
    w.lists = static_cast<uint16_t*>(p_lists);
    w.lists_stride = N * list_cap(W);
    w.light_list = static_cast<int32_t*>(p_ll);
    w.cand = static_cast<unsigned long long*>(p_cand);
    w.rowptr = static_cast<int32_t*>(p_rp);
    w.rp_stride = N + 1;
    w.dense_list = static_cast<int32_t*>(p_dl);
    c->ws = w;
    // TMA descriptor over X as a 3-D uint8 tensor [batch][cap][Kcap], 128×128 boxes, 128B swizzle (the
    // uint8 map when X holds uint8 rows, the e2m1 map when it holds packed rows)
    c->tmX_ok = false;
    c->tmX4_ok = false;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && encode) {
        const cuuint64_t dims[3] = {(cuuint64_t)Kcap, (cuuint64_t)cap, (cuuint64_t)B};
        const cuuint64_t strides[2] = {(cuuint64_t)Kcap, (cuuint64_t)(Kcap * cap)};
        const cuuint32_t box[3] = {trk::MMA_BK, trk::MMA_BM, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = encode(fp4 ? &c->tmX4 : &c->tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, p_X, dims, strides, box,
                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        (fp4 ? c->tmX4_ok : c->tmX_ok) = (r == CUDA_SUCCESS);
    }
    cudaGetLastError();
    return TURBOREG_OK;
}

void set_ws_params(turboreg_ctx* c) {
    drop_graphs(c);  // captured launches hold ws by value
    c->ws.heavy_cap = c->opt_heavy_cap > 0 ? std::min(c->opt_heavy_cap, c->heavy_cap_alloc) : c->heavy_cap_alloc;
    c->ws.heavy_min_rows = c->opt_heavy_min_rows;
    c->ws.heavy_min_deg = c->opt_heavy_min_deg;
    // the tensor-core block needs the tensor map of the layout X was allocated in; without it, popcount only
    c->ws.sc2_path = (c->opt_sc2_path == 0 && !(c->alloc_fp4 ? c->tmX4_ok : c->tmX_ok)) ? 1 : c->opt_sc2_path;
    c->ws.x_fp4 = (c->ws.sc2_path == 0 && c->alloc_fp4) ? 1 : 0;
    c->ws.mma_l2 = c->opt_mma_l2;
    c->ws.heavy_widen = c->opt_heavy_widen;
    c->ws.tau = c->prm.tau;
    c->ws.tau_base = c->prm.tau_base;
    c->ws.thr = c->prm.inlier_threshold;
    c->ws.k1 = c->prm.k1;
    c->ws.k2 = c->prm.k2;
    c->ws.mode = c->prm.graph_mode;
    c->ws.split_rank = 0;
    c->ws.split_world = 1;
    c->ws.compat_b0 = 0;
    {
        const int rank = (c->prm.flags & TURBOREG_F_RANK_MAE) ? 1 : (c->prm.flags & TURBOREG_F_RANK_MSE) ? 2 : 0;
        c->ws.err_mode = ((rank || (c->prm.flags & TURBOREG_F_HYP_ERRORS)) ? 1 : 0) | (rank << 1);
    }
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Next free descriptor slot of the pinned ring: waits until the H2D copy that last read it has run, so an
// asynchronous call's descriptors are never overwritten before the device has them.
trk::PairDesc* next_desc(turboreg_ctx* c, int* slot) {
    const int k = c->desc_slot;
    c->desc_slot = (k + 1) % turboreg_ctx::NDESC;
    cudaEventSynchronize(c->ev_desc[k]);
    *slot = k;
    return c->h_desc + (size_t)k * c->max_batch;
}

// Every call starts by making its stream wait for the previous call's completion (the workspace is shared,
// whatever stream either call ran on) and ends by recording its own.
cudaError_t begin_call(turboreg_ctx* c, cudaStream_t s) { return cudaStreamWaitEvent(s, c->ev_done, 0); }
cudaError_t end_call(turboreg_ctx* c, cudaStream_t s) { return cudaEventRecord(c->ev_done, s); }

// --------------------------------------------------------------------------------- launch sequencing
struct Launcher {
    turboreg_ctx* c;
    cudaStream_t s;
    bool timed;
    cudaEvent_t ev() {
        if (c->ev_used == c->ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            c->ev_pool.push_back(e);
        }
        return c->ev_pool[c->ev_used++];
    }
    template <typename F>
    cudaError_t run(int kid, F&& f) {
        cudaEvent_t a = nullptr, b = nullptr;
        if (timed) { a = ev(); b = ev(); cudaEventRecord(a, s); }
        f();
        cudaError_t e = cudaGetLastError();
        if (timed) { cudaEventRecord(b, s); c->ev_kid.push_back(kid); }
        c->launches++;
        c->k_launches[kid]++;
        return e;
    }
};

// Fold the recorded event pairs into the per-kernel accumulators (synchronises on the events).
void harvest_events(turboreg_ctx* c, float* stage_ms) {
    for (size_t k = 0; k < c->ev_kid.size(); ++k) {
        float ms = 0.f;
        cudaEventSynchronize(c->ev_pool[2 * k + 1]);
        cudaEventElapsedTime(&ms, c->ev_pool[2 * k], c->ev_pool[2 * k + 1]);
        c->k_ms[c->ev_kid[k]] += ms;
        if (stage_ms) stage_ms[kKernelStage[c->ev_kid[k]]] += ms;
    }
    c->ev_kid.clear();
    c->ev_used = 0;
}

enum RunMode { RUN_FULL = 0, RUN_FROM_ADJ = 1, RUN_RANSAC = 2 };

// phase (bit set): PH_HEAD = state reset + ingest + compat (per pipelined sub-batch); PH_GRAPH = degrees, row
// classes and the SC^2 assembly; PH_SEARCH = pivots, PGS, Kabsch, scoring, argmax.  PH_TAIL = everything after
// compat.  A split pair (NEXT(1)) runs the three separately, with an exchange between them.
enum Phase { PH_HEAD = 1, PH_GRAPH = 2, PH_SEARCH = 4, PH_TAIL = 6, PH_ALL = 7 };

turboreg_status launch_all(turboreg_ctx* c, int32_t batch, int32_t maxn_batch, cudaStream_t s, RunMode mode,
                           int32_t p0 = 0, int phase = PH_ALL) {
    trk::WS ws = p0 ? trk::ws_view(c->ws, p0, sizeof(turboreg_result)) : c->ws;
    ws.split_rank = c->split_rank;
    ws.split_world = c->split_world;
    const bool splitp = c->split_world > 1;
    const bool timed = c->profiling || (c->prm.flags & TURBOREG_F_STAGE_TIMING);
    Launcher L{c, s, timed};
    const int Wb = words_per_row(std::max(maxn_batch, 1));
    const unsigned B = (unsigned)batch;
    if (phase & PH_HEAD) {
        CK(cudaMemsetAsync(ws.st, 0, sizeof(trk::PairState) * batch, s));
        CK(cudaMemsetAsync(c->d_counters, 0, sizeof(int) * 16, s));
    }
    if (mode == RUN_RANSAC) {  // NEXT(4): ingest, sampled triples, then the model stage on them
        CK(L.run(KID_INGEST, [&] {
            trk::k_ingest<<<dim3((maxn_batch + 255) / 256, B), 256, 0, s>>>(ws);
        }));
        trk::WS wr = ws;
        wr.k1 = c->ransac_iters;
        wr.k2 = 1;
        wr.err_mode = 0;  // inlier-number ranking
        const int64_t KC = c->ransac_iters;
        CK(L.run(KID_RANSAC, [&] {
            trk::k_ransac_sample<<<dim3((unsigned)((KC + 255) / 256), B), 256, 0, s>>>(wr, c->ransac_seed);
        }));
        CK(L.run(KID_KABSCH, [&] { trk::k_kabsch<<<dim3((unsigned)((KC + 127) / 128), B), 128, 0, s>>>(wr); }));
        CK(L.run(KID_SCORE, [&] {
            const int npk = c->opt_score_pairs;
            const int hb = (int)((KC + trk::SCORE_HT * npk - 1) / (trk::SCORE_HT * npk));
            const int segs = std::max(2, std::min(16, (7 * c->num_sms + hb * batch - 1) / (hb * batch)));
            const dim3 g((unsigned)(hb * segs), B);
            if (npk == 2) trk::k_score<false, 2><<<g, trk::SCORE_THREADS, 0, s>>>(wr, segs);
            else trk::k_score<false, 1><<<g, trk::SCORE_THREADS, 0, s>>>(wr, segs);
        }));
        CK(L.run(KID_FINALIZE, [&] { trk::k_finalize<<<B, 1024, 0, s>>>(wr); }));
        return TURBOREG_OK;
    }
    if (mode == RUN_FULL && (phase & PH_HEAD)) {
        CK(L.run(KID_INGEST, [&] {
            trk::k_ingest<<<dim3((maxn_batch + 255) / 256, B), 256, 0, s>>>(ws);
        }));
        const int T = (maxn_batch + 31) / 32;
        // small batches: several blocks share a block-row pair so the grid still covers ~2 waves; a split pair
        // computes only this rank's block-row pairs, into a zeroed bit matrix (the ranks' matrices are summed)
        int bpp = (T + 1) / 2;
        if (splitp) {
            const int b0 = (int)((int64_t)c->split_rank * bpp / c->split_world);
            const int b1 = (int)((int64_t)(c->split_rank + 1) * bpp / c->split_world);
            ws.compat_b0 = b0;
            bpp = std::max(b1 - b0, 0);
            CK(cudaMemsetAsync(ws.bits, 0, sizeof(uint32_t) * (size_t)ws.bits_stride * batch, s));
        }
        const int split = std::max(1, std::min(16, (5 * c->num_sms + std::max(bpp, 1) * batch - 1) / (std::max(bpp, 1) * batch)));
        if (bpp > 0) CK(L.run(KID_COMPAT, [&] {
            const dim3 g((unsigned)(bpp * split), B);
            if (c->prm.tau_base > 0.f) trk::k_compat<true><<<g, 256, 0, s>>>(ws, split);
            else if (c->opt_compat_variant == 1) trk::k_compat<false, 5, 16, 1><<<g, 256, 0, s>>>(ws, split);
            else if (c->opt_compat_variant == 2) trk::k_compat<false, 5, 16, -1><<<g, 256, 0, s>>>(ws, split);
            else trk::k_compat<false, 4, 16, -2><<<g, 256, 0, s>>>(ws, split);
        }));
    }
    if (!(phase & PH_TAIL)) return TURBOREG_OK;
    ws.list_max = list_cap(Wb);
    if (phase & PH_GRAPH) {
    const int deg_rows = batch >= 256 ? trk::DEG_ROWS_PER_BLOCK_BIG : trk::DEG_ROWS_PER_BLOCK;
    const dim3 grow((maxn_batch + deg_rows - 1) / deg_rows, B);
    CK(L.run(KID_DEGREE, [&] { trk::k_degree<<<grow, 256, 0, s>>>(ws, deg_rows); }));
    CK(L.run(KID_HEAVY, [&] { trk::k_heavy<<<B, 1024, 0, s>>>(ws); }));
    CK(L.run(KID_ROWCLASS, [&] { trk::k_rowclass<<<B, 1024, 0, s>>>(ws); }));
#ifdef TRK_CHECKS
    const bool zero_edges = true;  // the checked build verifies every slot was written
#else
    const bool zero_edges = splitp;
#endif
    if (zero_edges) CK(L.run(KID_ZERO_EDGES, [&] { trk::k_zero_edges<<<dim3(2 * c->num_sms, B), 256, 0, s>>>(ws); }));
    if (ws.sc2_path != 1) {
        CK(L.run(KID_EXPAND, [&] {
            const dim3 ge((unsigned)(ws.heavy_X_stride / ws.heavy_Kcap / 8), B);
            if (ws.x_fp4) trk::k_expand<true><<<ge, 256, 0, s>>>(ws);
            else trk::k_expand<false><<<ge, 256, 0, s>>>(ws);
        }));
        if (ws.sc2_path == 2) {
            CK(L.run(KID_SC2_MMA, [&] {
                const unsigned g = (unsigned)(ws.heavy_cap / 64);
                trk::k_sc2_dp4a<<<dim3(g, g, B), 256, 0, s>>>(ws);
            }));
            CK(L.run(KID_EMIT_HH, [&] {
                trk::k_emit_hh<<<dim3((unsigned)(ws.heavy_cap / 8), B), 256, 0, s>>>(ws);
            }));
        } else {
            if (batch > trk::MMA_TABLE_PAIRS) {
                trk::k_tile_table<<<1, 1024, 0, s>>>(ws, batch, ws.x_fp4 ? 240 : trk::MMA_BN);
                CK(cudaGetLastError());
            }
            CK(cudaMemsetAsync(ws.tile_ctr, 0, sizeof(int32_t), s));
            CK(L.run(KID_SC2_MMA, [&] {
                if (ws.x_fp4) trk::k_sc2_mma<true><<<c->num_sms, trk::MMA_THREADS, trk::MMA_SMEM_BYTES, s>>>(c->tmX4, ws, B);
                else trk::k_sc2_mma<false><<<c->num_sms, trk::MMA_THREADS, trk::MMA_SMEM_BYTES, s>>>(c->tmX, ws, B);
            }));
        }
    }
    const int wpl = (Wb + 31) / 32;
    {
        const int sc2_bpp = std::max(batch >= 128 ? trk::SC2_BLOCKS_PER_PAIR_BIG : trk::SC2_BLOCKS_PER_PAIR,
                                     std::min((3 * c->num_sms + batch - 1) / batch, (maxn_batch + 7) / 8));
        const dim3 gp((unsigned)sc2_bpp, B);
        // chunks per item: whole rows for batches; 4 chunks (128 words) for large N, where one pair has
        // thousands of dense rows and a single-chunk item would re-stage its row W/32 times; else one chunk
        const int cpi = c->opt_sc2_chunks > 0 ? c->opt_sc2_chunks : (batch >= 32 ? 64 : Wb > 512 ? 4 : 1);
        // the sparse-row kernel needs only the row classes and lists: it runs on the side stream while the
        // dense-row kernel runs here (both are latency-bound; timed calls keep one stream for the events)
        const bool fork = c->use_fork && !timed;
        cudaStream_t sl = fork ? c->side_stream : s;
        if (fork) {
            CK(cudaEventRecord(c->ev_fork, s));
            CK(cudaStreamWaitEvent(sl, c->ev_fork, 0));
        }
        CK(L.run(KID_SC2, [&] {
            if (wpl <= 1) trk::k_sc2<1><<<gp, 256, trk::sc2_smem_bytes<1>(), s>>>(ws, cpi);
            else if (wpl <= 2) trk::k_sc2<2><<<gp, 256, trk::sc2_smem_bytes<2>(), s>>>(ws, cpi);
            else if (wpl <= 4) trk::k_sc2<4><<<gp, 256, trk::sc2_smem_bytes<4>(), s>>>(ws, cpi);
            else if (wpl <= 5) trk::k_sc2<5><<<gp, 256, trk::sc2_smem_bytes<5>(), s>>>(ws, cpi);
            else if (wpl <= 8) trk::k_sc2<8><<<gp, 256, trk::sc2_smem_bytes<8>(), s>>>(ws, cpi);
            else if (wpl <= 16) trk::k_sc2<16><<<gp, 256, trk::sc2_smem_bytes<16>(), s>>>(ws, cpi);
            else trk::k_sc2<32><<<gp, 256, trk::sc2_smem_bytes<32>(), s>>>(ws, cpi);
        }));
        // rows per warp group: light_rows<WPL>() of the rounded-up WPL, or 2 when that grid would not give
        // every SM two blocks (small batches)
        const int lg_def = wpl > 8 ? trk::light_rows<16>() : trk::light_rows<8>();
        const bool lg_small = lg_def > 2 && (int64_t)((maxn_batch + 8 * lg_def - 1) / (8 * lg_def)) * batch < 2 * c->num_sms;
        const int lgr = lg_small ? 2 : lg_def;
        const dim3 gl((unsigned)((maxn_batch + 8 * lgr - 1) / (8 * lgr)), B);
        CK(L.run(KID_SC2_LIGHT, [&] {
            if (lg_small) {
                if (wpl <= 1) trk::k_sc2_light<1, 2><<<gl, 256, trk::light_smem_bytes<1, 2>(), sl>>>(ws);
                else if (wpl <= 2) trk::k_sc2_light<2, 2><<<gl, 256, trk::light_smem_bytes<2, 2>(), sl>>>(ws);
                else if (wpl <= 4) trk::k_sc2_light<4, 2><<<gl, 256, trk::light_smem_bytes<4, 2>(), sl>>>(ws);
                else if (wpl <= 5) trk::k_sc2_light<5, 2><<<gl, 256, trk::light_smem_bytes<5, 2>(), sl>>>(ws);
                else trk::k_sc2_light<8, 2><<<gl, 256, trk::light_smem_bytes<8, 2>(), sl>>>(ws);
            } else if (wpl <= 1) trk::k_sc2_light<1><<<gl, 256, trk::light_smem_bytes<1>(), sl>>>(ws);
            else if (wpl <= 2) trk::k_sc2_light<2><<<gl, 256, trk::light_smem_bytes<2>(), sl>>>(ws);
            else if (wpl <= 4) trk::k_sc2_light<4><<<gl, 256, trk::light_smem_bytes<4>(), sl>>>(ws);
            else if (wpl <= 5) trk::k_sc2_light<5><<<gl, 256, trk::light_smem_bytes<5>(), sl>>>(ws);
            else if (wpl <= 8) trk::k_sc2_light<8><<<gl, 256, trk::light_smem_bytes<8>(), sl>>>(ws);
            else if (wpl <= 16) trk::k_sc2_light<16><<<gl, 256, trk::light_smem_bytes<16>(), sl>>>(ws);
            else trk::k_sc2_light<32><<<gl, 256, trk::light_smem_bytes<32>(), sl>>>(ws);
        }));
        if (fork) {
            CK(cudaEventRecord(c->ev_join, sl));
            CK(cudaStreamWaitEvent(s, c->ev_join, 0));
        }
    }
    if (c->prm.flags & TURBOREG_F_ROW_SUMS) {  // r_i = Σ_j Ĝ_ij (App. B), beside the path
        int32_t* rs = c->d_rowsum + (int64_t)p0 * c->max_n;
        CK(cudaMemsetAsync(rs, 0, sizeof(int32_t) * (size_t)c->max_n * batch, s));
        CK(L.run(KID_ROWSUM, [&] {
            trk::k_rowsum<<<dim3((unsigned)((maxn_batch + 63) / 64), B), 256, 0, s>>>(ws, rs, c->max_n);
        }));
    }
#ifdef TRK_CHECKS
    if (!splitp) {
        trk::k_check_edges<<<dim3((maxn_batch + 7) / 8, B), 256, 0, s>>>(ws);
        CK(cudaGetLastError());
    }
#endif
    }  // PH_GRAPH
    if (!(phase & PH_SEARCH)) return TURBOREG_OK;
#ifdef TRK_CHECKS
    if (splitp) {  // a split pair's edges are complete only after the exchange
        trk::k_check_edges<<<dim3((maxn_batch + 7) / 8, B), 256, 0, s>>>(ws);
        CK(cudaGetLastError());
    }
#endif
    const dim3 gsel((maxn_batch + trk::SEL_ROWS_PER_BLOCK - 1) / trk::SEL_ROWS_PER_BLOCK, B);
    const int sel_bpp = std::max(trk::SEL_BLOCKS_PER_PAIR, std::min((4 * c->num_sms + batch - 1) / batch, 256));
    const dim3 gflat((unsigned)sel_bpp, B);
    CK(L.run(KID_HIST_HI, [&] { trk::k_hist_hi<<<gflat, 256, 0, s>>>(ws); }));
    CK(L.run(KID_HIST_LO, [&] { trk::k_hist_lo<<<gflat, 256, 0, s>>>(ws); }));
    CK(L.run(KID_ALPHA, [&] { trk::k_alpha<<<B, 256, 0, s>>>(ws); }));
    CK(L.run(KID_COLLECT, [&] { trk::k_collect<<<gflat, 256, 0, s>>>(ws); }));
    CK(L.run(KID_PIVOT_SORT, [&] {
        trk::k_pivot_sort<<<B, 1024, trk::PIV_CAP * sizeof(unsigned long long) + trk::SORT_RP_CAP * sizeof(int32_t), s>>>(ws);
    }));
    CK(L.run(KID_SEL_COUNT, [&] { trk::k_select_count<<<gsel, 256, 0, s>>>(ws); }));
    CK(L.run(KID_SEL_SCAN, [&] { trk::k_select_scan<<<B, 1024, 0, s>>>(ws); }));
    CK(L.run(KID_SEL_EMIT, [&] { trk::k_select_emit<<<gsel, 256, 0, s>>>(ws); }));
    CK(L.run(KID_PGS, [&] {
        const dim3 g((c->prm.k1 + trk::PGS_WARPS - 1) / trk::PGS_WARPS, B);
        const int k2 = c->prm.k2, bt = trk::PGS_WARPS * 32;
        if (c->prm.graph_mode == 1) {
            if (k2 <= 2) trk::k_pgs<1, 2><<<g, bt, 0, s>>>(ws);
            else if (k2 <= 4) trk::k_pgs<1, 4><<<g, bt, 0, s>>>(ws);
            else if (k2 <= trk::PGS_KL) trk::k_pgs<1, trk::PGS_KL><<<g, bt, 0, s>>>(ws);
            else trk::k_pgs<1, 0><<<g, bt, 0, s>>>(ws);
        } else {
            if (k2 <= 2) trk::k_pgs<0, 2><<<g, bt, 0, s>>>(ws);
            else if (k2 <= 4) trk::k_pgs<0, 4><<<g, bt, 0, s>>>(ws);
            else if (k2 <= trk::PGS_KL) trk::k_pgs<0, trk::PGS_KL><<<g, bt, 0, s>>>(ws);
            else trk::k_pgs<0, 0><<<g, bt, 0, s>>>(ws);
        }
    }));
#ifdef TRK_CHECKS
    if (mode != RUN_RANSAC) {
        trk::k_check_cliques<<<dim3(8, B), 256, 0, s>>>(ws);
        CK(cudaGetLastError());
    }
#endif
    if (c->prm.graph_mode == 1) {  // canonical order + de-duplication of the SC^2-mode clique list (r9)
        int m2 = 1;
        while (m2 < c->prm.k1 * c->prm.k2) m2 <<= 1;
        CK(L.run(KID_CANON, [&] { trk::k_canon<<<B, 1024, sizeof(unsigned long long) * m2, s>>>(ws); }));
    }
    if (mode == RUN_FULL) {
        const int64_t KC = (int64_t)c->prm.k1 * c->prm.k2;
        if (ws.err_mode & 1)
            CK(cudaMemsetAsync(ws.herr, 0, sizeof(double2) * KC * trk::SCORE_SEGS_MAX * batch, s));
        CK(L.run(KID_KABSCH, [&] { trk::k_kabsch<<<dim3((unsigned)((KC + 127) / 128), B), 128, 0, s>>>(ws); }));
        CK(L.run(KID_SCORE, [&] {
            const int npk = c->opt_score_pairs;  // packed hypothesis pairs per thread
            const int hb = (int)((KC + trk::SCORE_HT * npk - 1) / (trk::SCORE_HT * npk));
            const int segs = std::max(2, std::min(16, (7 * c->num_sms + hb * batch - 1) / (hb * batch)));
            const dim3 g((unsigned)(hb * segs), B);
            if (ws.err_mode & 1) {
                if (npk == 2) trk::k_score<true, 2><<<g, trk::SCORE_THREADS, 0, s>>>(ws, segs);
                else trk::k_score<true, 1><<<g, trk::SCORE_THREADS, 0, s>>>(ws, segs);
            } else {
                if (npk == 2) trk::k_score<false, 2><<<g, trk::SCORE_THREADS, 0, s>>>(ws, segs);
                else trk::k_score<false, 1><<<g, trk::SCORE_THREADS, 0, s>>>(ws, segs);
            }
        }));
        CK(L.run(KID_FINALIZE, [&] { trk::k_finalize<<<B, 1024, 0, s>>>(ws); }));
    }
    return TURBOREG_OK;
}

// The launch sequence replayed from a CUDA graph (captured on first use of a (batch, max n, mode) shape):
// one graph launch instead of ~20 kernel launches, which is most of a single pair's latency.  Per-kernel
// timing needs the events between launches, so timed calls launch directly.
turboreg_status run_pipeline(turboreg_ctx* c, int32_t batch, int32_t maxn_batch, cudaStream_t s, RunMode mode,
                             int32_t p0 = 0, int phase = PH_ALL) {
    const bool timed = c->profiling || (c->prm.flags & TURBOREG_F_STAGE_TIMING);
    if (timed || !c->use_graphs || mode == RUN_RANSAC)  // RANSAC: iters / seed are launch arguments
        return launch_all(c, batch, maxn_batch, s, mode, p0, phase);
    turboreg_ctx::GraphEntry* ge = nullptr;
    for (auto& g : c->graphs)
        if (g.batch == batch && g.maxn == maxn_batch && g.mode == (int32_t)mode && g.p0 == p0 && g.phase == phase)
            ge = &g;
    if (!ge) {
        const int64_t l0 = c->launches;
        int64_t k0[KID_COUNT];
        std::memcpy(k0, c->k_launches, sizeof(k0));
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            return launch_all(c, batch, maxn_batch, s, mode, p0, phase);  // e.g. the legacy default stream
        }
        const turboreg_status st = launch_all(c, batch, maxn_batch, s, mode, p0, phase);
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(s, &g);
        c->launches = l0;
        turboreg_ctx::GraphEntry e{batch, maxn_batch, (int32_t)mode, p0, phase, nullptr, {}};
        for (int k = 0; k < KID_COUNT; ++k)
            for (int64_t r = k0[k]; r < c->k_launches[k]; ++r) e.kids.push_back(k);
        std::memcpy(c->k_launches, k0, sizeof(k0));
        if (st != TURBOREG_OK || ec != cudaSuccess || !g || cudaGraphInstantiate(&e.exec, g, 0) != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return st != TURBOREG_OK ? st : launch_all(c, batch, maxn_batch, s, mode, p0, phase);
        }
        cudaGraphDestroy(g);
        if (c->graphs.size() >= 16) drop_graphs(c);
        c->graphs.push_back(std::move(e));
        ge = &c->graphs.back();
    }
    CK(cudaGraphLaunch(ge->exec, s));
    c->launches += (int64_t)ge->kids.size();
    for (int k : ge->kids) c->k_launches[k]++;
    return TURBOREG_OK;
}

}  // namespace

extern "C" {

const char* turboreg_status_string(turboreg_status s) {
    switch (s) {
        case TURBOREG_OK: return "ok";
        case TURBOREG_ERR_INVALID_ARGUMENT: return "invalid argument";
        case TURBOREG_ERR_TOO_FEW_POINTS: return "too few points (N < 3)";
        case TURBOREG_ERR_TOO_MANY_POINTS: return "too many points (N > max_n)";
        case TURBOREG_ERR_NONFINITE_INPUT: return "non-finite input coordinate";
        case TURBOREG_ERR_NO_HYPOTHESIS: return "no hypothesis";
        case TURBOREG_ERR_CUDA: return "CUDA error";
        case TURBOREG_ERR_OUT_OF_MEMORY: return "out of device memory";
        case TURBOREG_ERR_EDGE_CAPACITY: return "edge capacity exceeded (more graph edges than max_edges)";
    }
    return "unknown status";
}

turboreg_status turboreg_create_ex(const turboreg_params* params, int device, int32_t max_n, int32_t max_batch,
                                   int64_t max_edges, turboreg_ctx** out) {
    if (!out || !params_valid(params) || max_n < 3 || max_n > 32768 || max_batch < 1 || max_batch > 65535 ||
        max_edges < 0)
        return TURBOREG_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    const int64_t full_edges = (int64_t)max_n * (max_n - 1) / 2;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return TURBOREG_ERR_CUDA;
    }
    turboreg_ctx* c = new (std::nothrow) turboreg_ctx();
    if (!c) return TURBOREG_ERR_OUT_OF_MEMORY;
    c->prm = *params;
    c->device = device;
    c->max_n = max_n;
    c->max_batch = max_batch;
    c->Wmax = words_per_row(max_n);
    // the tensor-core block holds up to 2048 heavy rows for max_n <= 8192 (config-E pairs: |H| ≈ 1250), and up
    // to half the rows beyond (large N: an inlier block of thousands of rows)
    const int64_t hcap = max_n <= 8192 ? HEAVY_CAP_MAX : round_up((max_n + 1) / 2, 256);
    c->heavy_cap_alloc = (int32_t)std::max<int64_t>(256, std::min<int64_t>(round_up(max_n, 256), hcap));
    c->edge_cap = (max_edges == 0 || max_edges > full_edges) ? full_edges : max_edges;
    turboreg_status st = TURBOREG_OK;
    // A blocking stream: it orders itself with the legacy default stream, so inputs produced there (e.g. by
    // torch's default stream) are complete before our kernels read them.
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreate(&c->own_stream) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming) != cudaSuccess) {
        st = TURBOREG_ERR_CUDA;
    }
    for (auto& e : c->ev_chunk)
        if (st == TURBOREG_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) st = TURBOREG_ERR_CUDA;
    for (auto& e : c->ev_desc)
        if (st == TURBOREG_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) st = TURBOREG_ERR_CUDA;
    if (st == TURBOREG_OK) cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (st == TURBOREG_OK) st = alloc_ws(c);
    if (st == TURBOREG_OK) {
        if (cudaMallocHost(&c->h_desc, sizeof(trk::PairDesc) * max_batch * turboreg_ctx::NDESC) != cudaSuccess ||
            cudaMallocHost(&c->h_results, sizeof(turboreg_result) * max_batch) != cudaSuccess)
            st = TURBOREG_ERR_OUT_OF_MEMORY;
    }
    if (st != TURBOREG_OK) {
        cudaGetLastError();
        turboreg_destroy(c);
        return st;
    }
    set_ws_params(c);
    if (cudaFuncSetAttribute(trk::k_sc2_mma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::MMA_SMEM_BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2_mma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::MMA_SMEM_BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_canon, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(unsigned long long) * trk::CANON_CAP)) != cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<1>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<2>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<4>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<5>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<8>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<16>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::sc2_smem_bytes<32>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_pivot_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             trk::PIV_CAP * (int)sizeof(unsigned long long) + trk::SORT_RP_CAP * 4) != cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2_light<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::light_smem_bytes<5>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2_light<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::light_smem_bytes<8>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2_light<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::light_smem_bytes<16>()) !=
            cudaSuccess ||
        cudaFuncSetAttribute(trk::k_sc2_light<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, trk::light_smem_bytes<32>()) !=
            cudaSuccess) {
        cudaGetLastError();
        turboreg_destroy(c);
        return TURBOREG_ERR_CUDA;
    }
    *out = c;
    return TURBOREG_OK;
}

turboreg_status turboreg_create(const turboreg_params* params, int device, int32_t max_n, int32_t max_batch,
                                turboreg_ctx** out) {
    return turboreg_create_ex(params, device, max_n, max_batch, 0, out);
}

turboreg_status turboreg_set_option(turboreg_ctx* c, const char* name, int64_t value) {
    if (!c || !name) return TURBOREG_ERR_INVALID_ARGUMENT;
    const std::string k(name);
    const int32_t old_sc2 = c->opt_sc2_path, old_fp4 = c->opt_mma_fp4;
    if (k == "sc2_path") {
        if (value < 0 || value > 2) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_sc2_path = (int32_t)value;
    } else if (k == "heavy_min_rows") {
        if (value < 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_heavy_min_rows = (int32_t)value;
    } else if (k == "heavy_min_degree") {
        if (value < 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_heavy_min_deg = (int32_t)value;
    } else if (k == "compat_variant") {
        if (value < 0 || value > 2) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_compat_variant = (int32_t)value;
    } else if (k == "pipeline_host_inputs") {
        if (value < 0 || value > 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->use_chunks = value != 0;
    } else if (k == "mma_fp4") {
        if (value < 0 || value > 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_mma_fp4 = (int32_t)value;
    } else if (k == "mma_l2_policy") {
        if (value < 0 || value > 2) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_mma_l2 = (int32_t)value;
        drop_graphs(c);  // captured launches hold the workspace descriptor by value
    } else if (k == "heavy_widen") {
        if (value < 0 || value > 65535) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_heavy_widen = (int32_t)value;
        drop_graphs(c);
    } else if (k == "sc2_chunks") {
        if (value < 0 || value > 64) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_sc2_chunks = (int32_t)value;
    } else if (k == "score_pairs") {
        if (value < 1 || value > 2) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_score_pairs = (int32_t)value;
    } else if (k == "concurrent_sc2") {
        if (value < 0 || value > 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->use_fork = value != 0;
    } else if (k == "cuda_graph") {
        if (value < 0 || value > 1) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->use_graphs = value != 0;
    } else if (k == "heavy_cap") {
        if (value < 0 || value % 256 || value > c->heavy_cap_alloc) return TURBOREG_ERR_INVALID_ARGUMENT;
        c->opt_heavy_cap = (int32_t)value;
    } else {
        return TURBOREG_ERR_INVALID_ARGUMENT;
    }
    if (want_fp4_layout(c) != c->alloc_fp4 || want_D(c) != c->alloc_D) {  // X / D layout changes: reallocate
        CK(cudaSetDevice(c->device));
        CK(cudaEventSynchronize(c->ev_done));
        drop_graphs(c);
        const turboreg_status st = alloc_ws(c);
        if (st != TURBOREG_OK) {  // keep the old workspace and the options it was laid out for
            c->opt_sc2_path = old_sc2;
            c->opt_mma_fp4 = old_fp4;
            set_ws_params(c);
            return st;
        }
    }
    set_ws_params(c);
    return TURBOREG_OK;
}

turboreg_status turboreg_set_params(turboreg_ctx* c, const turboreg_params* p) {
    if (!c || !params_valid(p)) return TURBOREG_ERR_INVALID_ARGUMENT;
    const bool realloc = (int64_t)p->k1 * p->k2 != (int64_t)c->prm.k1 * c->prm.k2 || p->k1 != c->prm.k1 ||
                         p->graph_mode != c->prm.graph_mode ||
                         ((p->tau_base > 0.f) != (c->prm.tau_base > 0.f)) || want_err(*p) != want_err(c->prm);
    CK(cudaSetDevice(c->device));
    const turboreg_params old = c->prm;
    c->prm = *p;
    if (realloc) {
        CK(cudaEventSynchronize(c->ev_done));  // every earlier call (any stream) is done with the old workspace
        drop_graphs(c);
        const turboreg_status st = alloc_ws(c);
        if (st != TURBOREG_OK) {  // the old workspace is intact: keep the parameters it was sized for
            c->prm = old;
            set_ws_params(c);
            return st;
        }
    }
    set_ws_params(c);
    return TURBOREG_OK;
}

void turboreg_destroy(turboreg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->ev_done) cudaEventSynchronize(c->ev_done);  // the last call (any stream) is done with the workspace
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    free_ws(c);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->h_desc) cudaFreeHost(c->h_desc);
    if (c->h_results) cudaFreeHost(c->h_results);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->side_stream) cudaStreamDestroy(c->side_stream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    for (auto e : c->ev_chunk)
        if (e) cudaEventDestroy(e);
    for (auto e : c->ev_desc)
        if (e) cudaEventDestroy(e);
    if (c->pr_buf) cudaFree(c->pr_buf);
    if (c->rank_buf) cudaFree(c->rank_buf);
    delete c;
}

turboreg_status turboreg_register_batch(turboreg_ctx* c, const float* src, const float* dst, const int64_t* offsets,
                                        const int32_t* n, int32_t batch, turboreg_result* out, void* stream) {
    if (!c || !src || !dst || !offsets || !n || !out || batch < 1 || batch > c->max_batch)
        return TURBOREG_ERR_INVALID_ARGUMENT;
    for (int32_t p = 0; p < batch; ++p)
        if (offsets[p] < 0 || n[p] < 0) return TURBOREG_ERR_INVALID_ARGUMENT;
    if (!c->d_base) return TURBOREG_ERR_OUT_OF_MEMORY;
    CK(cudaSetDevice(c->device));
    c->split_rank = 0;
    c->split_world = 1;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    const bool dev_in = is_device_ptr(src) && is_device_ptr(dst);
    const bool dev_out = is_device_ptr(out);
    if (is_device_ptr(src) != is_device_ptr(dst)) return TURBOREG_ERR_INVALID_ARGUMENT;
    // Host inputs of a large batch are pipelined: the batch is cut into NCHUNK sub-batches whose H2D copies
    // run on the copy stream while the previous sub-batch's ingest + compat run (on a view of the
    // workspace); the rest of the path then runs once on the whole batch.  Sub-batch sizes double (1/255,
    // 2/255, .., 128/255 of the batch): only the first, smallest copy is exposed, and every later copy
    // (at most twice the previous sub-batch, ≈ 4.4 µs per N = 5000 pair over PCIe) hides behind the
    // previous sub-batch's compat (≈ 10 µs per pair).  Device inputs and small batches run as one launch
    // sequence.
    // as many doubling sub-batches as keep the first one at >= 4 pairs (launch overhead of tiny sub-batches)
    int nchunk = 1;
    if (!dev_in && batch >= 16 && c->use_chunks)
        while (nchunk < NCHUNK && (int64_t)batch >= 4 * ((int64_t)(1 << (nchunk + 1)) - 1)) ++nchunk;
    int32_t bnd[NCHUNK + 1];
    for (int k = 0; k <= nchunk; ++k)
        bnd[k] = nchunk == 1 ? (k ? batch : 0) : (int32_t)((int64_t)batch * ((1 << k) - 1) / ((1 << nchunk) - 1));
    // host inputs: each pair's rows go to the device staging area (pairs packed contiguously)
    const float* dsrc = src;
    const float* ddst = dst;
    std::vector<int64_t> dev_off(offsets, offsets + batch);
    struct Copy { int64_t dst_off, src_off, len; int chunk; };
    std::vector<Copy> copies;
    if (!dev_in) {
        int64_t cursor = 0;
        int32_t p = 0;
        for (int k = 0; k < nchunk; ++k) {
            p = bnd[k];
            while (p < bnd[k + 1]) {  // coalesce runs of contiguous pairs into single copies
                int32_t q = p;
                int64_t len = (n[p] >= 3 && n[p] <= c->max_n) ? n[p] : 0;
                while (q + 1 < bnd[k + 1] && offsets[q + 1] == offsets[q] + n[q] && n[q + 1] >= 3 &&
                       n[q + 1] <= c->max_n && len > 0) {
                    ++q;
                    len += n[q];
                }
                if (len > 0) {
                    copies.push_back({cursor, offsets[p], len, k});
                    int64_t cc = cursor;
                    for (int32_t r = p; r <= q; ++r) { dev_off[r] = cc; cc += n[r]; }
                    cursor += len;
                }
                p = q + 1;
            }
        }
        dsrc = c->d_inputs;
        ddst = c->d_inputs + 3 * (int64_t)c->max_n * c->max_batch;
    }
    int32_t maxn_batch = 3;
    int32_t maxn_chunk[NCHUNK];
    for (int k = 0; k < NCHUNK; ++k) maxn_chunk[k] = 3;
    c->last_n.assign(n, n + batch);
    int dslot = 0;
    trk::PairDesc* hd = next_desc(c, &dslot);
    CK(begin_call(c, s));
    for (int32_t p = 0; p < batch; ++p) {
        trk::PairDesc& d = hd[p];
        d.src = dsrc + 3 * dev_off[p];
        d.dst = ddst + 3 * dev_off[p];
        d.host_status = 0;
        d.pad = 0;
        if (n[p] < 3) d.host_status = TURBOREG_ERR_TOO_FEW_POINTS;
        else if (n[p] > c->max_n) d.host_status = TURBOREG_ERR_TOO_MANY_POINTS;
        d.n = d.host_status ? 0 : n[p];
        d.W = d.n ? words_per_row(d.n) : 0;
        if (d.n > maxn_batch) maxn_batch = d.n;
        for (int k = 0; k < nchunk; ++k)
            if (p >= bnd[k] && p < bnd[k + 1] && d.n > maxn_chunk[k]) maxn_chunk[k] = d.n;
    }
    CK(cudaMemcpyAsync(c->d_desc, hd, sizeof(trk::PairDesc) * batch, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(c->ev_desc[dslot], s));
    c->last_batch = batch;
    cudaStream_t cs = nchunk > 1 ? c->copy_stream : s;
    if (nchunk > 1) {  // the staging area is free once everything queued before on s is done
        CK(cudaEventRecord(c->ev_start, s));
        CK(cudaStreamWaitEvent(cs, c->ev_start, 0));
    }
    for (int k = 0; k < nchunk; ++k) {
        for (const Copy& cp : copies) {
            if (cp.chunk != k) continue;
            CK(cudaMemcpyAsync(const_cast<float*>(dsrc) + 3 * cp.dst_off, src + 3 * cp.src_off,
                               sizeof(float) * 3 * cp.len, cudaMemcpyHostToDevice, cs));
            CK(cudaMemcpyAsync(const_cast<float*>(ddst) + 3 * cp.dst_off, dst + 3 * cp.src_off,
                               sizeof(float) * 3 * cp.len, cudaMemcpyHostToDevice, cs));
        }
        if (nchunk > 1) CK(cudaEventRecord(c->ev_chunk[k], cs));
    }
    if (nchunk == 1) {
        turboreg_status st = run_pipeline(c, batch, maxn_batch, s, c->ransac_iters > 0 ? RUN_RANSAC : RUN_FULL);
        if (st != TURBOREG_OK) return st;
    } else {  // compat of sub-batch k overlaps the copy of sub-batch k+1; the rest runs on the whole batch
        for (int k = 0; k < nchunk; ++k) {
            CK(cudaStreamWaitEvent(s, c->ev_chunk[k], 0));
            const int32_t cnt = bnd[k + 1] - bnd[k];
            if (cnt == 0) continue;
            turboreg_status st = run_pipeline(c, cnt, maxn_chunk[k], s, RUN_FULL, bnd[k], PH_HEAD);
            if (st != TURBOREG_OK) return st;
        }
        turboreg_status st = run_pipeline(c, batch, maxn_batch, s, RUN_FULL, 0, PH_TAIL);
        if (st != TURBOREG_OK) return st;
    }
    const bool want_stage = c->prm.flags & TURBOREG_F_STAGE_TIMING;
    if (dev_out) {
        CK(cudaMemcpyAsync(out, c->d_results, sizeof(turboreg_result) * batch, cudaMemcpyDeviceToDevice, s));
        CK(end_call(c, s));
        if (want_stage && !c->profiling) {
            CK(cudaStreamSynchronize(s));
            harvest_events(c, nullptr);
        }
    } else {
        CK(cudaMemcpyAsync(c->h_results, c->d_results, sizeof(turboreg_result) * batch, cudaMemcpyDeviceToHost, s));
        CK(end_call(c, s));
        CK(cudaStreamSynchronize(s));
        float stage[3] = {0, 0, 0};
        if (want_stage && !c->profiling) harvest_events(c, stage);
        std::memcpy(out, c->h_results, sizeof(turboreg_result) * batch);
        if (want_stage)
            for (int32_t p = 0; p < batch; ++p) std::memcpy(out[p].stage_ms, stage, sizeof(stage));
    }
    return TURBOREG_OK;
}

turboreg_status turboreg_register(turboreg_ctx* c, const float* src, const float* dst, int32_t n, turboreg_result* out) {
    if (!c || !out) return TURBOREG_ERR_INVALID_ARGUMENT;
    const int64_t off = 0;
    turboreg_result tmp;
    const bool dev_out = is_device_ptr(out);
    if (dev_out) return TURBOREG_ERR_INVALID_ARGUMENT;
    turboreg_status st = turboreg_register_batch(c, src, dst, &off, &n, 1, &tmp, nullptr);
    if (st != TURBOREG_OK) return st;
    *out = tmp;
    return (turboreg_status)tmp.status;
}

turboreg_status turboreg_point_resolution(turboreg_ctx* c, const float* xyz, int32_t n, float* out_pr) {
    if (!c || !xyz || !out_pr || n < 2 || n > TURBOREG_MAX_CLOUD_POINTS) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->own_stream;
    // its own buffers, grown on demand (a cloud is not bounded by max_n): [flag, result, pad] int32 x 4,
    // nn2[n] int32, then the staged points (host input) float32 [n][3]
    const size_t need = 16 + sizeof(int) * (size_t)n + sizeof(float) * 3 * (size_t)n;
    CK(cudaEventSynchronize(c->ev_done));  // an earlier asynchronous call may still read pr_buf's memory
    if (need > c->pr_bytes) {
        void* nb = nullptr;
        CK(cudaMalloc(&nb, need));
        if (c->pr_buf) cudaFree(c->pr_buf);
        c->pr_buf = nb;
        c->pr_bytes = need;
    }
    CK(begin_call(c, s));
    int* flag = static_cast<int*>(c->pr_buf);
    float* res = reinterpret_cast<float*>(flag + 1);
    int* nn2 = flag + 4;
    const float* pts = xyz;
    if (!is_device_ptr(xyz)) {  // stage the host cloud
        float* staged = reinterpret_cast<float*>(nn2 + n);
        CK(cudaMemcpyAsync(staged, xyz, sizeof(float) * 3 * (size_t)n, cudaMemcpyHostToDevice, s));
        pts = staged;
    }
    CK(cudaMemsetAsync(flag, 0, sizeof(int) * 2, s));
    trk::k_fill_inf<<<(n + 255) / 256, 256, 0, s>>>(nn2, n);
    // candidate splits so the grid covers ~4 blocks per SM (each split at least one shared-memory tile)
    const int pb = (n + 255) / 256;
    const int splits = std::max(1, std::min((4 * c->num_sms + pb - 1) / pb, (n + trk::NN_TILE - 1) / trk::NN_TILE));
    const int span = (n + splits - 1) / splits;
    trk::k_nn_dist<<<dim3((unsigned)pb, (unsigned)splits), 256, 0, s>>>(pts, n, span, nn2, flag);
    CK(cudaGetLastError());
    trk::k_select_kth<<<1, 1024, 0, s>>>(nn2, n, (n - 1) / 2, res);
    CK(cudaGetLastError());
    int h[2];
    CK(cudaMemcpyAsync(h, flag, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(end_call(c, s));
    CK(cudaStreamSynchronize(s));
    c->launches += 3;
    if (h[0]) return TURBOREG_ERR_NONFINITE_INPUT;
    std::memcpy(out_pr, &h[1], sizeof(float));
    return TURBOREG_OK;
}

turboreg_status turboreg_ransac(turboreg_ctx* c, const float* src, const float* dst, int32_t n, int32_t iters,
                                uint64_t seed, turboreg_result* out) {
    if (!c || !out || iters < 1 || (int64_t)iters > (int64_t)c->ws.cl_stride) return TURBOREG_ERR_INVALID_ARGUMENT;
    c->ransac_iters = iters;
    c->ransac_seed = (unsigned long long)seed;
    const turboreg_status st = turboreg_register(c, src, dst, n, out);
    c->ransac_iters = 0;
    return st;
}

turboreg_status turboreg_get_intermediates(turboreg_ctx* c, int32_t pair, int32_t what, void* dst, size_t bytes,
                                           size_t* needed) {
    if (!c || pair < 0 || pair >= c->last_batch) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    const int n = c->last_n[pair];
    if (n < 3 || n > c->max_n) return TURBOREG_ERR_INVALID_ARGUMENT;
    const int W = words_per_row(n);
    const trk::WS& w = c->ws;
    trk::PairState st;
    CK(cudaMemcpy(&st, w.st + pair, sizeof(st), cudaMemcpyDeviceToHost));
    size_t need = 0;
    switch (what) {
        case TURBOREG_I_BITS:
        case TURBOREG_I_BITS_BASE: {
            if (what == TURBOREG_I_BITS_BASE && !w.bits_base) return TURBOREG_ERR_INVALID_ARGUMENT;
            need = sizeof(uint32_t) * (size_t)n * W;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            const uint32_t* src = (what == TURBOREG_I_BITS ? w.bits : w.bits_base) + pair * w.bits_stride;
            CK(cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
            return TURBOREG_OK;
        }
        case TURBOREG_I_SC2: {
            need = sizeof(int32_t) * (size_t)n * n;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            std::vector<int32_t> rp(n + 1);
            CK(cudaMemcpy(rp.data(), w.rowptr + pair * w.rp_stride, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
            std::vector<uint32_t> e(std::max(rp[n], 1));
            if (rp[n]) CK(cudaMemcpy(e.data(), w.edges + pair * w.edges_stride, sizeof(uint32_t) * rp[n], cudaMemcpyDeviceToHost));
            int32_t* G = static_cast<int32_t*>(dst);
            std::memset(G, 0, need);
            for (int64_t i = 0; i < n; ++i) {
                for (int k = rp[i]; k < rp[i + 1]; ++k) {
                    const uint32_t v = e[k];
                    const int64_t j = v >> 16;
                    const int32_t wt = (int32_t)(v & 0xffffu);
                    G[i * n + j] = wt;
                    G[j * n + i] = wt;
                }
            }
            return TURBOREG_OK;
        }
        case TURBOREG_I_EDGES: {  // compact O2 rows: uint32 rowptr[n+1], then the E edge words
            int32_t E = 0;
            CK(cudaMemcpy(&E, w.rowptr + pair * w.rp_stride + n, sizeof(int32_t), cudaMemcpyDeviceToHost));
            need = sizeof(uint32_t) * ((size_t)n + 1 + (size_t)E);
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            uint32_t* o = static_cast<uint32_t*>(dst);
            CK(cudaMemcpy(o, w.rowptr + pair * w.rp_stride, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
            if (E) CK(cudaMemcpy(o + n + 1, w.edges + pair * w.edges_stride, sizeof(uint32_t) * E, cudaMemcpyDeviceToHost));
            return TURBOREG_OK;
        }
        case TURBOREG_I_PIVOTS: {
            const int P = st.npiv;
            need = sizeof(int32_t) * 3 * (size_t)P;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            std::vector<int4> v(P);
            if (P) CK(cudaMemcpy(v.data(), w.piv + pair * w.piv_stride, sizeof(int4) * P, cudaMemcpyDeviceToHost));
            int32_t* o = static_cast<int32_t*>(dst);
            for (int k = 0; k < P; ++k) { o[3 * k] = v[k].x; o[3 * k + 1] = v[k].y; o[3 * k + 2] = v[k].z; }
            return TURBOREG_OK;
        }
        case TURBOREG_I_CLIQUES: {
            need = sizeof(int4) * (size_t)w.cl_stride;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            CK(cudaMemcpy(dst, w.cliq + pair * w.cl_stride, need, cudaMemcpyDeviceToHost));
            return TURBOREG_OK;
        }
        case TURBOREG_I_HYPS: {
            need = sizeof(float) * 16 * (size_t)w.cl_stride;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            CK(cudaMemcpy(dst, w.hyp + pair * w.cl_stride * 16, need, cudaMemcpyDeviceToHost));
            return TURBOREG_OK;
        }
        case TURBOREG_I_ERRORS: {  // (MAE, MSE) per slot; NaN for empty / degenerate slots (reading r20)
            need = sizeof(double) * 2 * (size_t)w.cl_stride;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            if (!(w.err_mode & 1)) return TURBOREG_ERR_INVALID_ARGUMENT;
            std::vector<double2> e((size_t)w.cl_stride * trk::SCORE_SEGS_MAX);
            std::vector<float> h((size_t)w.cl_stride * 16);
            CK(cudaMemcpy(e.data(), w.herr + pair * w.cl_stride * trk::SCORE_SEGS_MAX, sizeof(double2) * e.size(),
                          cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h.data(), w.hyp + pair * w.cl_stride * 16, sizeof(float) * h.size(), cudaMemcpyDeviceToHost));
            const double nn = (double)c->last_n[pair];
            double* out = static_cast<double*>(dst);
            for (size_t s = 0; s < (size_t)w.cl_stride; ++s) {
                int32_t flag;
                std::memcpy(&flag, &h[16 * s + 13], 4);
                const double2 v = e[s * trk::SCORE_SEGS_MAX];  // slot 0 holds the ordered sum (k_finalize)
                out[2 * s] = flag == 0 ? v.x / nn : std::nan("");
                out[2 * s + 1] = flag == 0 ? v.y / nn : std::nan("");
            }
            return TURBOREG_OK;
        }
        case TURBOREG_I_ROWSUM: {
            if (!(c->prm.flags & TURBOREG_F_ROW_SUMS)) return TURBOREG_ERR_INVALID_ARGUMENT;
            need = sizeof(int32_t) * (size_t)n;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            CK(cudaMemcpy(dst, c->d_rowsum + (int64_t)pair * c->max_n, need, cudaMemcpyDeviceToHost));
            return TURBOREG_OK;
        }
        case TURBOREG_I_STATE: {
            need = sizeof(int64_t) * 16;
            if (needed) *needed = need;
            if (!dst) return TURBOREG_OK;
            if (bytes < need) return TURBOREG_ERR_INVALID_ARGUMENT;
            int64_t* o = static_cast<int64_t*>(dst);
            const int64_t vals[16] = {n, W, st.edges, st.epos, st.alpha, st.c_gt, st.need, st.npiv,
                                      st.nonfinite, st.b1, st.above, st.edges_base, st.heavy_h, st.heavy_thr,
                                      (int64_t)st.deg_sum, 0};
            std::memcpy(o, vals, sizeof(vals));
            return TURBOREG_OK;
        }
        default: return TURBOREG_ERR_INVALID_ARGUMENT;
    }
}

turboreg_status turboreg_ranked_hypotheses(turboreg_ctx* c, int32_t pair, int32_t metric, int32_t top_k,
                                           turboreg_hypothesis* out, int32_t* count) {
    if (!c || !count || top_k < 0 || (top_k > 0 && !out) || metric < 0 || metric > 2) return TURBOREG_ERR_INVALID_ARGUMENT;
    if (pair < 0 || pair >= c->last_batch) return TURBOREG_ERR_INVALID_ARGUMENT;
    const int n = c->last_n[pair];
    if (n < 3 || n > c->max_n) return TURBOREG_ERR_INVALID_ARGUMENT;
    if (metric > 0 && !c->ws.herr) return TURBOREG_ERR_INVALID_ARGUMENT;
    const int64_t K = c->ws.cl_stride;
    if (K > ((int64_t)1 << 22)) return TURBOREG_ERR_INVALID_ARGUMENT;
    int m2 = 2;
    while (m2 < K) m2 <<= 1;
    CK(cudaSetDevice(c->device));
    CK(cudaEventSynchronize(c->ev_done));
    const size_t need = sizeof(trk::RankKey) * m2 + sizeof(int32_t) * m2 + 16 +
                        sizeof(trk::DevHypothesis) * (size_t)std::min<int64_t>(std::max(top_k, 1), K);
    if (need > c->rank_bytes) {
        void* nb = nullptr;
        CK(cudaMalloc(&nb, need));
        if (c->rank_buf) cudaFree(c->rank_buf);
        c->rank_buf = nb;
        c->rank_bytes = need;
    }
    cudaStream_t s = c->own_stream;
    CK(begin_call(c, s));
    trk::RankKey* keys = static_cast<trk::RankKey*>(c->rank_buf);
    int32_t* idx = reinterpret_cast<int32_t*>(keys + m2);
    int* d_cnt = idx + m2;
    trk::DevHypothesis* d_out = reinterpret_cast<trk::DevHypothesis*>(reinterpret_cast<char*>(c->rank_buf) +
                                                                      sizeof(trk::RankKey) * m2 + sizeof(int32_t) * m2 + 16);
    CK(cudaMemsetAsync(d_cnt, 0, sizeof(int), s));
    trk::k_rank_prep<<<(m2 + 255) / 256, 256, 0, s>>>(c->ws, pair, metric, keys, idx, m2);
    CK(cudaGetLastError());
    for (int size = 2; size <= m2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            trk::k_rank_step<<<(m2 / 2 + 255) / 256, 256, 0, s>>>(keys, idx, m2, size, stride);
            CK(cudaGetLastError());
        }
    trk::k_rank_count<<<1, 1024, 0, s>>>(keys, idx, m2, d_cnt);
    CK(cudaGetLastError());
    int valid = 0;
    CK(cudaMemcpyAsync(&valid, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int top = std::min(top_k, valid);
    if (top > 0) {
        trk::k_rank_emit<<<(top + 127) / 128, 128, 0, s>>>(c->ws, pair, keys, idx, top, n, d_out);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, d_out, sizeof(turboreg_hypothesis) * top, cudaMemcpyDeviceToHost, s));
    }
    CK(end_call(c, s));
    CK(cudaStreamSynchronize(s));
    *count = top;
    return TURBOREG_OK;
}

// ------------------------------------------------------------------------------------------ NEXT(1)
turboreg_status turboreg_split_begin(turboreg_ctx* c, const float* src, const float* dst, int32_t n, int32_t rank,
                                     int32_t world, void* stream) {
    if (!c || !src || !dst || world < 1 || world > 4096 || rank < 0 || rank >= world) return TURBOREG_ERR_INVALID_ARGUMENT;
    // the split covers the paper's path: O2 mode, inlier-number ranking, the tensor-core or popcount SC^2 block
    if (c->prm.graph_mode != 0 || c->opt_sc2_path == 2 ||
        (c->prm.flags & (TURBOREG_F_HYP_ERRORS | TURBOREG_F_RANK_MAE | TURBOREG_F_RANK_MSE | TURBOREG_F_ROW_SUMS)))
        return TURBOREG_ERR_INVALID_ARGUMENT;
    if (n < 3) return TURBOREG_ERR_TOO_FEW_POINTS;
    if (n > c->max_n) return TURBOREG_ERR_TOO_MANY_POINTS;
    if (!c->d_base) return TURBOREG_ERR_OUT_OF_MEMORY;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    if (is_device_ptr(src) != is_device_ptr(dst)) return TURBOREG_ERR_INVALID_ARGUMENT;
    int dslot = 0;
    trk::PairDesc* hd = next_desc(c, &dslot);
    CK(begin_call(c, s));
    const float* ds = src;
    const float* dd = dst;
    if (!is_device_ptr(src)) {  // stage host inputs in the context's input area
        float* in = c->d_inputs;
        CK(cudaMemcpyAsync(in, src, sizeof(float) * 3 * (size_t)n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(in + 3 * (size_t)c->max_n * c->max_batch, dst, sizeof(float) * 3 * (size_t)n,
                           cudaMemcpyHostToDevice, s));
        ds = in;
        dd = in + 3 * (size_t)c->max_n * c->max_batch;
    }
    hd[0] = trk::PairDesc{ds, dd, n, words_per_row(n), 0, 0};
    CK(cudaMemcpyAsync(c->d_desc, hd, sizeof(trk::PairDesc), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(c->ev_desc[dslot], s));
    c->split_rank = rank;
    c->split_world = world;
    c->last_batch = 1;
    c->last_n.assign(1, n);
    const turboreg_status st = launch_all(c, 1, n, s, RUN_FULL, 0, PH_HEAD);
    if (st != TURBOREG_OK) return st;
    CK(end_call(c, s));
    return TURBOREG_OK;
}

turboreg_status turboreg_split_buffer(turboreg_ctx* c, int32_t which, void** dev_ptr, size_t* bytes) {
    if (!c || !dev_ptr || !bytes || c->last_batch < 1 || c->last_n.empty()) return TURBOREG_ERR_INVALID_ARGUMENT;
    const int n = c->last_n[0];
    if (n < 3 || n > c->max_n) return TURBOREG_ERR_INVALID_ARGUMENT;
    switch (which) {
        case TURBOREG_SPLIT_BITS: *dev_ptr = c->ws.bits; *bytes = sizeof(uint32_t) * (size_t)n * words_per_row(n); break;
        case TURBOREG_SPLIT_EDGES: *dev_ptr = c->ws.edges; *bytes = sizeof(uint32_t) * (size_t)c->ws.edges_stride; break;
        case TURBOREG_SPLIT_RESULT: *dev_ptr = c->d_results; *bytes = sizeof(turboreg_result); break;
        default: return TURBOREG_ERR_INVALID_ARGUMENT;
    }
    return TURBOREG_OK;
}

turboreg_status turboreg_split_sc2(turboreg_ctx* c, int64_t* num_edges, void* stream) {
    if (!c || !num_edges || c->split_world < 1 || c->last_n.empty()) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    CK(begin_call(c, s));
    const turboreg_status st = launch_all(c, 1, c->last_n[0], s, RUN_FULL, 0, PH_GRAPH);
    if (st != TURBOREG_OK) return st;
    int32_t E = 0;
    CK(cudaMemcpyAsync(&E, &c->ws.st[0].edges, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(end_call(c, s));
    CK(cudaStreamSynchronize(s));
    *num_edges = E;
    return TURBOREG_OK;
}

turboreg_status turboreg_split_search(turboreg_ctx* c, void* stream) {
    if (!c || c->last_n.empty()) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    CK(begin_call(c, s));
    const turboreg_status st = launch_all(c, 1, c->last_n[0], s, RUN_FULL, 0, PH_SEARCH);
    if (st != TURBOREG_OK) return st;
    CK(end_call(c, s));
    return TURBOREG_OK;
}

turboreg_status turboreg_split_merge(turboreg_ctx* c, const void* parts, int32_t world, turboreg_result* out,
                                     void* stream) {
    if (!c || !parts || !out || world < 1 || !is_device_ptr(parts)) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    CK(begin_call(c, s));
    trk::k_split_merge<<<1, 32, 0, s>>>(static_cast<const trk::DevResult*>(parts), world,
                                        static_cast<trk::DevResult*>(c->d_results));
    CK(cudaGetLastError());
    c->launches++;
    c->k_launches[KID_MERGE]++;
    c->split_rank = 0;
    c->split_world = 1;
    if (is_device_ptr(out)) {
        CK(cudaMemcpyAsync(out, c->d_results, sizeof(turboreg_result), cudaMemcpyDeviceToDevice, s));
        CK(end_call(c, s));
    } else {
        CK(cudaMemcpyAsync(c->h_results, c->d_results, sizeof(turboreg_result), cudaMemcpyDeviceToHost, s));
        CK(end_call(c, s));
        CK(cudaStreamSynchronize(s));
        std::memcpy(out, c->h_results, sizeof(turboreg_result));
    }
    return TURBOREG_OK;
}

turboreg_status turboreg_pgs_from_adjacency(turboreg_ctx* c, const uint32_t* bits, int32_t n, int32_t stride_words) {
    if (!c || !bits || n < 3 || n > c->max_n || stride_words < (n + 31) / 32) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    const int W = words_per_row(n);
    std::vector<uint32_t> rows((size_t)n * W, 0u);
    const int used = (n + 31) / 32;
    for (int r = 0; r < n; ++r)
        for (int k = 0; k < used; ++k) {
            uint32_t v = bits[(size_t)r * stride_words + k];
            if (k == used - 1 && (n & 31)) v &= (1u << (n & 31)) - 1u;
            rows[(size_t)r * W + k] = v;
        }
    cudaStream_t s = c->own_stream;
    c->split_rank = 0;
    c->split_world = 1;
    int dslot = 0;
    trk::PairDesc* hd = next_desc(c, &dslot);
    CK(begin_call(c, s));
    CK(cudaMemcpyAsync(c->ws.bits, rows.data(), sizeof(uint32_t) * rows.size(), cudaMemcpyHostToDevice, s));
    trk::PairDesc& d = hd[0];
    d.src = nullptr;
    d.dst = nullptr;
    d.n = n;
    d.W = W;
    d.host_status = 0;
    d.pad = 0;
    CK(cudaMemcpyAsync(c->d_desc, hd, sizeof(trk::PairDesc), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(c->ev_desc[dslot], s));
    c->last_batch = 1;
    c->last_n.assign(1, n);
    turboreg_status st = run_pipeline(c, 1, n, s, RUN_FROM_ADJ);
    if (st != TURBOREG_OK) return st;
    CK(end_call(c, s));
    CK(cudaStreamSynchronize(s));
    if (!c->profiling) harvest_events(c, nullptr);
    return TURBOREG_OK;
}

turboreg_status turboreg_profile_begin(turboreg_ctx* c) {
    if (!c || !(c->prm.flags & TURBOREG_F_KERNEL_TIMING)) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    harvest_events(c, nullptr);
    for (int k = 0; k < KID_COUNT; ++k) { c->k_ms[k] = 0.0; c->k_launches[k] = 0; }
    c->profiling = true;
    return TURBOREG_OK;
}

turboreg_status turboreg_profile_end(turboreg_ctx* c, const char** names, float* ms, int64_t* launches, int32_t cap,
                                     int32_t* count) {
    if (!c) return TURBOREG_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(c->device));
    harvest_events(c, nullptr);
    c->profiling = false;
    for (int k = 0; k < KID_COUNT && k < cap; ++k) {
        if (names) names[k] = kKernelNames[k];
        if (ms) ms[k] = (float)c->k_ms[k];
        if (launches) launches[k] = c->k_launches[k];
    }
    if (count) *count = KID_COUNT;
    return TURBOREG_OK;
}

int64_t turboreg_launch_count(const turboreg_ctx* c) { return c ? c->launches : 0; }

size_t turboreg_workspace_bytes(const turboreg_ctx* c) { return c ? c->ws_bytes : 0; }

}  // extern "C"
