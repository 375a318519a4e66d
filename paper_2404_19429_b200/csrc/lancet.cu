// lancet.cu -- the C-ABI (include/lancet_moe.h): context, workspace, and the stream/event
// chunk scheduler of the MoE layer step (S1 forward, S2 backward).
//
// Scheduling (Lancet, PAPER.md):
//   * forward (S1): the MoE input/output is partitioned on the batch dimension and
//     the all-to-all and experts irregularly inside (fig:proposed_partition); chunk
//     c's all-to-all overlaps other chunks' expert compute; the comm lane runs
//     the chunks in stage order D0..D(n-1), C0..C(n-1).
//   * backward (S2): the dW GEMMs of chunk c are enqueued right after chunk c's dX GEMMs, i.e.
//     right after the launch of the all-to-all they overlap.
//   * the irregular all-to-all is a size exchange followed by the data exchange of only the
//     real rows; the size exchange happens once per forward for all chunks
//     (R11) -- the only host synchronisation of the step (world > 1).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "context.h"
#include "kernels.h"
#include "peer.h"
#include "internal.h"

#define LANCET_API extern "C" __attribute__((visibility("default")))

using namespace lancet;

struct lancet_local_group {
    LocalGroupImpl* impl;
    int world;
};

namespace {

thread_local std::string g_thread_err;

lancet_status fail(lancet_ctx* c, lancet_status st, const std::string& msg)
{
    if (c) {
        c->err = msg;
        if (st == LANCET_ERR_CUDA || st == LANCET_ERR_NCCL) c->poisoned = true;
    }
    g_thread_err = msg;
    return st;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(c, LANCET_ERR_CUDA,                                             \
                        std::string(#call) + ": " + cudaGetErrorString(e_));            \
    } while (0)

#define CHECK_LAUNCH()                                                                  \
    do {                                                                                \
        cudaError_t e_ = cudaGetLastError();                                            \
        if (e_ != cudaSuccess)                                                          \
            return fail(c, LANCET_ERR_CUDA, std::string("kernel launch: ") +            \
                                                cudaGetErrorString(e_));                \
    } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int capacity_of(int T, int k, int E, double cf)
{
    // R4: C = max(1, min(T, ceil(cf*k*T/E))) in double
    const double v = std::ceil(cf * (double)k * (double)T / (double)E);
    long c = (long)v;
    if (c > T) c = T;
    if (c < 1) c = 1;
    return (int)c;
}

unsigned long long cfg_hash(const lancet_layer_config& c)
{
    unsigned long long h = 1469598103934665603ull;
    const int32_t v[] = {c.d_model, c.d_ffn, c.n_experts, c.max_k, c.max_chunks, c.dtype, c.act,
                         (int32_t)(c.flags & LANCET_FLAG_RENORMALIZE)};
    for (int32_t x : v) { h ^= (unsigned)x; h *= 1099511628211ull; }
    return h;
}

template <typename T>
lancet_status dalloc(lancet_ctx* c, T** p, size_t bytes)
{
    bytes = std::max<size_t>(bytes, 256);
    void* q = nullptr;
    if (c->nccl_mem && (q = nccl_mem_alloc(bytes))) {
        cudaGetLastError();
        c->allocs.push_back({q, bytes, true});
        if (c->comm && c->comm->register_buffer(q, bytes) == 0) ++c->nccl_registered;
        *p = reinterpret_cast<T*>(q);
        return LANCET_OK;
    }
    if (cudaMalloc(&q, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, LANCET_ERR_NOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    c->allocs.push_back({q, bytes, false});
    *p = reinterpret_cast<T*>(q);
    return LANCET_OK;
}

void dfree(const lancet::DevBuf& b)
{
    if (b.nccl) nccl_mem_free(b.p);
    else cudaFree(b.p);
}

void free_all(lancet_ctx* c)
{
    for (auto& b : c->allocs) dfree(b);
    c->allocs.clear();
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->h_grp) cudaFreeHost(c->h_grp);
    c->h_counts = c->h_grp = nullptr;
}

// ---- timeline -----------------------------------------------------------------------------
struct OpScope {
    lancet_ctx* c;
    size_t i;
    cudaStream_t s;
    OpScope(lancet_ctx* ctx, const char* name, int lane, int chunk, cudaStream_t st) : c(ctx), s(st) {
        i = (size_t)-1;
        if (!(c->cfg.flags & LANCET_FLAG_TIMELINE)) return;
        if ((c->cfg.flags & LANCET_FLAG_TIMELINE_GEMM_ONLY) && strncmp(name, "expert_", 7) != 0) return;
        if (c->tl_used + 2 > c->tl_events.size()) {
            for (int q = 0; q < 64; ++q) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                c->tl_events.push_back(e);
            }
        }
        OpEvent op;
        op.name = name;
        op.lane = lane;
        op.chunk = chunk;
        op.beg = c->tl_events[c->tl_used++];
        op.end = c->tl_events[c->tl_used++];
        cudaEventRecord(op.beg, s);
        c->ops.push_back(op);
        i = c->ops.size() - 1;
    }
    ~OpScope() {
        if (i != (size_t)-1) cudaEventRecord(c->ops[i].end, s);
    }
};

// ---- grouped GEMM dispatch ---------------------------------------------------------------
constexpr int kTcMaxGroups = 128;   // gemm_tc.cu tc::kMaxGroups

lancet_status run_gemm(lancet_ctx* c, GemmArgs& a, cudaStream_t s, int* launches)
{
    if (c->bf16 && !(c->cfg.flags & LANCET_FLAG_SIMT_GEMM)) {
        a.multicast = (c->cfg.flags & LANCET_FLAG_GEMM_MULTICAST) != 0;
        // leave LANCET_COMM_SMS SMs to the exchange kernels running beside the persistent GEMMs:
        // NCCL's (world > 1) and the fused push kernels on the comm stream (push mode)
        const bool reserve = (c->comm && c->comm->is_nccl()) ||
                             (c->push && !(c->cfg.flags & LANCET_FLAG_SERIAL));
        const int all = reserve ? c->num_sms - LANCET_COMM_SMS : c->num_sms;
        const int sms = c->cfg.gemm_sms > 0 ? std::min(c->cfg.gemm_sms, c->num_sms) : all;
        // the kernel caches at most kTcMaxGroups group entries: larger tables go in batches,
        // each inside one cycle of the weights (B and C pointers shifted to its first group)
        const int ng = a.n_groups, nw = a.n_weights > 0 ? a.n_weights : ng;
        if (ng > kTcMaxGroups && a.gpw != 1)
            return fail(c, LANCET_ERR_UNSUPPORTED, "tcgen05 GEMM: > 128 groups with several groups per weight");
        if (ng > kTcMaxGroups && a.cs.wait_flags)
            return fail(c, LANCET_ERR_UNSUPPORTED, "tcgen05 GEMM: the chunk pipeline needs <= 128 groups per launch");
        for (int g0 = 0; g0 < ng;) {
            GemmArgs b = a;
            int g1 = std::min(ng, g0 + kTcMaxGroups);
            if (a.mode == GEMM_M_GROUPED) {
                g1 = std::min(g1, (g0 / nw + 1) * nw);
                const int w0 = g0 % nw;
                b.B = (const char*)a.B + (size_t)w0 * a.b_group_stride * c->elt;
                b.b_rows = a.b_rows - (long)w0 * (a.b_mn ? a.K : a.N);
                b.n_weights = nw - w0;
            } else {
                b.C = (char*)a.C + (size_t)g0 * a.c_group_stride * 4;
            }
            b.n_groups = g1 - g0;
            b.grp_rows = a.grp_rows + g0;
            b.grp_off = a.grp_off + g0;
            const int r = launch_gemm_tc(b, sms, s);
            if (r < 0) {
                CHECK_LAUNCH();
                return fail(c, LANCET_ERR_UNSUPPORTED,
                            "tcgen05 GEMM: shape or layout not supported (N=" + std::to_string(a.N) + " K=" +
                                std::to_string(a.K) + " M=" + std::to_string(a.M) + " groups=" +
                                std::to_string(a.n_groups) + ") or tensor-map encoding failed");
            }
            *launches += r;
            g0 = g1;
        }
    } else {
        if (a.cs.wait_flags)
            return fail(c, LANCET_ERR_UNSUPPORTED, "the device-side chunk pipeline runs on the tcgen05 GEMM only");
        *launches += launch_gemm_simt(a, c->bf16, s);
    }
    CHECK_LAUNCH();
    return LANCET_OK;
}

// M-grouped expert GEMMs of the forward over groups [g0, g0+ng) of the expert-side table.
GemmArgs grouped_args(lancet_ctx* c, const int* grp_rows, const int* grp_off, int ng, int max_rows)
{
    GemmArgs a{};
    a.mode = GEMM_M_GROUPED; a.n_groups = ng; a.gpw = 1; a.n_weights = c->E_l;
    a.grp_rows = grp_rows; a.grp_off = grp_off; a.max_rows = max_rows; a.act = c->cfg.act;
    a.c_rows = c->rows_exp;
    return a;
}

// fc1: H = act(X W1^T), G' = act'(X W1^T).  cs (push mode): the TMA producer waits for each
// chunk's rows on the device (ChunkSync)
lancet_status expert_fc1(lancet_ctx* c, const int* grp_rows, const int* grp_off, int ng, int max_rows,
                         cudaStream_t s, int chunk, int* launches, const ChunkSync* cs = nullptr)
{
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    GemmArgs a = grouped_args(c, grp_rows, grp_off, ng, max_rows);
    if (cs) a.cs = *cs;
    OpScope op(c, "expert_fc1", 0, chunk, s);
    a.A = c->ep ? c->xe : c->xs; a.lda = d; a.a_rows = c->rows_exp;
    a.B = c->w1; a.ldb = d; a.b_group_stride = (long)f * d; a.b_mn = false; a.a_mn = false;
    a.b_rows = (long)c->E_l * f;
    a.C = c->H; a.C2 = c->Gp; a.ldc = f; a.N = f; a.K = d; a.epi = EPI_ACT;
    return run_gemm(c, a, s, launches);
}

// fc2: O = H W2^T
lancet_status expert_fc2(lancet_ctx* c, const int* grp_rows, const int* grp_off, int ng, int max_rows,
                         cudaStream_t s, int chunk, int* launches)
{
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    GemmArgs a = grouped_args(c, grp_rows, grp_off, ng, max_rows);
    OpScope op(c, "expert_fc2", 0, chunk, s);
    a.A = c->H; a.lda = f; a.a_rows = c->rows_exp; a.a_mn = false;
    a.B = c->w2; a.ldb = f; a.b_group_stride = (long)d * f; a.b_rows = (long)c->E_l * d; a.b_mn = false;
    a.C = c->out; a.C2 = nullptr; a.ldc = d; a.N = d; a.K = f; a.epi = EPI_STORE;
    return run_gemm(c, a, s, launches);
}

// M-grouped expert GEMMs of the forward over groups [g0, g0+ng) of the expert-side table.
lancet_status expert_forward(lancet_ctx* c, const int* grp_rows, const int* grp_off, int ng,
                             int max_rows, cudaStream_t s, int chunk, int* launches)
{
    lancet_status st = expert_fc1(c, grp_rows, grp_off, ng, max_rows, s, chunk, launches);
    if (st) return st;
    return expert_fc2(c, grp_rows, grp_off, ng, max_rows, s, chunk, launches);
}

// dX GEMMs (critical path) of the backward.
// dA = (dO W2) * act'(A):  B(n=f, k=d) = W2[e][k][n]  (MN-major).  cs: device-side waits.
lancet_status expert_dfc2(lancet_ctx* c, const void* dout, const int* grp_rows, const int* grp_off, int ng,
                          int max_rows, cudaStream_t s, int chunk, int* launches, const ChunkSync* cs = nullptr)
{
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    GemmArgs a = grouped_args(c, grp_rows, grp_off, ng, max_rows);
    if (cs) a.cs = *cs;
    OpScope op(c, "expert_dfc2", 0, chunk, s);
    a.A = dout; a.lda = d; a.a_mn = false; a.a_rows = c->rows_exp;
    a.B = c->w2; a.ldb = f; a.b_group_stride = (long)d * f; a.b_mn = true;
    a.b_rows = (long)c->E_l * d;
    a.C = c->dA; a.ldc = f; a.aux = c->Gp; a.N = f; a.K = d; a.epi = EPI_DACT;
    return run_gemm(c, a, s, launches);
}

// dX = dA W1:  B(n=d, k=f) = W1[e][k][n]  (MN-major)
lancet_status expert_dfc1(lancet_ctx* c, const int* grp_rows, const int* grp_off, int ng, int max_rows,
                          cudaStream_t s, int chunk, int* launches)
{
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    GemmArgs a = grouped_args(c, grp_rows, grp_off, ng, max_rows);
    OpScope op(c, "expert_dfc1", 0, chunk, s);
    a.A = c->dA; a.lda = f; a.a_mn = false; a.a_rows = c->rows_exp;
    a.B = c->w1; a.ldb = d; a.b_group_stride = (long)f * d; a.b_mn = true;
    a.b_rows = (long)c->E_l * f;
    a.C = c->dXe; a.ldc = d; a.aux = nullptr; a.N = d; a.K = f; a.epi = EPI_STORE;
    return run_gemm(c, a, s, launches);
}

// dX GEMMs (critical path) of the backward.
lancet_status expert_backward_dx(lancet_ctx* c, const void* dout, const int* grp_rows,
                                 const int* grp_off, int ng, int max_rows, cudaStream_t s,
                                 int chunk, int* launches)
{
    lancet_status st = expert_dfc2(c, dout, grp_rows, grp_off, ng, max_rows, s, chunk, launches);
    if (st) return st;
    return expert_dfc1(c, grp_rows, grp_off, ng, max_rows, s, chunk, launches);
}

// dW GEMMs (K-grouped over each group's token rows): dW2 (+)= dO^T H, dW1 (+)= dA^T X.
lancet_status expert_backward_dw(lancet_ctx* c, const void* dout, const int* grp_rows,
                                 const int* grp_off, int ng, float* dw1, float* dw2,
                                 int accumulate, cudaStream_t s, int chunk, int* launches, int which = 3)
{
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    GemmArgs a{};
    a.mode = GEMM_K_GROUPED; a.n_groups = ng; a.gpw = 1; a.n_weights = c->E_l;
    a.grp_rows = grp_rows; a.grp_off = grp_off; a.accumulate = accumulate;
    a.a_mn = true; a.b_mn = true; a.epi = EPI_F32; a.b_group_stride = 0;
    a.a_rows = c->rows_exp; a.b_rows = c->rows_exp;
    if (which & 2) {
        OpScope op(c, "expert_dw2", 0, chunk, s);
        a.A = dout; a.lda = d; a.B = c->H; a.ldb = f;
        a.C = dw2; a.ldc = f; a.c_group_stride = (long)d * f; a.M = d; a.N = f;
        lancet_status st = run_gemm(c, a, s, launches);
        if (st) return st;
    }
    if (which & 1) {
        OpScope op(c, "expert_dw1", 0, chunk, s);
        a.A = c->dA; a.lda = f; a.B = c->ep ? c->xe : c->xs; a.ldb = d;
        a.C = dw1; a.ldc = d; a.c_group_stride = (long)f * d; a.M = f; a.N = d;
        return run_gemm(c, a, s, launches);
    }
    return LANCET_OK;
}

// Cross-layer dW scheduling (R17): enqueue the pending dW part(s) `which` of context o on
// stream s, after o's dX GEMMs (o->ev_dw_ready), all chunks in chunk order.
lancet_status enqueue_pending_dw(lancet_ctx* c, int which, cudaStream_t s, int* launches)
{
    if (which < 1 || which > 3) return fail(c, LANCET_ERR_ARG, "which must be 1 (dW1), 2 (dW2) or 3");
    if ((c->dw_pending & which) != which) return fail(c, LANCET_ERR_STATE, "requested dW GEMMs are not pending");
    CK(cudaStreamWaitEvent(s, c->ev_dw_ready, 0));
    lancet_status st;
    if (!c->ep) {
        st = expert_backward_dw(c, c->dcomb, c->send_rows, c->send_off, c->cfg.n_experts, c->pend_dw1,
                                c->pend_dw2, 0, s, -1, launches, which);
    } else {
        const int E_l = c->E_l, n = c->n;
        const int* rows = c->grp_dev;
        const int* off = c->grp_dev + n * E_l;
        st = LANCET_OK;
        for (int ch = 0; ch < n && !st; ++ch)
            st = expert_backward_dw(c, c->dout, rows + ch * E_l, off + ch * E_l, E_l, c->pend_dw1, c->pend_dw2,
                                    ch > 0, s, ch, launches, which);
    }
    if (st) return st;
    c->dw_pending &= ~which;
    return LANCET_OK;
}

lancet_status validate_cfg(const lancet_layer_config* cfg, int world)
{
    if (!cfg) return fail(nullptr, LANCET_ERR_ARG, "cfg is NULL");
    if (cfg->d_model <= 0 || cfg->d_model % 8) return fail(nullptr, LANCET_ERR_ARG, "d_model must be a positive multiple of 8");
    if (cfg->d_ffn <= 0 || cfg->d_ffn % 8) return fail(nullptr, LANCET_ERR_ARG, "d_ffn must be a positive multiple of 8");
    if (cfg->n_experts < 1 || cfg->n_experts > kMaxExperts) return fail(nullptr, LANCET_ERR_ARG, "n_experts must be in [1, 256]");
    if (world < 1 || cfg->n_experts % world) return fail(nullptr, LANCET_ERR_ARG, "n_experts % world != 0");
    if (cfg->max_tokens < 1) return fail(nullptr, LANCET_ERR_ARG, "max_tokens < 1");
    if (cfg->max_k < 1 || cfg->max_k > kMaxK || cfg->max_k > cfg->n_experts) return fail(nullptr, LANCET_ERR_ARG, "max_k must be in [1, min(8, E)]");
    if (cfg->max_chunks < 1 || cfg->max_chunks > kMaxChunks) return fail(nullptr, LANCET_ERR_ARG, "max_chunks must be in [1, 64]");
    if (cfg->dtype != LANCET_BF16 && cfg->dtype != LANCET_FP32) return fail(nullptr, LANCET_ERR_ARG, "bad dtype");
    if (cfg->act < 0 || cfg->act > 2) return fail(nullptr, LANCET_ERR_ARG, "bad act");
    return LANCET_OK;
}

lancet_status create_common(lancet_ctx* c, int world, int rank, int device, const lancet_layer_config* cfg)
{
    c->world = world;
    c->ep = world > 1 || (cfg->flags & LANCET_FLAG_FORCE_EP);
    c->rank = rank;
    c->device = device;
    c->cfg = *cfg;
    c->E_l = cfg->n_experts / world;
    c->bf16 = cfg->dtype == LANCET_BF16;
    c->elt = c->bf16 ? 2 : 4;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(c, LANCET_ERR_UNSUPPORTED, std::string("lancet_moe needs an sm_100 (B200) device, found ") + prop.name);
    c->num_sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_comp2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_gate, cudaStreamNonBlocking));
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->s_comm, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_counts, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_dw_ready, cudaEventDisableTiming));
    CK(cudaEventCreate(&c->ev_tl_base));
    for (int i = 0; i < 8 * kMaxChunks + 16; ++i) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_pool.push_back(e);
    }

    const int E = cfg->n_experts, T = cfg->max_tokens, K = cfg->max_k, d = cfg->d_model, f = cfg->d_ffn;
    const int n_tiles = ceil_div(T, kScanTile);
    c->rows_src = T * K + E * kRowAlign;
    lancet_status st;
#define AL(ptr, bytes) if ((st = dalloc(c, &(ptr), (bytes)))) return st
    AL(c->logits, sizeof(float) * (size_t)T * E);
    AL(c->idx, sizeof(int) * (size_t)T * K);
    AL(c->w, sizeof(float) * (size_t)T * K);
    AL(c->slot, sizeof(int) * (size_t)T * K);
    AL(c->hist, sizeof(int) * (size_t)n_tiles * E);
    AL(c->bpr_score, sizeof(double) * (size_t)T);
    AL(c->bpr_list, sizeof(int) * (size_t)T * K);
    AL(c->bpr_adm, (size_t)T * K);
    AL(c->bpr_hist, sizeof(int) * (size_t)n_tiles * E);
    AL(c->bpr_meta, sizeof(int) * E);
    AL(c->S, sizeof(int) * (size_t)E * (kMaxChunks + 1));
    AL(c->send_rows, sizeof(int) * E);
    AL(c->send_off, sizeof(int) * E);
    AL(c->g, sizeof(float) * (size_t)T * K);
    AL(c->prow, sizeof(int) * (size_t)T * K);
    AL(c->dlogit, sizeof(float) * (size_t)T * E);
    AL(c->dwg_partial, sizeof(float) * dwg_partial_floats(T, d, E));
    AL(c->wgT, sizeof(float) * (size_t)d * E);
    AL(c->counts_dev, sizeof(int) * 2 * (size_t)E * kMaxChunks);
    AL(c->carry, sizeof(int) * (size_t)E * (kMaxChunks + 1));
    AL(c->grp_dev, sizeof(int) * (2 * (size_t)c->E_l * kMaxChunks + 2 * (size_t)c->E_l));   // + merged dW table
    const size_t rs = (size_t)c->rows_src * d * c->elt;
    AL(c->xs, rs);
    AL(c->dcomb, rs);
    if (!c->ep) {
        c->rows_exp = c->rows_src;
        c->xe = c->xs;
        c->comb = nullptr;                      // world 1: comb == out
        c->dout = c->dcomb;
        c->dxcomb = nullptr;                    // world 1: dxcomb == dXe
        const size_t rf = (size_t)c->rows_exp * f * c->elt, rd = (size_t)c->rows_exp * d * c->elt;
        if (cfg->act != LANCET_ACT_IDENTITY_EXPERT) {
            AL(c->H, rf); AL(c->Gp, rf); AL(c->dA, rf);
            AL(c->out, rd); AL(c->dXe, rd);
        }
    } else {
        AL(c->comb, rs);
        AL(c->dxcomb, rs);
        CK(cudaMallocHost(&c->h_counts, sizeof(int) * 2 * (size_t)E * kMaxChunks));
        CK(cudaMallocHost(&c->h_grp, sizeof(int) * 2 * (size_t)c->E_l * kMaxChunks));
        c->rows_exp = 0;                        // grown on demand by the forward
    }
#undef AL
    CK(cudaMemset(c->xs, 0, rs));
    CK(cudaMemset(c->dcomb, 0, rs));
    CK(cudaMemset(c->send_off, 0, sizeof(int) * E));     // block mode never writes them; the
    CK(cudaMemset(c->send_rows, 0, sizeof(int) * E));    // push kernels' row arithmetic cancels them
    CK(cudaDeviceSynchronize());
    return LANCET_OK;
}

// Expert-side buffers for world > 1, grown to `rows` rows.
lancet_status ensure_expert_rows(lancet_ctx* c, int rows)
{
    if (rows <= c->rows_exp) return LANCET_OK;
    // peers map these buffers (CUDA IPC): never reallocate under them
    if (c->peer) return fail(c, LANCET_ERR_ARG, "peer transport: the step needs " + std::to_string(rows) +
                                                    " expert-side rows, more than the " + std::to_string(c->rows_exp) +
                                                    " allocated at creation");
    const int d = c->cfg.d_model, f = c->cfg.d_ffn;
    const int newrows = round_up(std::max(rows, c->rows_exp + c->rows_exp / 4), kRowAlign);
    CK(cudaDeviceSynchronize());
    void* olds[] = {c->xe, c->H, c->Gp, c->out, c->dout, c->dA, c->dXe};
    for (void* p : olds) {
        if (!p) continue;
        for (size_t i = 0; i < c->allocs.size(); ++i)
            if (c->allocs[i].p == p) {
                if (c->comm && c->allocs[i].nccl && c->nccl_registered > 0) {
                    c->comm->deregister_buffer(p);
                    --c->nccl_registered;
                }
                dfree(c->allocs[i]);
                c->allocs.erase(c->allocs.begin() + i);
                break;
            }
    }
    c->xe = c->H = c->Gp = c->out = c->dout = c->dA = c->dXe = nullptr;
    const size_t rf = (size_t)newrows * f * c->elt, rd = (size_t)newrows * d * c->elt;
    lancet_status st;
    if ((st = dalloc(c, &c->xe, rd))) return st;
    if ((st = dalloc(c, &c->dout, rd))) return st;
    if (c->cfg.act != LANCET_ACT_IDENTITY_EXPERT) {
        if ((st = dalloc(c, &c->H, rf))) return st;
        if ((st = dalloc(c, &c->Gp, rf))) return st;
        if ((st = dalloc(c, &c->dA, rf))) return st;
        if ((st = dalloc(c, &c->out, rd))) return st;
        if ((st = dalloc(c, &c->dXe, rd))) return st;
    }
    c->rows_exp = newrows;
    return LANCET_OK;
}

lancet_status check_ready(lancet_ctx* c)
{
    if (!c) return fail(nullptr, LANCET_ERR_ARG, "ctx is NULL");
    if (c->poisoned) return fail(c, LANCET_ERR_STATE, "context poisoned by an earlier error: " + c->err);
    if (const uint32_t pe = lancet::peer_error(c)) {
        c->poisoned = true;
        return fail(c, LANCET_ERR_STATE, "context poisoned: " + lancet::peer_error_text(pe));
    }
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, LANCET_ERR_CUDA, cudaGetErrorString(e));
    return LANCET_OK;
}

// ---- world > 1 exchange plans -----------------------------------------------------------
// Host view of the routing sizes after the counts exchange.
// Send side of the exchange (host): S[e][c] = prefix over chunks of the rows this rank
// admitted to expert e, send_off[e] = 128-aligned packed row offset of expert e (the same
// layout the device computes in K2) -- chunk c of expert e is rows
// [send_off[e] + S[e][c], send_off[e] + S[e][c+1]).
void plan_send(int E, int n, const int* send, int* S, int* send_off)
{
    int off = 0;
    for (int e = 0; e < E; ++e) {
        S[e * (n + 1)] = 0;
        for (int c = 0; c < n; ++c) S[e * (n + 1) + c + 1] = S[e * (n + 1) + c] + send[e * n + c];
        send_off[e] = off;
        off += round_up(S[e * (n + 1) + n], kRowAlign);
    }
}

// Receive side (host): one GEMM group per (chunk, local expert), table order chunk-major
// [n][E_l]; buffer order expert-major (e_l, c) so an expert's rows over all chunks form one
// K range for its dW GEMM; inside a group rows are ordered by source rank (R12).
int plan_recv(int G, int E_l, int n, const int* recv, int* grp_rows, int* grp_off, int* src_off)
{
    int row = 0;
    for (int el = 0; el < E_l; ++el)
        for (int c = 0; c < n; ++c) {
            int r = 0;
            for (int src = 0; src < G; ++src) {
                src_off[(src * E_l + el) * n + c] = r;
                r += recv[(src * E_l + el) * n + c];
            }
            grp_rows[c * E_l + el] = r;
            grp_off[c * E_l + el] = row;
            row += round_up(r, kRowAlign);
        }
    return row;
}

struct Plan {
    int E, E_l, G, n;
    std::vector<int> send;      // [E][n]
    std::vector<int> recv;      // [G][E_l][n]
    std::vector<int> S;         // [E][n+1] prefix of send over chunks
    std::vector<int> send_off;  // [E]
    std::vector<int> grp_rows;  // [n][E_l]  (table order: chunk-major)
    std::vector<int> grp_off;   // [n][E_l]  row offsets, buffer order (e_l, c)
    std::vector<int> src_off;   // [G][E_l][n] row offset of src's rows inside group (e_l, c)
    int rows_total = 0;

    void build(const int* h_send, const int* h_recv) {
        send.assign(h_send, h_send + E * n);
        recv.assign(h_recv, h_recv + G * E_l * n);
        S.assign(E * (n + 1), 0);
        send_off.assign(E, 0);
        plan_send(E, n, send.data(), S.data(), send_off.data());
        grp_rows.assign(n * E_l, 0);
        grp_off.assign(n * E_l, 0);
        src_off.assign(G * E_l * n, 0);
        rows_total = plan_recv(G, E_l, n, recv.data(), grp_rows.data(), grp_off.data(), src_off.data());
    }
};

// Every rank's send and receive layout from the all-gathered count matrix M [G][E][n] (peer
// transport: a pull needs the source rank's offsets).
struct GlobalPlan {
    int G = 0, E = 0, E_l = 0, n = 0;
    std::vector<int> M;
    std::vector<Plan> rank;     // rank[g] = g's Plan (its send counts and its receive counts)
    void build(int G_, int E_, int E_l_, int n_, const int* m) {
        G = G_; E = E_; E_l = E_l_; n = n_;
        M.assign(m, m + (size_t)G * E * n);
        rank.clear();
        for (int g = 0; g < G; ++g) {
            std::vector<int> recv((size_t)G * E_l * n);
            for (int src = 0; src < G; ++src)
                for (int el = 0; el < E_l; ++el)
                    for (int c = 0; c < n; ++c)
                        recv[((size_t)src * E_l + el) * n + c] = M[((size_t)src * E + g * E_l + el) * n + c];
            Plan pl{E, E_l, G, n};
            pl.build(&M[(size_t)g * E * n], recv.data());
            rank.push_back(pl);
        }
    }
    // pulls of rank `me` for chunks [c0, c1): toward_experts (dispatch-like: token-side source,
    // expert-side destination `dst`) or back (combine-like: expert-side source, token-side `dst`)
    std::vector<PeerCopy> pulls(int me, bool toward_experts, int c0, int c1, char* dst, size_t rowb) const {
        std::vector<PeerCopy> v;
        for (int p = 0; p < G; ++p)
            for (int el = 0; el < E_l; ++el)
                for (int ch = c0; ch < c1; ++ch) {
                    if (toward_experts) {          // rows p admitted to my expert e
                        const int e = me * E_l + el;
                        const Plan& src = rank[p];
                        const Plan& dstp = rank[me];
                        v.push_back({p, (size_t)(src.send_off[e] + src.S[e * (n + 1) + ch]) * rowb,
                                     dst + (size_t)(dstp.grp_off[ch * E_l + el] + dstp.src_off[(p * E_l + el) * n + ch]) * rowb,
                                     (size_t)M[((size_t)p * E + e) * n + ch] * rowb});
                    } else {                       // my rows back from expert e on rank p
                        const int e = p * E_l + el;
                        const Plan& src = rank[p];
                        const Plan& dstp = rank[me];
                        v.push_back({p, (size_t)(src.grp_off[ch * E_l + el] + src.src_off[(me * E_l + el) * n + ch]) * rowb,
                                     dst + (size_t)(dstp.send_off[e] + dstp.S[e * (n + 1) + ch]) * rowb,
                                     (size_t)M[((size_t)me * E + e) * n + ch] * rowb});
                    }
                }
        return v;
    }
};

// K6 for the tokens of chunk cc of nc (nc == 1: all tokens): dx = expert path + gate term.
lancet_status gate_backward_dx(lancet_ctx* c, const DispatchArgs& da, const void* dxe, void* dx,
                               cudaStream_t s, int cc, int nc, int* L)
{
    const int T = c->T, d = c->cfg.d_model, E = c->cfg.n_experts;
    const int t0 = chunk_start(T, nc, cc), t1 = chunk_start(T, nc, cc + 1);
    OpScope op(c, "unpermute_gate_bwd", s == c->s_comp ? 0 : 2, nc > 1 ? cc : -1, s);
    if (cc == 0 && gate_bwd_needs_wgT(d, E)) *L += launch_wg_transpose(c->wg, d, E, c->wgT, s);
    *L += launch_unpermute_gate_bwd(da, dxe, c->prow, c->dlogit, c->wg, c->wgT, dx, t0, t1, c->num_sms, c->bf16, s);
    CHECK_LAUNCH();
    return LANCET_OK;
}

// K7: dWg = x^T dlogit over all tokens (after every K5 has written its dlogit rows).
lancet_status gate_backward_dwg(lancet_ctx* c, float* dwg, cudaStream_t s, int* L)
{
    OpScope op(c, "gate_dwg", s == c->s_comp ? 0 : 2, -1, s);
    *L += launch_dwg(c->x, c->dlogit, c->T, c->cfg.d_model, c->cfg.n_experts, c->dwg_partial, dwg, c->bf16, c->num_sms, s);
    CHECK_LAUNCH();
    return LANCET_OK;
}

__global__ void send_counts_kernel(const int* __restrict__ S, int E, int n, int* __restrict__ out)
{
    pdl_wait();   // programmatic dependent launch: predecessor's writes visible
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= E * n) return;
    const int e = q / n, c = q % n;
    out[q] = S[e * (n + 1) + c + 1] - S[e * (n + 1) + c];
}


// ---- push mode (LANCET_FLAG_PEER_PUSH on the peer transport) -------------------------------
// All four exchanges are fused into the token kernels over peer memory: K3 writes each admitted
// row into the owner's receive buffer (dispatch), K4 reads the expert outputs where the owners'
// fc2 wrote them (combine), K5 writes its dO rows into the owners' dO buffers (backward #1) and
// K6 reads the dX rows where the owners' dfc1 wrote them (backward #2).  The exchange plan is
// built on the device from the gathered count matrix and every flag is a kernel (peer.cu
// dev_*), so nothing waits on the host: the step is graph-capturable.
//
// Streams (S1 / S2): the compute stream runs routing, the plan and
// the expert GEMMs of chunk after chunk; the comm stream runs the fused exchange kernels --
// chunk c+1's push and chunk c-1's combine under chunk c's GEMMs, on the SMs the persistent
// GEMMs leave free (gemm_sms = all - LANCET_COMM_SMS by default).  LANCET_FLAG_SERIAL puts
// everything on one stream with the chunks merged (the unoverlapped baseline).

#define DEV(call)                                                                       \
    do {                                                                                \
        if (call) return fail(c, LANCET_ERR_CUDA, std::string(#call) + ": " +           \
                                                     cudaGetErrorString(cudaGetLastError())); \
    } while (0)

// push mode with the device-side chunk pipeline in the GEMMs (ChunkSync): tcgen05 GEMMs, one
// launch over all chunks (<= 128 groups), not the serial baseline, not the per-chunk-launch A/B
bool push_pipelined(const lancet_ctx* c)
{
    return c->bf16 && c->cfg.act != LANCET_ACT_IDENTITY_EXPERT &&
           !(c->cfg.flags & (LANCET_FLAG_SERIAL | LANCET_FLAG_SIMT_GEMM | LANCET_FLAG_CHUNK_LAUNCHES)) &&
           c->n * c->E_l <= kTcMaxGroups;
}

// Per-chunk GEMM launches of the push pipeline: chunk ch on sc (even) or s_comp2 (odd), both
// ordered after everything already on sc, and sc ordered after all of them at the end.
template <typename F>
lancet_status per_chunk_alternating(lancet_ctx* c, int n, cudaStream_t sc, F&& body)
{
    cudaEvent_t ev_in = c->ev_pool[3], ev_out = c->ev_pool[4];
    CK(cudaEventRecord(ev_in, sc));
    CK(cudaStreamWaitEvent(c->s_comp2, ev_in, 0));
    for (int ch = 0; ch < n; ++ch) {
        lancet_status st = body(ch, (ch & 1) ? c->s_comp2 : sc);
        if (st) return st;
    }
    CK(cudaEventRecord(ev_out, c->s_comp2));
    CK(cudaStreamWaitEvent(sc, ev_out, 0));
    return LANCET_OK;
}

int push_group_rows_bound(const lancet_ctx* c)
{
    // a group (e_l, c) holds at most min(C, T) <= max_tokens rows of each source rank
    return std::min(c->rows_exp, round_up(c->world * c->cfg.max_tokens, kRowAlign));
}

lancet_status forward_push(lancet_ctx* c, const RouteArgs& ra, const DispatchArgs& da, const void* x,
                           void* y, cudaStream_t s, int& L)
{
    lancet::PeerLinks* pr = c->peer;
    const int E = c->cfg.n_experts, E_l = c->E_l, n = c->n, T = c->T;
    const bool ident = c->cfg.act == LANCET_ACT_IDENTITY_EXPERT;
    const bool serial = c->cfg.flags & LANCET_FLAG_SERIAL;
    const bool nocomm = c->cfg.flags & LANCET_FLAG_NO_COMM;
    cudaStream_t sc = c->s_comp, sm = serial ? c->s_comp : c->s_comm;
    using namespace lancet;
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(sc, c->ev_fork, 0));
    CK(cudaStreamWaitEvent(c->s_comm, c->ev_fork, 0));
    // a forward without backward: release the owners' outputs the last forward read (with
    // that step's number: before the bump)
    if (c->out_consume_pending) {
        DEV(dev_signal(c, 1, PK_OUT, 0, sc));
        c->out_consume_pending = false;
    }
    ++pr->seq;
    DEV(dev_seq_bump(c, sc));
    // this rank's receive buffer is free for the step's pushes: its readers (the previous
    // step's GEMMs) are behind on this stream
    DEV(dev_signal(c, 0, PK_XEFREE, 0, sc));
    { OpScope op(c, "gate", 0, -1, sc); L += launch_routing(ra, c->bf16, sc); }
    int* d_send = c->counts_dev;
    launch_k(send_counts_kernel, ceil_div(E * n, 256), 256, 0, sc, c->S, E, n, d_send);
    ++L;
    CHECK_LAUNCH();
    {   // C1: the size exchange -- the count matrix all-gathered through peer memory
        OpScope op(c, "a2a_counts", 1, -1, sc);
        DEV(dev_counts(c, d_send, n, sc));
        L += 2;
    }
    DEV(dev_plan(c, n, sc));
    ++L;
    int* d_grp_rows = c->grp_dev;
    int* d_grp_off = c->grp_dev + n * E_l;
    L += launch_zero_pads(c->xe, c->cfg.d_model, d_grp_off, d_grp_rows, n * E_l, (int)c->elt, sc);
    CHECK_LAUNCH();
    cudaEvent_t ev_plan = c->ev_pool[0];
    CK(cudaEventRecord(ev_plan, sc));
    CK(cudaStreamWaitEvent(sm, ev_plan, 0));
    // K3 + C2-d fused: chunk c's rows go straight to the owners' receive buffers
    DEV(dev_wait(c, 0, PK_XEFREE, 0, TGT_STEP, sm));
    cudaEvent_t ev_first = c->ev_pool[2];
    for (int ch = 0; ch < n; ++ch) {
        {
            OpScope op(c, "a2a_dispatch_push", 1, serial ? -1 : ch, sm);
            if (!nocomm)
                L += launch_permute_push(da, x, chunk_start(T, n, ch), chunk_start(T, n, ch + 1), E_l,
                                         pr->d_push_base + (size_t)ch * E, pr->d_xe, c->bf16, sm);
            else if (ch == 0)       // NO_COMM (timing): the same permute into local rows
                L += launch_permute(da, x, c->xs, c->bf16, sm);
        }
        CHECK_LAUNCH();
        DEV(dev_signal(c, 0, PK_PUSH, ch, sm));
        if (ch == 0) CK(cudaEventRecord(ev_first, sm));
    }
    const int nc = serial ? 1 : n;
    const int mr = push_group_rows_bound(c);
    if (push_pipelined(c)) {
        // one fc1 and one fc2 launch over all chunks: fc1's TMA producer waits for chunk c's
        // rows of every rank on the device, fc2 publishes chunk c's outputs as soon as its last
        // tile is stored -- chunk c+1's dispatch runs under chunk c's GEMMs and chunk c's
        // combine under chunk c+1's, with no launch boundary between chunks
        DEV(dev_wait(c, 1, PK_OUT, 0, TGT_PREV, sc));   // peers done with last step's outputs
        // the persistent fc1 starts once this rank's chunk-0 push is done (so that push has
        // every SM; fc1's CTAs would otherwise hold them while waiting for chunk 0), and waits
        // for the rest -- every rank's chunk c -- on the device
        CK(cudaStreamWaitEvent(sc, ev_first, 0));
        const ChunkSync w = chunk_sync(c, PK_PUSH);
        lancet_status st = expert_fc1(c, d_grp_rows, d_grp_off, n * E_l, mr, sc, -1, &L, &w);
        if (st) return st;
        // fc2 per chunk, each published by a flag kernel once it completed (kernel completion
        // makes its TMA-stored rows visible to the peers' fused combine); even chunks on the
        // compute stream, odd ones on a second one, so a chunk's last wave overlaps the next
        st = per_chunk_alternating(c, n, sc, [&](int ch, cudaStream_t st_) -> lancet_status {
            lancet_status r = expert_fc2(c, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l, mr, st_, ch, &L);
            if (r) return r;
            DEV(dev_signal(c, 0, PK_OUT, ch, st_));
            return LANCET_OK;
        });
        if (st) return st;
    } else {
        for (int cc = 0; cc < nc; ++cc) {
            const int c0 = serial ? 0 : cc, c1 = serial ? n : cc + 1;
            for (int ch = c0; ch < c1; ++ch) DEV(dev_wait(c, 0, PK_PUSH, ch, TGT_STEP, sc));
            if (cc == 0) DEV(dev_wait(c, 1, PK_OUT, 0, TGT_PREV, sc));   // peers done with last step's outputs
            if (!ident) {
                lancet_status st = expert_forward(c, d_grp_rows + c0 * E_l, d_grp_off + c0 * E_l, (c1 - c0) * E_l,
                                                  mr, sc, serial ? -1 : cc, &L);
                if (st) return st;
            }
            DEV(dev_signal(c, 0, PK_OUT, cc, sc));
        }
    }
    // C2-c + K4 fused: chunk c's tokens gather the expert outputs from the owners' buffers
    for (int cc = 0; cc < nc; ++cc) {
        const int c0 = serial ? 0 : cc, c1 = serial ? n : cc + 1;
        DEV(dev_wait(c, 0, PK_OUT, cc, TGT_STEP, sm));
        for (int ch = c0; ch < c1; ++ch) {
            OpScope op(c, "a2a_combine_fused", 1, serial ? -1 : ch, sm);
                // NO_COMM (timing): the same gather from local rows
            L += launch_combine(da, c->comb, y, chunk_start(T, n, ch), chunk_start(T, n, ch + 1), c->bf16, sm,
                                nocomm ? nullptr : pr->d_push_base + (size_t)ch * E, pr->d_outsrc, E_l);
        }
        CHECK_LAUNCH();
    }
    c->out_consume_pending = true;
    CK(cudaEventRecord(c->ev_join, sc));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    if (sm != sc) {
        cudaEvent_t e2 = c->ev_pool[1];
        CK(cudaEventRecord(e2, sm));
        CK(cudaStreamWaitEvent(s, e2, 0));
    }
    return LANCET_OK;
}

lancet_status backward_push(lancet_ctx* c, const DispatchArgs& da, const void* dy, void* dx, float* dwg,
                            float* dw1, float* dw2, int renorm, cudaStream_t s, int& L)
{
    using namespace lancet;
    lancet::PeerLinks* pr = c->peer;
    const int E = c->cfg.n_experts, E_l = c->E_l, n = c->n, T = c->T, d = c->cfg.d_model;
    const bool ident = c->cfg.act == LANCET_ACT_IDENTITY_EXPERT;
    const bool serial = c->cfg.flags & LANCET_FLAG_SERIAL;
    const bool late_dw = serial || (c->cfg.flags & LANCET_FLAG_NO_DW_OVERLAP);
    const bool nocomm = c->cfg.flags & LANCET_FLAG_NO_COMM;
    cudaStream_t sc = c->s_comp, sm = serial ? c->s_comp : c->s_comm;
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(sc, c->ev_fork, 0));
    CK(cudaStreamWaitEvent(c->s_comm, c->ev_fork, 0));
    int* d_grp_rows = c->grp_dev;
    int* d_grp_off = c->grp_dev + n * E_l;
    // this rank's dO buffer is free (its readers, the previous step's GEMMs, are behind on
    // this stream); its pads must be zero for the K-grouped dW GEMMs
    DEV(dev_signal(c, 0, PK_DOUTFREE, 0, sc));
    L += launch_zero_pads(c->dout, d, d_grp_off, d_grp_rows, n * E_l, (int)c->elt, sc);
    CHECK_LAUNCH();
    cudaEvent_t ev0 = c->ev_pool[0];
    CK(cudaEventRecord(ev0, sc));
    CK(cudaStreamWaitEvent(sm, ev0, 0));
    // K5 + C2-b1 fused: dO rows straight into the owners' dO buffers; o read in place
    DEV(dev_wait(c, 0, PK_DOUTFREE, 0, TGT_STEP, sm));
    for (int ch = 0; ch < n; ++ch) {
        {
            OpScope op(c, "a2a_bwd_dispatch_push", 1, serial ? -1 : ch, sm);
            L += launch_combine_bwd(da, dy, c->comb, c->g, c->dcomb, chunk_start(T, n, ch), chunk_start(T, n, ch + 1),
                                    false, c->logits, renorm, c->dlogit, c->prow, c->bf16, sm,
                                    nocomm ? nullptr : pr->d_push_base + (size_t)ch * E, pr->d_dout, E_l,
                                    nocomm ? nullptr : pr->d_outsrc);
        }
        CHECK_LAUNCH();
        DEV(dev_signal(c, 0, PK_PUSH2, ch, sm));
        if (ch == 0) CK(cudaEventRecord(c->ev_pool[2], sm));
    }
    DEV(dev_signal(c, 1, PK_OUT, 0, sm));   // the owners' outputs are consumed (K4 and K5 done)
    c->out_consume_pending = false;
    lancet_status st = gate_backward_dwg(c, dwg, sm, &L);     // K7 beside the dX GEMMs
    if (st) return st;
    // dX GEMMs per chunk, each followed by its dW GEMMs
    const int nc = serial ? 1 : n;
    const int mr = push_group_rows_bound(c);
    if (push_pipelined(c)) {
        // one dfc2 and one dfc1 launch over all chunks (dfc2 waits for chunk c's dO rows on the
        // device, dfc1 publishes chunk c's dX rows as soon as they are stored), then the dW
        // GEMMs once over every chunk's rows (merged table: one K range per expert, no per-chunk
        // fp32 reduce-add) -- under the fused dX return of the last chunks
        DEV(dev_wait(c, 1, PK_DXE, 0, TGT_LAST_BWD, sc));   // last backward's K6 readers done
        CK(cudaStreamWaitEvent(sc, c->ev_pool[2], 0));          // this rank's chunk-0 K5 push done
        const ChunkSync w = chunk_sync(c, PK_PUSH2);
        st = expert_dfc2(c, c->dout, d_grp_rows, d_grp_off, n * E_l, mr, sc, -1, &L, &w);
        if (st) return st;
        st = per_chunk_alternating(c, n, sc, [&](int ch, cudaStream_t st_) -> lancet_status {
            lancet_status r = expert_dfc1(c, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l, mr, st_, ch, &L);
            if (r) return r;
            DEV(dev_signal(c, 0, PK_DXE, ch, st_));
            return LANCET_OK;
        });
        if (st) return st;
        const int* merged = c->grp_dev + 2 * kMaxChunks * E_l;
        st = expert_backward_dw(c, c->dout, merged, merged + E_l, E_l, dw1, dw2, 0, sc, -1, &L);
        if (st) return st;
    } else
    for (int cc = 0; cc < nc; ++cc) {
        const int c0 = serial ? 0 : cc, c1 = serial ? n : cc + 1;
        for (int ch = c0; ch < c1; ++ch) DEV(dev_wait(c, 0, PK_PUSH2, ch, TGT_STEP, sc));
        if (cc == 0) DEV(dev_wait(c, 1, PK_DXE, 0, TGT_LAST_BWD, sc));   // last backward's K6 readers done
        if (!ident) {
            st = expert_backward_dx(c, c->dout, d_grp_rows + c0 * E_l, d_grp_off + c0 * E_l, (c1 - c0) * E_l, mr, sc,
                                    serial ? -1 : cc, &L);
            if (st) return st;
        }
        DEV(dev_signal(c, 0, PK_DXE, cc, sc));
        if (!ident && !late_dw)
            for (int ch = c0; ch < c1; ++ch) {
                st = expert_backward_dw(c, c->dout, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l, dw1, dw2,
                                        ch > 0, sc, ch, &L);
                if (st) return st;
            }
    }
    if (!ident && late_dw && !push_pipelined(c))
        for (int ch = 0; ch < n; ++ch) {
            st = expert_backward_dw(c, c->dout, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l, dw1, dw2, ch > 0,
                                    sc, ch, &L);
            if (st) return st;
        }
    // C2-b2 + K6 fused: chunk c's tokens sum their dX rows where the owners' dfc1 wrote them
    for (int cc = 0; cc < nc; ++cc) {
        const int c0 = serial ? 0 : cc, c1 = serial ? n : cc + 1;
        DEV(dev_wait(c, 0, PK_DXE, cc, TGT_STEP, sm));
        for (int ch = c0; ch < c1; ++ch) {
            const int t0 = chunk_start(T, n, ch), t1 = chunk_start(T, n, ch + 1);
            OpScope op(c, "a2a_bwd_combine_fused", 1, serial ? -1 : ch, sm);
            if (ch == 0 && gate_bwd_needs_wgT(d, E)) L += launch_wg_transpose(c->wg, d, E, c->wgT, sm);
            L += launch_unpermute_gate_bwd(da, c->dxcomb, c->prow, c->dlogit, c->wg, c->wgT, dx, t0, t1, c->num_sms,
                                           c->bf16, sm, nocomm ? nullptr : (const char* const*)pr->d_dxesrc);
        }
        CHECK_LAUNCH();
    }
    DEV(dev_signal(c, 1, PK_DXE, 0, sm, /*mark_bwd=*/true));
    c->bwd_seq = pr->seq;
    CK(cudaEventRecord(c->ev_join, sc));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    if (sm != sc) {
        cudaEvent_t e2 = c->ev_pool[1];
        CK(cudaEventRecord(e2, sm));
        CK(cudaStreamWaitEvent(s, e2, 0));
    }
    return LANCET_OK;
}
}  // namespace


// =========================================================================================
// Block mode (internal.h): the MoE forward whose input arrives chunk by chunk
// =========================================================================================
namespace lancet {

lancet_status record_error(lancet_ctx* c, lancet_status st, const std::string& msg) { return fail(c, st, msg); }
lancet_status ctx_ready(lancet_ctx* c) { return check_ready(c); }
int capacity_rows(int T, int k, int E, double cf) { return capacity_of(T, k, E, cf); }

size_t op_begin(lancet_ctx* c, const char* name, int lane, int chunk, cudaStream_t s)
{
    OpScope op(c, name, lane, chunk, s);
    const size_t h = op.i;
    op.i = (size_t)-1;          // the end event is recorded by op_end
    return h;
}

void op_end(lancet_ctx* c, size_t h, cudaStream_t s)
{
    if (h != (size_t)-1) cudaEventRecord(c->ops[h].end, s);
}

lancet_status dense_gemm(lancet_ctx* c, const void* A, long a_rows, const void* B, int N, int K, void* C,
                         long c_rows, const int* grp_rows, const int* grp_off, int n_groups, int max_rows,
                         cudaStream_t s, int* launches)
{
    GemmArgs a{};
    a.mode = GEMM_M_GROUPED; a.n_groups = n_groups; a.gpw = n_groups; a.n_weights = 1;
    a.grp_rows = grp_rows; a.grp_off = grp_off; a.max_rows = max_rows; a.act = 0;
    a.A = A; a.lda = K; a.a_rows = a_rows; a.a_mn = false;
    a.B = B; a.ldb = K; a.b_group_stride = 0; a.b_rows = N; a.b_mn = false;
    a.C = C; a.C2 = nullptr; a.ldc = N; a.c_rows = c_rows; a.N = N; a.K = K; a.epi = EPI_STORE;
    return run_gemm(c, a, s, launches);
}

lancet_status dense_gemm_bmn(lancet_ctx* c, const void* A, long a_rows, const void* B, int N, int K, void* C,
                             long c_rows, const int* grp_rows, const int* grp_off, int n_groups, int max_rows,
                             cudaStream_t s, int* launches)
{
    GemmArgs a{};
    a.mode = GEMM_M_GROUPED; a.n_groups = n_groups; a.gpw = n_groups; a.n_weights = 1;
    a.grp_rows = grp_rows; a.grp_off = grp_off; a.max_rows = max_rows; a.act = 0;
    a.A = A; a.lda = K; a.a_rows = a_rows; a.a_mn = false;
    a.B = B; a.ldb = N; a.b_group_stride = 0; a.b_rows = K; a.b_mn = true;
    a.C = C; a.C2 = nullptr; a.ldc = N; a.c_rows = c_rows; a.N = N; a.K = K; a.epi = EPI_STORE;
    return run_gemm(c, a, s, launches);
}

lancet_status dense_wgrad(lancet_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int N, long rows_ext,
                          const int* grp_rows, const int* grp_off, float* C, cudaStream_t s, int* launches)
{
    GemmArgs a{};
    a.mode = GEMM_K_GROUPED; a.n_groups = 1; a.gpw = 1; a.n_weights = 1;
    a.grp_rows = grp_rows; a.grp_off = grp_off; a.accumulate = 0;
    a.a_mn = true; a.b_mn = true; a.epi = EPI_F32; a.b_group_stride = 0;
    a.a_rows = rows_ext; a.b_rows = rows_ext;
    a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
    a.C = C; a.ldc = N; a.c_group_stride = (long)M * N; a.M = M; a.N = N;
    return run_gemm(c, a, s, launches);
}

// Forward of the MoE layer in block mode (push transport; LANCET_FLAG_PEER_PUSH).  Per chunk
// ch, stage by stage (S1 with the non-MoE part in the pipeline, fig:part_all):
//   producer stream:  produce(ch) [the block's LN1 / attention / projections / LN2], then the
//                     gate of chunk ch with the carried capacity state (K1 + K2 in carry mode);
//   comm stream:      size exchange of chunk ch (column ch of the count matrix), the
//                     chunk's plan (static regions: final before later chunks are gated), pad
//                     zeroing, and the fused permute + dispatch push of chunk ch;
//   compute stream:   once every rank's rows of chunk ch landed: fc1, fc2 of chunk ch;
//   combine stream:   once every owner's outputs of chunk ch are stored: the fused combine
//                     (+ residual) of chunk ch.
// The producer never waits for the exchange: chunk ch+1's attention runs while chunk ch is
// exchanged and its experts run.  The resulting routing, plan tables, buffers and flags are
// those of forward_push, so lancet_moe_backward works unchanged.
lancet_status moe_forward_chunked(lancet_ctx* c, const void* x, const float* wg, const void* w1, const void* w2,
                                  int T, int k, double cf, void* y, const ChunkedInput& in, cudaStream_t s)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    const int E = c->cfg.n_experts, d = c->cfg.d_model, E_l = c->E_l, n = in.n;
    if (!c->ep || !c->push || !c->peer) return fail(c, LANCET_ERR_UNSUPPORTED, "block mode needs the peer transport in push mode");
    if (!c->peer_ready) return fail(c, LANCET_ERR_STATE, "peer transport: lancet_peer_import not called");
    if (!c->bf16 || c->cfg.act == LANCET_ACT_IDENTITY_EXPERT) return fail(c, LANCET_ERR_UNSUPPORTED, "block mode: bf16 experts only");
    if (c->cfg.flags & LANCET_FLAG_GATE_BPR)
        return fail(c, LANCET_ERR_UNSUPPORTED, "Batch Prioritized Routing needs the whole batch: no partition before the gate (PAPER.md L270-L271)");
    if (T < 1 || T > c->cfg.max_tokens) return fail(c, LANCET_ERR_ARG, "T must be in [1, max_tokens]");
    if (k < 1 || k > c->cfg.max_k || k > E) return fail(c, LANCET_ERR_ARG, "k must be in [1, min(E, max_k)]");
    if (!(cf > 0.0) || !std::isfinite(cf) || cf > in.cf_max) return fail(c, LANCET_ERR_ARG, "capacity_factor must be in (0, max_capacity_factor]");
    if (n < 1 || n > c->cfg.max_chunks || in.bounds[0] != 0 || in.bounds[n] != T)
        return fail(c, LANCET_ERR_ARG, "bad chunk bounds");
    for (int ch = 0; ch < n; ++ch)
        if (in.bounds[ch + 1] - in.bounds[ch] != chunk_start(T, n, ch + 1) - chunk_start(T, n, ch))
            return fail(c, LANCET_ERR_ARG, "block chunks must be the layer's chunks (R9)");
    if (c->dw_pending) return fail(c, LANCET_ERR_STATE, "deferred dW GEMMs of the last backward were never enqueued");
    // static receive regions per local expert: every source admits <= C(max_tokens) rows of an
    // expert over all chunks, plus < 128 pad rows per chunk group
    const int Cb = capacity_of(c->cfg.max_tokens, k, E, cf);
    const long region = round_up((int)std::min<long>((long)c->world * Cb + 127L * n, 1L << 28), kRowAlign);
    if ((long)E_l * region > c->peer->rows_cap)
        return fail(c, LANCET_ERR_ARG, "block mode: the expert-side buffers hold " + std::to_string(c->peer->rows_cap) +
                                           " rows, the static regions need " + std::to_string((long)E_l * region));
    lancet::g_pdl = (c->cfg.flags & LANCET_FLAG_NO_PDL) == 0;
    c->have_fwd = false;
    c->x = x; c->wg = wg; c->w1 = w1; c->w2 = w2;
    c->T = T; c->k = k; c->n = n; c->cf = cf;
    c->C = capacity_of(T, k, E, cf);
    c->launches_fwd = 0;
    int& L = c->launches_fwd;
    if (!c->tl_accumulate) {
        c->ops.clear();
        c->tl_used = 0;
        if (c->cfg.flags & LANCET_FLAG_TIMELINE) CK(cudaEventRecord(c->ev_tl_base, s));
    }
    lancet::PeerLinks* pr = c->peer;
    const bool serial = c->cfg.flags & LANCET_FLAG_SERIAL;
    const bool nocomm = c->cfg.flags & LANCET_FLAG_NO_COMM;
    cudaStream_t sp = serial ? c->s_comp : in.s_pre;
    cudaStream_t sm = serial ? c->s_comp : c->s_comm;
    cudaStream_t sc = c->s_comp;
    cudaStream_t sb = serial ? c->s_comp : c->s_comp2;
    size_t ev_i = 0;
    auto next_ev = [&]() { return c->ev_pool[ev_i++]; };
    CK(cudaEventRecord(c->ev_fork, s));
    for (cudaStream_t q : {sp, sm, sc, sb}) CK(cudaStreamWaitEvent(q, c->ev_fork, 0));
    if (c->out_consume_pending) {
        DEV(dev_signal(c, 1, PK_OUT, 0, sc));
        c->out_consume_pending = false;
    }
    ++pr->seq;
    DEV(dev_seq_bump(c, sc));
    DEV(dev_signal(c, 0, PK_XEFREE, 0, sc));    // this rank's receive buffer is free for the step
    int* carry = c->carry;
    CK(cudaMemsetAsync(carry, 0, sizeof(int) * E, sc));
    cudaEvent_t ev_start = next_ev();
    CK(cudaEventRecord(ev_start, sc));
    for (cudaStream_t q : {sp, sm, sb}) CK(cudaStreamWaitEvent(q, ev_start, 0));

    RouteArgs ra{};
    ra.wg = wg; ra.d = d; ra.E = E; ra.k = k; ra.C = c->C; ra.n_chunks = 1;
    ra.renorm = (c->cfg.flags & LANCET_FLAG_RENORMALIZE) ? 1 : 0;
    ra.hist = c->hist; ra.S = c->S; ra.send_rows = c->send_rows; ra.send_off = c->send_off;
    ra.random = (c->cfg.flags & LANCET_FLAG_GATE_RANDOM) ? 1 : 0;
    ra.seed = c->gate_seed;
    ra.carry_n = n; ra.carry_counts = c->counts_dev;
    DispatchArgs da{T, k, d, E, c->idx, c->slot, c->w, c->send_off, c->send_rows};
    int* d_grp_rows = c->grp_dev;
    int* d_grp_off = c->grp_dev + n * E_l;
    const int mr = push_group_rows_bound(c);
    const size_t xrow = (size_t)d * c->elt;
    for (int ch = 0; ch < n; ++ch) {
        const int t0 = in.bounds[ch], t1 = in.bounds[ch + 1];
        // ---- producer: the chunk's MoE input, then its gate with the carried capacity state
        if (in.ev_in) CK(cudaStreamWaitEvent(sp, in.ev_in[ch], 0));
        st = in.produce(ch, t0, t1, sp);
        if (st) return st;
        ra.x = (const char*)x + (size_t)t0 * xrow;
        ra.T = t1 - t0; ra.t_base = t0;
        ra.logits = c->logits + (size_t)t0 * E; ra.idx = c->idx + (size_t)t0 * k; ra.w = c->w + (size_t)t0 * k;
        ra.slot = c->slot + (size_t)t0 * k;
        ra.carry_in = carry + (size_t)ch * E; ra.carry_out = carry + (size_t)(ch + 1) * E; ra.carry_chunk = ch;
        { OpScope op(c, "gate", 0, ch, sp); L += launch_routing(ra, c->bf16, sp); }
        CHECK_LAUNCH();
        cudaEvent_t ev_route = next_ev();
        CK(cudaEventRecord(ev_route, sp));
        // ---- comm: sizes of chunk ch, its plan, the fused permute + dispatch push
        CK(cudaStreamWaitEvent(sm, ev_route, 0));
        {
            OpScope op(c, "a2a_counts", 1, ch, sm);
            DEV(dev_counts_chunk(c, c->counts_dev, n, ch, sm));
            L += 2;
        }
        DEV(dev_plan_chunk(c, n, ch, (int)region, sm));
        ++L;
        L += launch_zero_pads(c->xe, d, d_grp_off + ch * E_l, d_grp_rows + ch * E_l, E_l, (int)c->elt, sm);
        CHECK_LAUNCH();
        cudaEvent_t ev_plan = next_ev();
        CK(cudaEventRecord(ev_plan, sm));
        if (ch == 0) DEV(dev_wait(c, 0, PK_XEFREE, 0, TGT_STEP, sm));
        {
            OpScope op(c, "a2a_dispatch_push", 1, ch, sm);
            if (!nocomm)
                L += launch_permute_push(da, x, t0, t1, E_l, pr->d_push_base + (size_t)ch * E, pr->d_xe, c->bf16, sm);
        }
        CHECK_LAUNCH();
        DEV(dev_signal(c, 0, PK_PUSH, ch, sm));
        // ---- compute: the experts of chunk ch once every rank's rows landed
        CK(cudaStreamWaitEvent(sc, ev_plan, 0));
        DEV(dev_wait(c, 0, PK_PUSH, ch, TGT_STEP, sc));
        if (ch == 0) DEV(dev_wait(c, 1, PK_OUT, 0, TGT_PREV, sc));   // peers done with last step's outputs
        st = expert_forward(c, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l, mr, sc, ch, &L);
        if (st) return st;
        DEV(dev_signal(c, 0, PK_OUT, ch, sc));
        // ---- combine: chunk ch's tokens gather their outputs from the owners (+ residual)
        CK(cudaStreamWaitEvent(sb, ev_plan, 0));
        DEV(dev_wait(c, 0, PK_OUT, ch, TGT_STEP, sb));
        {
            OpScope op(c, "a2a_combine_fused", 1, ch, sb);
            L += launch_combine(da, c->comb, y, t0, t1, c->bf16, sb, nocomm ? nullptr : pr->d_push_base + (size_t)ch * E,
                                pr->d_outsrc, E_l, in.resid);
        }
        CHECK_LAUNCH();
        if (in.ev_out) CK(cudaEventRecord(in.ev_out[ch], sb));
    }
    c->out_consume_pending = true;
    c->n_groups = n * E_l;
    if (in.join) {
        for (cudaStream_t q : {sp, sm, sc, sb}) {
            cudaEvent_t e = next_ev();
            CK(cudaEventRecord(e, q));
            CK(cudaStreamWaitEvent(s, e, 0));
        }
    }
    c->have_fwd = true;
    return LANCET_OK;
}

lancet_status moe_join(lancet_ctx* c, cudaStream_t extra, cudaStream_t s)
{
    int i = (int)c->ev_pool.size() - 6;
    for (cudaStream_t q : {extra, c->s_comp, c->s_comm, c->s_comp2, c->s_gate}) {
        if (!q) continue;
        cudaEvent_t e = c->ev_pool[i++];
        CK(cudaEventRecord(e, q));
        CK(cudaStreamWaitEvent(s, e, 0));
    }
    return LANCET_OK;
}

}  // namespace lancet

// =========================================================================================
// C-ABI
// =========================================================================================

LANCET_API int32_t lancet_abi_version(void) { return LANCET_ABI_VERSION; }

LANCET_API const char* lancet_last_error(const lancet_ctx* ctx)
{
    return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

LANCET_API lancet_status lancet_nccl_unique_id(void* id_out)
{
    if (!id_out) return fail(nullptr, LANCET_ERR_ARG, "id_out is NULL");
    std::string err;
    if (nccl_unique_id(id_out, err)) return fail(nullptr, LANCET_ERR_NCCL, err);
    return LANCET_OK;
}

LANCET_API lancet_status lancet_create(lancet_ctx** out, int32_t world, int32_t rank,
                                       int32_t cuda_device, const void* nccl_id,
                                       const lancet_layer_config* cfg)
{
    if (!out) return fail(nullptr, LANCET_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, LANCET_ERR_ARG, "bad world/rank");
    const bool ep = world > 1 || (cfg && (cfg->flags & LANCET_FLAG_FORCE_EP));
    if (ep && !nccl_id) return fail(nullptr, LANCET_ERR_ARG, "world > 1 (or FORCE_EP) needs an NCCL id");
    lancet_status st = validate_cfg(cfg, world);
    if (st) return st;
    auto* c = new lancet_ctx();
    // NCCL data plane: buffers from ncclMemAlloc, registered with the communicator below
    // (LANCET_NCCL_REGISTER=0: plain cudaMalloc, unregistered -- the A/B)
    const char* reg_env = getenv("LANCET_NCCL_REGISTER");
    c->nccl_mem = ep && !(reg_env && reg_env[0] == '0');
    st = create_common(c, world, rank, cuda_device, cfg);
    if (!st && ep) {
        std::string err;
        c->comm = make_nccl_transport(world, rank, nccl_id, LANCET_COMM_SMS, err);
        if (!c->comm) st = fail(c, LANCET_ERR_NCCL, err);
        else if (c->comm->check_same(cfg_hash(*cfg), c->s_comm, err)) st = fail(c, LANCET_ERR_ARG, err);
        else
            for (const lancet::DevBuf& b : c->allocs)
                if (b.nccl && c->comm->register_buffer(b.p, b.bytes) == 0) ++c->nccl_registered;
    }
    if (st) {
        g_thread_err = c->err;
        lancet_destroy(c);
        return st;
    }
    *out = c;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_local_group_create(lancet_local_group** out, int32_t world)
{
    if (!out || world < 1) return fail(nullptr, LANCET_ERR_ARG, "bad arguments");
    *out = new lancet_local_group{local_group_create(world), world};
    return LANCET_OK;
}

LANCET_API lancet_status lancet_local_group_destroy(lancet_local_group* g)
{
    if (g) {
        local_group_destroy(g->impl);
        delete g;
    }
    return LANCET_OK;
}

LANCET_API lancet_status lancet_create_local(lancet_ctx** out, lancet_local_group* group,
                                             int32_t rank, int32_t cuda_device,
                                             const lancet_layer_config* cfg)
{
    if (!out || !group) return fail(nullptr, LANCET_ERR_ARG, "bad arguments");
    *out = nullptr;
    const int world = group->world;
    if (rank < 0 || rank >= world) return fail(nullptr, LANCET_ERR_ARG, "bad rank");
    lancet_status st = validate_cfg(cfg, world);
    if (st) return st;
    auto* c = new lancet_ctx();
    st = create_common(c, world, rank, cuda_device, cfg);
    if (!st && world > 1) {
        std::string err;
        c->comm = make_local_transport(group->impl, rank, err);
        if (!c->comm) st = fail(c, LANCET_ERR_ARG, err);
        else if (c->comm->check_same(cfg_hash(*cfg), c->s_comm, err)) st = fail(c, LANCET_ERR_ARG, err);
    }
    if (st) {
        g_thread_err = c->err;
        lancet_destroy(c);
        return st;
    }
    *out = c;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_create_peer(lancet_ctx** out, int32_t world, int32_t rank,
                                            int32_t cuda_device, const lancet_layer_config* cfg)
{
    return lancet::create_peer_ctx(out, world, rank, cuda_device, cfg, 0);
}

lancet_status lancet::create_peer_ctx(lancet_ctx** out, int world, int rank, int cuda_device,
                                      const lancet_layer_config* cfg, long min_rows)
{
    if (!out) return fail(nullptr, LANCET_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, LANCET_ERR_ARG, "bad world/rank");
    lancet_status st = validate_cfg(cfg, world);
    if (st) return st;
    lancet_layer_config cf2 = *cfg;
    cf2.flags |= LANCET_FLAG_FORCE_EP;                  // the expert-parallel path, even at world 1
    auto* c = new lancet_ctx();
    c->push = (cfg->flags & LANCET_FLAG_PEER_PUSH) != 0;
    st = create_common(c, world, rank, cuda_device, &cf2);
    if (!st && c->push) {
        // push mode: K5 hands K6 (owner, row) packed in one int32 (lancet::kPeerRowBits)
        const long rows = (long)world * cfg->max_tokens * cfg->max_k + (long)c->E_l * cfg->max_chunks * kRowAlign;
        if (rows >= (1L << kPeerRowBits) || world > (1 << (31 - kPeerRowBits)))
            st = fail(c, LANCET_ERR_ARG, "push mode: world * max_tokens * max_k must stay below 2^24 rows and world <= 128");
    }
    if (!st) {
        // the expert-side buffers are mapped by the peers: allocate them at their bound once
        // (every source sends at most max_tokens * max_k rows; + 128-row padding per group)
        const long rows = std::max(min_rows, (long)world * cfg->max_tokens * cfg->max_k +
                                                 (long)c->E_l * cfg->max_chunks * kRowAlign);
        if (rows > (1L << 30) || (c->push && rows >= (1L << kPeerRowBits)))
            st = fail(c, LANCET_ERR_ARG, "expert-side row bound too large");
        else st = ensure_expert_rows(c, (int)rows);
    }
    if (!st) {
        std::string err;
        if (peer_init(c, err)) st = fail(c, LANCET_ERR_CUDA, err);
        else {
            unsigned long long h = cfg_hash(*cfg);
            for (long v : {(long)cfg->max_tokens, (long)(cfg->flags & LANCET_FLAG_PEER_PUSH), (long)world, min_rows}) {
                h ^= (unsigned long long)v;
                h *= 1099511628211ull;
            }
            c->peer->cfg_hash = h;
            c->peer->rows_cap = c->rows_exp;
        }
    }
    if (st) {
        g_thread_err = c->err;
        lancet_destroy(c);
        return st;
    }
    *out = c;
    return LANCET_OK;
}

LANCET_API size_t lancet_peer_blob_bytes(void) { return peer_blob_bytes(); }

LANCET_API lancet_status lancet_peer_export(lancet_ctx* c, void* blob)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->peer || !blob) return fail(c, LANCET_ERR_ARG, "not a peer-transport context, or blob is NULL");
    std::string err;
    if (peer_export(c, blob, err)) return fail(c, LANCET_ERR_CUDA, err);
    return LANCET_OK;
}

LANCET_API lancet_status lancet_peer_import(lancet_ctx* c, const void* blobs)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->peer || !blobs) return fail(c, LANCET_ERR_ARG, "not a peer-transport context, or blobs is NULL");
    std::string err;
    if (peer_import(c, blobs, err)) return fail(c, LANCET_ERR_CUDA, err);
    c->peer_ready = true;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_destroy(lancet_ctx* c)
{
    if (!c) return LANCET_OK;
    cudaSetDevice(c->device);
    if (c->peer) {
        cudaDeviceSynchronize();
        if (!c->poisoned && c->peer_ready) lancet::peer_quiesce(c);
        peer_destroy(c);
    }
    if (c->comm) {
        if (c->poisoned) c->comm->abort();
        else cudaDeviceSynchronize();
        delete c->comm;
    }
    free_all(c);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : c->tl_events) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_counts) cudaEventDestroy(c->ev_counts);
    if (c->ev_dw_ready) cudaEventDestroy(c->ev_dw_ready);
    if (c->ev_tl_base) cudaEventDestroy(c->ev_tl_base);
    if (c->s_comp) cudaStreamDestroy(c->s_comp);
    if (c->s_comp2) cudaStreamDestroy(c->s_comp2);
    if (c->s_gate) cudaStreamDestroy(c->s_gate);
    if (c->s_comm) cudaStreamDestroy(c->s_comm);
    delete c;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_set_peer_timeout_ms(lancet_ctx* c, int64_t ms)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->peer || ms <= 0) return fail(c, LANCET_ERR_ARG, "not a peer-transport context, or ms <= 0");
    c->peer->timeout_ns = (unsigned long long)ms * 1000000ull;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_peer_abort(lancet_ctx* c)
{
    if (!c) return fail(nullptr, LANCET_ERR_ARG, "ctx is NULL");
    if (!c->peer) return fail(c, LANCET_ERR_ARG, "not a peer-transport context");
    cudaSetDevice(c->device);
    if (lancet::peer_poison(c, 0xFFFFFFFFu)) return fail(c, LANCET_ERR_CUDA, "peer abort: cudaMemsetAsync of the flags failed");
    c->poisoned = true;
    c->err = "peer transport aborted (lancet_peer_abort)";
    return LANCET_OK;
}

LANCET_API lancet_status lancet_peer_status(lancet_ctx* c)
{
    return check_ready(c);
}

LANCET_API lancet_status lancet_set_flags(lancet_ctx* c, uint32_t flags)
{
    if (!c) return fail(nullptr, LANCET_ERR_ARG, "ctx is NULL");
    // FORCE_EP is fixed at creation (the workspace layout depends on it): keep the creation bit
    // FORCE_EP and PEER_PUSH are fixed at creation (the workspace layout and the peer protocol
    // depend on them): keep the creation bits
    const uint32_t fixed = LANCET_FLAG_FORCE_EP | LANCET_FLAG_PEER_PUSH;
    flags = (flags & ~fixed) | (c->cfg.flags & fixed);
    if ((flags & LANCET_FLAG_RENORMALIZE) != (c->cfg.flags & LANCET_FLAG_RENORMALIZE) && c->world > 1)
        return fail(c, LANCET_ERR_ARG, "RENORMALIZE must be set at creation (checked across ranks)");
    c->cfg.flags = flags;
    return LANCET_OK;
}

namespace lancet { thread_local bool g_pdl = false; }

LANCET_API lancet_status lancet_moe_forward(lancet_ctx* c, const void* x, const float* wg,
                                            const void* w1, const void* w2, int32_t T, int32_t k,
                                            double cf, int32_t n, void* y, int32_t* expert_idx,
                                            int32_t* slot_out, float* combine_w,
                                            lancet_stream_t stream_)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    const bool ident = c->cfg.act == LANCET_ACT_IDENTITY_EXPERT;
    const int E = c->cfg.n_experts, d = c->cfg.d_model;
    if (!x || !wg || !y || (!ident && (!w1 || !w2))) return fail(c, LANCET_ERR_ARG, "null required pointer");
    if (!aligned16(x) || !aligned16(wg) || !aligned16(y) || (!ident && (!aligned16(w1) || !aligned16(w2))))
        return fail(c, LANCET_ERR_ARG, "x, wg, w1, w2 and y must be 16-byte aligned (vector loads, TMA)");
    if (T < 1 || T > c->cfg.max_tokens) return fail(c, LANCET_ERR_ARG, "T must be in [1, max_tokens]");
    if (k < 1 || k > c->cfg.max_k || k > E) return fail(c, LANCET_ERR_ARG, "k must be in [1, min(E, max_k)]");
    if (!(cf > 0.0) || !std::isfinite(cf)) return fail(c, LANCET_ERR_ARG, "capacity_factor must be > 0");
    if (n < 1 || n > std::min<int>(T, c->cfg.max_chunks)) return fail(c, LANCET_ERR_ARG, "n_chunks must be in [1, min(T, max_chunks)]");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    lancet::g_pdl = (c->cfg.flags & LANCET_FLAG_NO_PDL) == 0;
    if (c->dw_pending) return fail(c, LANCET_ERR_STATE, "deferred dW GEMMs of the last backward were never enqueued");
    c->have_fwd = false;
    c->x = x; c->wg = wg; c->w1 = w1; c->w2 = w2;
    c->T = T; c->k = k; c->n = n; c->cf = cf;
    c->C = capacity_of(T, k, E, cf);
    c->launches_fwd = 0;
    int& L = c->launches_fwd;
    if (!c->tl_accumulate) {
        c->ops.clear();
        c->tl_used = 0;
        if (c->cfg.flags & LANCET_FLAG_TIMELINE) CK(cudaEventRecord(c->ev_tl_base, s));
    }

    RouteArgs ra{};
    ra.x = x; ra.wg = wg; ra.T = T; ra.d = d; ra.E = E; ra.k = k; ra.C = c->C; ra.n_chunks = n;
    ra.renorm = (c->cfg.flags & LANCET_FLAG_RENORMALIZE) ? 1 : 0;
    ra.logits = c->logits; ra.idx = c->idx; ra.w = c->w; ra.slot = c->slot; ra.hist = c->hist;
    ra.S = c->S; ra.send_rows = c->send_rows; ra.send_off = c->send_off;
    ra.bpr = (c->cfg.flags & LANCET_FLAG_GATE_BPR) ? 1 : 0;
    ra.random = (c->cfg.flags & LANCET_FLAG_GATE_RANDOM) ? 1 : 0;
    ra.seed = c->gate_seed;
    if (ra.bpr && ra.random) return fail(c, LANCET_ERR_ARG, "LANCET_FLAG_GATE_BPR and LANCET_FLAG_GATE_RANDOM are exclusive");
    ra.score = c->bpr_score; ra.list = c->bpr_list; ra.bpr_adm = c->bpr_adm; ra.hist2 = c->bpr_hist;
    ra.bpr_meta = c->bpr_meta;
    DispatchArgs da{T, k, d, E, c->idx, c->slot, c->w, c->send_off, c->send_rows};

    if (c->ep && c->push) {
        if (!c->peer_ready) return fail(c, LANCET_ERR_STATE, "peer transport: lancet_peer_import not called");
        st = forward_push(c, ra, da, x, y, s, L);
        if (st) return st;
    } else if (!c->ep) {
        // ---- single GPU: no exchange, no host synchronisation --------------------------
        { OpScope op(c, "gate", 0, -1, s); L += launch_routing(ra, c->bf16, s); }
        CHECK_LAUNCH();
        { OpScope op(c, "permute", 0, -1, s); L += launch_permute(da, x, c->xs, c->bf16, s); }
        CHECK_LAUNCH();
        const void* comb = c->xs;
        if (!ident) {
            const int max_rows = round_up(c->C, kRowAlign);
            st = expert_forward(c, c->send_rows, c->send_off, E, max_rows, s, -1, &L);
            if (st) return st;
            comb = c->out;
        }
        { OpScope op(c, "combine", 0, -1, s); L += launch_combine(da, comb, y, 0, T, c->bf16, s); }
        CHECK_LAUNCH();
    } else {
        // ---- expert parallel over world ranks ---------------------------------------------
        const int G = c->world, E_l = c->E_l;
        const bool serial = c->cfg.flags & LANCET_FLAG_SERIAL;
        const bool nocomm_ = c->cfg.flags & LANCET_FLAG_NO_COMM;   // timing only: no data exchange
        cudaStream_t sc = c->s_comp, sm = serial ? c->s_comp : c->s_comm;
        CK(cudaEventRecord(c->ev_fork, s));
        CK(cudaStreamWaitEvent(sc, c->ev_fork, 0));
        CK(cudaStreamWaitEvent(c->s_comm, c->ev_fork, 0));
        size_t ev_i = 0;
        auto next_ev = [&]() { return c->ev_pool[ev_i++]; };
        lancet::PeerLinks* pr = c->peer;
        if (pr) {
            if (!c->peer_ready) return fail(c, LANCET_ERR_STATE, "peer transport: lancet_peer_import not called");
            ++pr->seq;
            // every peer has pulled the previous step's rows from this rank's pull sources (the
            // backward's only if that step had a backward: a forward may follow a forward)
            if (peer_wait_consumed(c, sc, false, c->bwd_seq == pr->seq - 1))
                return fail(c, LANCET_ERR_CUDA, "cuStreamWaitValue32");
        }

        { OpScope op(c, "gate", 0, -1, sc); L += launch_routing(ra, c->bf16, sc); }
        int* d_send = c->counts_dev;                       // [E][n]
        int* d_recv = c->counts_dev + E * n;               // [G][E_l][n]
        launch_k(send_counts_kernel, ceil_div(E * n, 256), 256, 0, sc, c->S, E, n, d_send);
        ++L;
        CHECK_LAUNCH();
        cudaEvent_t ev_route = next_ev();
        CK(cudaEventRecord(ev_route, sc));
        {   // C1: size exchange, once for all chunks (R11)
            CK(cudaStreamWaitEvent(sm, ev_route, 0));
            OpScope op(c, "a2a_counts", 1, -1, sm);
            std::string err;
            if (pr) {       // all-gather of the count matrix [G][E][n] through peer memory
                if (peer_counts(c, d_send, n, sm, err)) return fail(c, LANCET_ERR_CUDA, err);
                CK(cudaMemcpyAsync(pr->h_matrix, pr->my_counts, sizeof(int) * (size_t)G * E * n,
                                   cudaMemcpyDeviceToHost, sm));
            } else {
                std::vector<P2P> sends, recvs;
                const size_t b = sizeof(int) * E_l * n;
                for (int p = 0; p < G; ++p) {
                    sends.push_back({p, d_send + p * E_l * n, b});
                    recvs.push_back({p, d_recv + p * E_l * n, b});
                }
                if (c->comm->exchange(sends, recvs, sm, err)) return fail(c, LANCET_ERR_NCCL, err);
                CK(cudaMemcpyAsync(c->h_counts, c->counts_dev, sizeof(int) * (E * n + G * E_l * n),
                                   cudaMemcpyDeviceToHost, sm));
            }
            CK(cudaEventRecord(c->ev_counts, sm));
        }
        // K3 permute overlaps the size exchange
        {
            { OpScope op(c, "permute", 0, -1, sc); L += launch_permute(da, x, c->xs, c->bf16, sc); }
            CHECK_LAUNCH();
            if (pr)         // the dispatch sources of every chunk are ready
                for (int cc = 0; cc < (serial ? 1 : n); ++cc)
                    if (peer_signal(c, 0, lancet::PK_XS, cc, sc)) return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
        }
        cudaEvent_t ev_perm = next_ev();
        CK(cudaEventRecord(ev_perm, sc));
        CK(cudaEventSynchronize(c->ev_counts));            // the one host synchronisation
        GlobalPlan gp;
        if (pr) {           // this rank's send / recv counts out of the matrix
            gp.build(G, E, E_l, n, pr->h_matrix);
            pr->matrix = gp.M;
            memcpy(c->h_counts, &gp.M[(size_t)c->rank * E * n], sizeof(int) * E * n);
            for (int src = 0; src < G; ++src)
                for (int el = 0; el < E_l; ++el)
                    for (int ch = 0; ch < n; ++ch)
                        c->h_counts[E * n + (src * E_l + el) * n + ch] = gp.M[((size_t)src * E + c->rank * E_l + el) * n + ch];
        }
        Plan pl{E, E_l, G, n};
        pl.build(c->h_counts, c->h_counts + E * n);
        st = ensure_expert_rows(c, std::max(pl.rows_total, kRowAlign));
        if (st) return st;
        c->host_send = pl.send;
        c->host_recv = pl.recv;
        c->host_grp_rows = pl.grp_rows;
        c->host_grp_off = pl.grp_off;
        c->n_groups = n * E_l;
        int* d_grp_rows = c->grp_dev;
        int* d_grp_off = c->grp_dev + n * E_l;
        memcpy(c->h_grp, pl.grp_rows.data(), sizeof(int) * n * E_l);
        memcpy(c->h_grp + n * E_l, pl.grp_off.data(), sizeof(int) * n * E_l);
        CK(cudaMemcpyAsync(c->grp_dev, c->h_grp, sizeof(int) * 2 * n * E_l, cudaMemcpyHostToDevice, sc));
        L += launch_zero_pads(c->xe, d, d_grp_off, d_grp_rows, n * E_l, (int)c->elt, sc);
        CHECK_LAUNCH();
        const size_t rowb = (size_t)d * c->elt;
        char* xs = (char*)c->xs;
        char* xe = (char*)c->xe;
        char* comb = (char*)c->comb;
        const int nc = serial ? 1 : n;                     // serial baseline: chunks merged
        auto chunk_range = [&](int cc, int& c0, int& c1) {
            if (serial) { c0 = 0; c1 = n; } else { c0 = cc; c1 = cc + 1; }
        };
        // S1: dispatch all-to-alls D0..D(n-1) on the comm lane (stage order)
        std::vector<cudaEvent_t> ev_disp(nc), ev_exp(nc), ev_comb(nc);
        CK(cudaStreamWaitEvent(sm, ev_perm, 0));
        cudaEvent_t ev_pads = next_ev();
        CK(cudaEventRecord(ev_pads, sc));
        CK(cudaStreamWaitEvent(sm, ev_pads, 0));
        for (int cc = 0; cc < nc; ++cc) {
            int c0, c1;
            chunk_range(cc, c0, c1);
            OpScope op(c, "a2a_dispatch", 1, serial ? -1 : cc, sm);
            if (pr) {
                std::string err;
                if (peer_pull(c, lancet::PK_XS, cc, (nocomm_ ? std::vector<lancet::PeerCopy>{} : gp.pulls(c->rank, true, c0, c1, xe, rowb)), cc == nc - 1, sm, err))
                    return fail(c, LANCET_ERR_CUDA, err);
                if (ident && peer_signal(c, 0, lancet::PK_OUT, cc, sm))   // identity: xe is the combine source
                    return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
                ev_disp[cc] = next_ev();
                CK(cudaEventRecord(ev_disp[cc], sm));
                continue;
            }
            std::vector<P2P> sends, recvs;
            for (int p = 0; p < G; ++p)
                for (int i = 0; i < E_l; ++i) {
                    const int e = p * E_l + i;
                    for (int ch = c0; ch < c1; ++ch)
                        sends.push_back({p, xs + (size_t)(pl.send_off[e] + pl.S[e * (n + 1) + ch]) * rowb,
                                         (size_t)pl.send[e * n + ch] * rowb});
                }
            for (int p = 0; p < G; ++p)
                for (int el = 0; el < E_l; ++el)
                    for (int ch = c0; ch < c1; ++ch)
                        recvs.push_back({p, xe + (size_t)(pl.grp_off[ch * E_l + el] + pl.src_off[(p * E_l + el) * n + ch]) * rowb,
                                         (size_t)pl.recv[(p * E_l + el) * n + ch] * rowb});
            std::string err;
            if (!nocomm_ && c->comm->exchange(sends, recvs, sm, err)) return fail(c, LANCET_ERR_NCCL, err);
            ev_disp[cc] = next_ev();
            CK(cudaEventRecord(ev_disp[cc], sm));
        }
        // experts per chunk on the compute lane
        for (int cc = 0; cc < nc; ++cc) {
            int c0, c1;
            chunk_range(cc, c0, c1);
            CK(cudaStreamWaitEvent(sc, ev_disp[cc], 0));
            if (!ident) {
                int mr = 0;
                for (int ch = c0; ch < c1; ++ch)
                    for (int el = 0; el < E_l; ++el) mr = std::max(mr, round_up(pl.grp_rows[ch * E_l + el], kRowAlign));
                st = expert_forward(c, d_grp_rows + c0 * E_l, d_grp_off + c0 * E_l, (c1 - c0) * E_l,
                                    std::max(mr, kRowAlign), sc, serial ? -1 : cc, &L);
                if (st) return st;
                if (pr && peer_signal(c, 0, lancet::PK_OUT, cc, sc)) return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
            }
            ev_exp[cc] = next_ev();
            CK(cudaEventRecord(ev_exp[cc], sc));
        }
        // combine all-to-alls C0..C(n-1)
        const char* eout = ident ? xe : (const char*)c->out;
        for (int cc = 0; cc < nc; ++cc) {
            int c0, c1;
            chunk_range(cc, c0, c1);
            CK(cudaStreamWaitEvent(sm, ev_exp[cc], 0));
            OpScope op(c, "a2a_combine", 1, serial ? -1 : cc, sm);
            if (pr) {
                std::string err;
                if (peer_pull(c, lancet::PK_OUT, cc, (nocomm_ ? std::vector<lancet::PeerCopy>{} : gp.pulls(c->rank, false, c0, c1, comb, rowb)), cc == nc - 1, sm, err))
                    return fail(c, LANCET_ERR_CUDA, err);
                ev_comb[cc] = next_ev();
                CK(cudaEventRecord(ev_comb[cc], sm));
                continue;
            }
            std::vector<P2P> sends, recvs;
            for (int p = 0; p < G; ++p)
                for (int el = 0; el < E_l; ++el)
                    for (int ch = c0; ch < c1; ++ch)
                        sends.push_back({p, (void*)(eout + (size_t)(pl.grp_off[ch * E_l + el] + pl.src_off[(p * E_l + el) * n + ch]) * rowb),
                                         (size_t)pl.recv[(p * E_l + el) * n + ch] * rowb});
            for (int p = 0; p < G; ++p)
                for (int i = 0; i < E_l; ++i) {
                    const int e = p * E_l + i;
                    for (int ch = c0; ch < c1; ++ch)
                        recvs.push_back({p, comb + (size_t)(pl.send_off[e] + pl.S[e * (n + 1) + ch]) * rowb,
                                         (size_t)pl.send[e * n + ch] * rowb});
                }
            std::string err;
            if (!nocomm_ && c->comm->exchange(sends, recvs, sm, err)) return fail(c, LANCET_ERR_NCCL, err);
            ev_comb[cc] = next_ev();
            CK(cudaEventRecord(ev_comb[cc], sm));
        }
        // gather per chunk (chunk c's tokens are final as soon as combine c lands)
        for (int cc = 0; cc < nc; ++cc) {
            CK(cudaStreamWaitEvent(sc, ev_comb[cc], 0));
            const int t0 = serial ? 0 : chunk_start(T, n, cc), t1 = serial ? T : chunk_start(T, n, cc + 1);
            OpScope op(c, "combine", 0, serial ? -1 : cc, sc);
            L += launch_combine(da, comb, y, t0, t1, c->bf16, sc);
        }
        CHECK_LAUNCH();
        CK(cudaEventRecord(c->ev_join, sc));
        CK(cudaStreamWaitEvent(s, c->ev_join, 0));
        if (sm != sc) {
            cudaEvent_t e2 = next_ev();
            CK(cudaEventRecord(e2, sm));
            CK(cudaStreamWaitEvent(s, e2, 0));
        }
    }
    const size_t tk = (size_t)T * k;
    if (expert_idx) CK(cudaMemcpyAsync(expert_idx, c->idx, tk * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (slot_out) CK(cudaMemcpyAsync(slot_out, c->slot, tk * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (combine_w) CK(cudaMemcpyAsync(combine_w, c->w, tk * sizeof(float), cudaMemcpyDeviceToDevice, s));
    c->have_fwd = true;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_moe_forward_partitioned(lancet_ctx* c, const void* x, const float* wg,
                                                        const void* w1, const void* w2, int32_t T, int32_t k,
                                                        double cf, int32_t n, const void* resid, void* y,
                                                        int32_t* expert_idx, int32_t* slot_out, float* combine_w,
                                                        lancet_stream_t stream_)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!x || !wg || !w1 || !w2 || !y) return fail(c, LANCET_ERR_ARG, "null required pointer");
    if (!aligned16(x) || !aligned16(wg) || !aligned16(y) || !aligned16(w1) || !aligned16(w2) || (resid && !aligned16(resid)))
        return fail(c, LANCET_ERR_ARG, "x, wg, w1, w2, resid and y must be 16-byte aligned (vector loads, TMA)");
    if (n < 1 || n > std::min<int>(T, c->cfg.max_chunks)) return fail(c, LANCET_ERR_ARG, "n_chunks must be in [1, min(T, max_chunks)]");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    std::vector<int> bounds(n + 1);
    for (int ch = 0; ch <= n; ++ch) bounds[ch] = chunk_start(T, n, ch);
    lancet::ChunkedInput in;
    in.n = n;
    in.bounds = bounds.data();
    in.resid = resid;
    in.s_pre = c->s_gate;      // the input is resident: the producer stream only gates
    in.cf_max = cf;
    in.produce = [](int, int, int, cudaStream_t) { return LANCET_OK; };
    st = lancet::moe_forward_chunked(c, x, wg, w1, w2, T, k, cf, y, in, s);
    if (st) return st;
    const size_t tk = (size_t)T * k;
    if (expert_idx) CK(cudaMemcpyAsync(expert_idx, c->idx, tk * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (slot_out) CK(cudaMemcpyAsync(slot_out, c->slot, tk * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (combine_w) CK(cudaMemcpyAsync(combine_w, c->w, tk * sizeof(float), cudaMemcpyDeviceToDevice, s));
    return LANCET_OK;
}

namespace lancet {
lancet_status moe_backward_into(lancet_ctx* c, const void* dy, void* dx, float* dwg, float* dw1, float* dw2,
                                cudaStream_t s)
{
    return lancet_moe_backward(c, dy, dx, dwg, dw1, dw2, reinterpret_cast<lancet_stream_t>(s));
}
}  // namespace lancet

LANCET_API lancet_status lancet_moe_backward(lancet_ctx* c, const void* dy, void* dx, float* dwg,
                                             float* dw1, float* dw2, lancet_stream_t stream_)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->have_fwd) return fail(c, LANCET_ERR_STATE, "backward without a preceding forward");
    const bool ident = c->cfg.act == LANCET_ACT_IDENTITY_EXPERT;
    if (!dy || !dx || !dwg || (!ident && (!dw1 || !dw2))) return fail(c, LANCET_ERR_ARG, "null required pointer");
    if (!aligned16(dy) || !aligned16(dx) || !aligned16(dwg) || (!ident && (!aligned16(dw1) || !aligned16(dw2))))
        return fail(c, LANCET_ERR_ARG, "dy, dx, dwg, dw1 and dw2 must be 16-byte aligned (vector loads, TMA)");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    lancet::g_pdl = (c->cfg.flags & LANCET_FLAG_NO_PDL) == 0;
    const int E = c->cfg.n_experts, d = c->cfg.d_model, T = c->T, k = c->k, n = c->n;
    const int renorm = (c->cfg.flags & LANCET_FLAG_GATE_RANDOM) ? 2 : (c->cfg.flags & LANCET_FLAG_RENORMALIZE) ? 1 : 0;
    c->launches_bwd = 0;
    int& L = c->launches_bwd;
    DispatchArgs da{T, k, d, E, c->idx, c->slot, c->w, c->send_off, c->send_rows};
    const bool defer = (c->cfg.flags & LANCET_FLAG_DEFER_DW) && !ident;
    if (c->dw_pending) return fail(c, LANCET_ERR_STATE, "the previous backward's deferred dW GEMMs were never enqueued");
    // the fillers set for this backward, each served once right after its all-to-all's launch
    std::vector<bool> served(c->fillers.size(), false);
    struct ClearFillers { lancet_ctx* c; ~ClearFillers() { c->fillers.clear(); } } clear_fillers{c};
    auto run_fillers = [&](lancet_ctx*, int lo, int hi, cudaStream_t fs, int* launches) -> lancet_status {
        for (size_t i = 0; i < c->fillers.size(); ++i) {
            const auto& fl = c->fillers[i];
            if (served[i] || fl.a2a < lo || fl.a2a >= hi) continue;
            served[i] = true;
            lancet_status fst = enqueue_pending_dw(fl.other, fl.which, fs, launches);
            if (fst) {
                c->fillers.clear();
                return fail(c, fst, std::string("dW filler: ") + fl.other->err);
            }
        }
        return LANCET_OK;
    };

    if (!c->ep) {
        const void* comb = ident ? c->xs : c->out;
        { OpScope op(c, "combine_bwd", 0, -1, s);
          L += launch_combine_bwd(da, dy, comb, c->g, c->dcomb, 0, T, true, c->logits, renorm, c->dlogit,
                                  c->prow, c->bf16, s); }
        CHECK_LAUNCH();
        const void* dxe = c->dcomb;
        const int max_rows = round_up(c->C, kRowAlign);
        // K6 (dx) and K7 (dWg).  Default: on a side stream beside the persistent GEMMs, K7 right
        // after K5 (under the dX GEMMs) and K6 after the dX GEMMs (under the dW GEMMs) -- measured
        // fastest.  With LANCET_FLAG_NO_SIDE_STREAM they run in line on the
        // caller's stream, fused into one pass over the tokens after the dX GEMMs where the shape
        // allows (LANCET_FLAG_UNFUSED_GATE_BWD keeps two kernels).
        const bool inline_gate = (c->cfg.flags & LANCET_FLAG_NO_SIDE_STREAM) != 0;
        cudaStream_t sa = inline_gate ? s : c->s_comm;
        cudaEvent_t ev_k5 = c->ev_pool[0], ev_dx = c->ev_pool[1], ev_side = c->ev_pool[2];
        const bool fused = inline_gate && !ident && gate_bwd_fused_ok(d, E, k) &&
                           !(c->cfg.flags & LANCET_FLAG_UNFUSED_GATE_BWD);
        if (!fused) {
            CK(cudaEventRecord(ev_k5, s));
            CK(cudaStreamWaitEvent(sa, ev_k5, 0));
            st = gate_backward_dwg(c, dwg, sa, &L);
            if (st) return st;
        }
        if (!ident) {
            st = expert_backward_dx(c, c->dcomb, c->send_rows, c->send_off, E, max_rows, s, -1, &L);
            if (st) return st;
            dxe = c->dXe;
        }
        CK(cudaEventRecord(ev_dx, s));
        CK(cudaStreamWaitEvent(sa, ev_dx, 0));
        if (fused) {
            OpScope op(c, "gate_bwd_fused", sa == c->s_comp || sa == s ? 0 : 2, -1, sa);
            L += launch_gate_bwd_fused(da, dxe, c->prow, c->dlogit, c->wg, c->x, dx, c->dwg_partial, dwg,
                                       c->num_sms, c->bf16, sa);
            CHECK_LAUNCH();
        } else {
            st = gate_backward_dx(c, da, dxe, dx, sa, 0, 1, &L);
            if (st) return st;
        }
        CK(cudaEventRecord(ev_side, sa));
        if (!ident) {
            if (defer) {
                CK(cudaEventRecord(c->ev_dw_ready, s));
                c->dw_pending = 3; c->pend_dw1 = dw1; c->pend_dw2 = dw2;
            } else {
                st = expert_backward_dw(c, c->dcomb, c->send_rows, c->send_off, E, dw1, dw2, 0, s, -1, &L);
                if (st) return st;
            }
        }
        st = run_fillers(c, 0, 1 << 30, s, &L);       // no all-to-all at world 1
        if (st) return st;
        CK(cudaStreamWaitEvent(s, ev_side, 0));
        return LANCET_OK;
    }

    // ---- expert parallel (S2) ---------------------------------------------------------------
    if (c->push) return backward_push(c, da, dy, dx, dwg, dw1, dw2, renorm, s, L);
    const int G = c->world, E_l = c->E_l;
    const bool serial = c->cfg.flags & LANCET_FLAG_SERIAL;
    const bool nocomm_ = c->cfg.flags & LANCET_FLAG_NO_COMM;   // timing only: no data exchange
    const bool late_dw = serial || (c->cfg.flags & LANCET_FLAG_NO_DW_OVERLAP);
    cudaStream_t sc = c->s_comp, sm = serial ? c->s_comp : c->s_comm;
    CK(cudaEventRecord(c->ev_fork, s));
    CK(cudaStreamWaitEvent(sc, c->ev_fork, 0));
    CK(cudaStreamWaitEvent(c->s_comm, c->ev_fork, 0));
    size_t ev_i = 0;
    auto next_ev = [&]() { return c->ev_pool[ev_i++]; };
    Plan pl{E, E_l, G, n};
    pl.build(c->host_send.data(), c->host_recv.data());
    lancet::PeerLinks* pr = c->peer;
    GlobalPlan gp;
    if (pr) gp.build(G, E, E_l, n, pr->matrix.data());
    int* d_grp_rows = c->grp_dev;
    int* d_grp_off = c->grp_dev + n * E_l;
    const size_t rowb = (size_t)d * c->elt;
    const int nc = serial ? 1 : n;
    auto chunk_range = [&](int cc, int& c0, int& c1) {
        if (serial) { c0 = 0; c1 = n; } else { c0 = cc; c1 = cc + 1; }
    };
    auto tok_range = [&](int cc, int& t0, int& t1) {
        t0 = serial ? 0 : chunk_start(T, n, cc);
        t1 = serial ? T : chunk_start(T, n, cc + 1);
    };
    // pads of the received dO rows must be zero (K-grouped dW reads whole 128-row blocks)
    L += launch_zero_pads(c->dout, d, d_grp_off, d_grp_rows, n * E_l, (int)c->elt, sc);
    const void* comb = c->comb;     // o_tj returned by the combine all-to-all (source side)
    std::vector<cudaEvent_t> ev_k5(nc), ev_b1(nc), ev_dx(nc), ev_b2(nc);
    for (int cc = 0; cc < nc; ++cc) {
        int t0, t1;
        tok_range(cc, t0, t1);
        OpScope op(c, "combine_bwd", 0, serial ? -1 : cc, sc);
        L += launch_combine_bwd(da, dy, comb, c->g, c->dcomb, t0, t1, cc == 0, c->logits, renorm, c->dlogit,
                                c->prow, c->bf16, sc);
        if (pr && peer_signal(c, 0, lancet::PK_DCOMB, cc, sc)) return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
        ev_k5[cc] = next_ev();
        CK(cudaEventRecord(ev_k5[cc], sc));
    }
    CHECK_LAUNCH();
    char* dcomb = (char*)c->dcomb;
    char* dout = (char*)c->dout;
    // backward a2a #1: dO rows to the experts (same plan as the dispatch)
    for (int cc = 0; cc < nc; ++cc) {
        int c0, c1;
        chunk_range(cc, c0, c1);
        CK(cudaStreamWaitEvent(sm, ev_k5[cc], 0));
        OpScope op(c, "a2a_bwd_dispatch", 1, serial ? -1 : cc, sm);
        if (pr) {
            std::string err;
            if (peer_pull(c, lancet::PK_DCOMB, cc, (nocomm_ ? std::vector<lancet::PeerCopy>{} : gp.pulls(c->rank, true, c0, c1, dout, rowb)), cc == nc - 1, sm, err))
                return fail(c, LANCET_ERR_CUDA, err);
            if (ident && peer_signal(c, 0, lancet::PK_DXE, cc, sm))   // identity: dout is the source back
                return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
            ev_b1[cc] = next_ev();
            CK(cudaEventRecord(ev_b1[cc], sm));
            continue;
        }
        std::vector<P2P> sends, recvs;
        for (int p = 0; p < G; ++p)
            for (int i = 0; i < E_l; ++i) {
                const int e = p * E_l + i;
                for (int ch = c0; ch < c1; ++ch)
                    sends.push_back({p, dcomb + (size_t)(pl.send_off[e] + pl.S[e * (n + 1) + ch]) * rowb,
                                     (size_t)pl.send[e * n + ch] * rowb});
            }
        for (int p = 0; p < G; ++p)
            for (int el = 0; el < E_l; ++el)
                for (int ch = c0; ch < c1; ++ch)
                    recvs.push_back({p, dout + (size_t)(pl.grp_off[ch * E_l + el] + pl.src_off[(p * E_l + el) * n + ch]) * rowb,
                                     (size_t)pl.recv[(p * E_l + el) * n + ch] * rowb});
        std::string err;
        if (!nocomm_ && c->comm->exchange(sends, recvs, sm, err)) return fail(c, LANCET_ERR_NCCL, err);
        ev_b1[cc] = next_ev();
        CK(cudaEventRecord(ev_b1[cc], sm));
    }
    // dW GEMMs of other layers placed under this layer's dO all-to-all (R17): on the compute
    // stream ahead of the dX GEMMs, which wait for that all-to-all anyway
    st = run_fillers(c, 0, n, sc, &L);
    if (st) return st;
    // dX GEMMs per chunk, each followed immediately by the chunk's dW GEMMs
    for (int cc = 0; cc < nc; ++cc) {
        int c0, c1;
        chunk_range(cc, c0, c1);
        CK(cudaStreamWaitEvent(sc, ev_b1[cc], 0));
        if (!ident) {
            int mr = 0;
            for (int ch = c0; ch < c1; ++ch)
                for (int el = 0; el < E_l; ++el) mr = std::max(mr, round_up(pl.grp_rows[ch * E_l + el], kRowAlign));
            st = expert_backward_dx(c, c->dout, d_grp_rows + c0 * E_l, d_grp_off + c0 * E_l,
                                    (c1 - c0) * E_l, std::max(mr, kRowAlign), sc, serial ? -1 : cc, &L);
            if (st) return st;
            if (pr && peer_signal(c, 0, lancet::PK_DXE, cc, sc)) return fail(c, LANCET_ERR_CUDA, "cuStreamWriteValue32");
        }
        ev_dx[cc] = next_ev();
        CK(cudaEventRecord(ev_dx[cc], sc));
        if (!ident && !late_dw && !defer) {
            for (int ch = c0; ch < c1; ++ch) {
                st = expert_backward_dw(c, c->dout, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l,
                                        dw1, dw2, ch > 0, sc, ch, &L);
                if (st) return st;
            }
        }
    }
    if (defer) {                // this layer's dW GEMMs stay pending (R17)
        CK(cudaEventRecord(c->ev_dw_ready, sc));
        c->dw_pending = 3; c->pend_dw1 = dw1; c->pend_dw2 = dw2;
    }
    // backward a2a #2: dX rows back to the token owners (same plan as the combine)
    const char* dxe = ident ? (const char*)c->dout : (const char*)c->dXe;
    char* dxcomb = (char*)c->dxcomb;
    for (int cc = 0; cc < nc; ++cc) {
        int c0, c1;
        chunk_range(cc, c0, c1);
        CK(cudaStreamWaitEvent(sm, ev_dx[cc], 0));
        OpScope op(c, "a2a_bwd_combine", 1, serial ? -1 : cc, sm);
        if (pr) {
            std::string err;
            if (peer_pull(c, lancet::PK_DXE, cc, (nocomm_ ? std::vector<lancet::PeerCopy>{} : gp.pulls(c->rank, false, c0, c1, dxcomb, rowb)), cc == nc - 1, sm, err))
                return fail(c, LANCET_ERR_CUDA, err);
            ev_b2[cc] = next_ev();
            CK(cudaEventRecord(ev_b2[cc], sm));
            st = run_fillers(c, serial ? n : n + cc, serial ? 2 * n : n + cc + 1, sc, &L);
            if (st) return st;
            continue;
        }
        std::vector<P2P> sends, recvs;
        for (int p = 0; p < G; ++p)
            for (int el = 0; el < E_l; ++el)
                for (int ch = c0; ch < c1; ++ch)
                    sends.push_back({p, (void*)(dxe + (size_t)(pl.grp_off[ch * E_l + el] + pl.src_off[(p * E_l + el) * n + ch]) * rowb),
                                     (size_t)pl.recv[(p * E_l + el) * n + ch] * rowb});
        for (int p = 0; p < G; ++p)
            for (int i = 0; i < E_l; ++i) {
                const int e = p * E_l + i;
                for (int ch = c0; ch < c1; ++ch)
                    recvs.push_back({p, dxcomb + (size_t)(pl.send_off[e] + pl.S[e * (n + 1) + ch]) * rowb,
                                     (size_t)pl.send[e * n + ch] * rowb});
            }
        std::string err;
        if (!nocomm_ && c->comm->exchange(sends, recvs, sm, err)) return fail(c, LANCET_ERR_NCCL, err);
        ev_b2[cc] = next_ev();
        CK(cudaEventRecord(ev_b2[cc], sm));
        st = run_fillers(c, serial ? n : n + cc, serial ? 2 * n : n + cc + 1, sc, &L);
        if (st) return st;
    }
    st = run_fillers(c, 0, 1 << 30, sc, &L);     // indices this backward never reached
    if (st) return st;
    if (!ident && late_dw && !defer) {    // ablation / serial baseline: all dW after the last a2a
        for (int ch = 0; ch < n; ++ch) {
            st = expert_backward_dw(c, c->dout, d_grp_rows + ch * E_l, d_grp_off + ch * E_l, E_l,
                                    dw1, dw2, ch > 0, sc, ch, &L);
            if (st) return st;
        }
    }
    for (int cc = 0; cc < nc; ++cc) {
        CK(cudaStreamWaitEvent(sc, ev_b2[cc], 0));
        st = gate_backward_dx(c, da, dxcomb, dx, sc, cc, nc, &L);
        if (st) return st;
    }
    st = gate_backward_dwg(c, dwg, sc, &L);
    if (st) return st;
    if (pr) c->bwd_seq = pr->seq;
    CK(cudaEventRecord(c->ev_join, sc));
    CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    if (sm != sc) {
        cudaEvent_t e2 = next_ev();
        CK(cudaEventRecord(e2, sm));
        CK(cudaStreamWaitEvent(s, e2, 0));
    }
    return LANCET_OK;
}

LANCET_API lancet_status lancet_set_gate_seed(lancet_ctx* c, uint64_t seed)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    c->gate_seed = seed;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_moe_backward_dw(lancet_ctx* c, int32_t which, lancet_stream_t stream)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    lancet::g_pdl = (c->cfg.flags & LANCET_FLAG_NO_PDL) == 0;
    int L = 0;
    st = enqueue_pending_dw(c, which, reinterpret_cast<cudaStream_t>(stream), &L);
    if (st) return st;
    CK(cudaGetLastError());
    return LANCET_OK;
}

LANCET_API lancet_status lancet_set_dw_fillers(lancet_ctx* c, int32_t n, lancet_ctx* const* others,
                                               const int32_t* which, const int32_t* a2a_index)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (n < 0 || (n > 0 && (!others || !which || !a2a_index))) return fail(c, LANCET_ERR_ARG, "bad filler arrays");
    std::vector<lancet_ctx::Filler> f;
    for (int i = 0; i < n; ++i) {
        if (!others[i] || which[i] < 1 || which[i] > 3 || a2a_index[i] < 0)
            return fail(c, LANCET_ERR_ARG, "filler " + std::to_string(i) + ": null context, which not in 1..3 or negative index");
        f.push_back({others[i], which[i], a2a_index[i]});
    }
    c->fillers = f;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_get_counts(lancet_ctx* c, int32_t* send_counts,
                                           int32_t* recv_counts, int32_t* capacity)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->have_fwd) return fail(c, LANCET_ERR_STATE, "no forward yet");
    const int E = c->cfg.n_experts, n = c->n, G = c->world, E_l = c->E_l;
    CK(cudaDeviceSynchronize());
    std::vector<int> S(E * (n + 1));
    CK(cudaMemcpy(S.data(), c->S, sizeof(int) * S.size(), cudaMemcpyDeviceToHost));
    std::vector<int> send(E * n);
    for (int e = 0; e < E; ++e)
        for (int ch = 0; ch < n; ++ch) send[e * n + ch] = S[e * (n + 1) + ch + 1] - S[e * (n + 1) + ch];
    if (send_counts) memcpy(send_counts, send.data(), sizeof(int) * E * n);
    if (recv_counts) {
        if (c->push) {          // the plan lives on the device: recv from the gathered matrix
            std::vector<int> M((size_t)G * E * n);
            CK(cudaMemcpy(M.data(), c->peer->my_counts, sizeof(int) * M.size(), cudaMemcpyDeviceToHost));
            for (int src = 0; src < G; ++src)
                for (int el = 0; el < E_l; ++el)
                    for (int ch = 0; ch < n; ++ch)
                        recv_counts[(src * E_l + el) * n + ch] = M[((size_t)src * E + c->rank * E_l + el) * n + ch];
        } else if (G == 1 && !c->ep) {
            memcpy(recv_counts, send.data(), sizeof(int) * E * n);
        } else {
            memcpy(recv_counts, c->host_recv.data(), sizeof(int) * G * E_l * n);
        }
    }
    if (capacity) *capacity = c->C;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_timeline_begin(lancet_ctx* c, lancet_stream_t stream)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    CK(cudaDeviceSynchronize());
    c->ops.clear();
    c->tl_used = 0;
    c->tl_accumulate = true;
    CK(cudaEventRecord(c->ev_tl_base, reinterpret_cast<cudaStream_t>(stream)));
    return LANCET_OK;
}

LANCET_API lancet_status lancet_last_timeline(lancet_ctx* c, lancet_op_record* out, int32_t cap,
                                              int32_t* n_out)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    CK(cudaDeviceSynchronize());
    int m = 0;
    for (const OpEvent& op : c->ops) {
        if (m >= cap) break;
        lancet_op_record& r = out[m++];
        memset(&r, 0, sizeof(r));
        strncpy(r.name, op.name.c_str(), sizeof(r.name) - 1);
        r.lane = op.lane;
        r.chunk = op.chunk;
        CK(cudaEventElapsedTime(&r.start_us, c->ev_tl_base, op.beg));
        CK(cudaEventElapsedTime(&r.end_us, c->ev_tl_base, op.end));
        r.start_us *= 1000.f;
        r.end_us *= 1000.f;
    }
    if (n_out) *n_out = m;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_debug_copy(lancet_ctx* c, int32_t which, void* host_dst, size_t bytes)
{
    lancet_status st = check_ready(c);
    if (st) return st;
    if (!c->have_fwd) return fail(c, LANCET_ERR_STATE, "no forward yet");
    const void* src = nullptr;
    size_t need = 0;
    const size_t rowb = (size_t)c->cfg.d_model * c->elt;
    switch (which) {
    case 0: src = c->logits; need = sizeof(float) * (size_t)c->T * c->cfg.n_experts; break;
    case 1: src = c->out; need = (size_t)c->rows_exp * rowb; break;
    case 2: src = c->H; need = (size_t)c->rows_exp * c->cfg.d_ffn * c->elt; break;
    case 3: src = c->xe; need = (size_t)c->rows_exp * rowb; break;
    case 4: src = c->grp_dev; need = sizeof(int) * 2 * (size_t)c->n * c->E_l; break;
    case 5: if (c->peer) { src = c->peer->my_flags; need = sizeof(uint32_t) * lancet::peer_flag_words(c->world, c->peer->n_max); } break;
    case 6: if (c->peer) { src = c->peer->d_push_base; need = sizeof(int) * (size_t)c->n * c->cfg.n_experts; } break;
    default: break;
    }
    if (!src) return fail(c, LANCET_ERR_ARG, "unknown buffer");
    if (!host_dst || bytes < need) return fail(c, LANCET_ERR_ARG, "destination too small");
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(host_dst, src, need, cudaMemcpyDeviceToHost));
    return LANCET_OK;
}

LANCET_API lancet_status lancet_plan_exchange(int32_t G, int32_t E_l, int32_t n,
                                              const int32_t* send_counts, const int32_t* recv_counts,
                                              int32_t* send_off, int32_t* S, int32_t* grp_rows,
                                              int32_t* grp_off, int32_t* src_off, int32_t* total_rows)
{
    if (G < 1 || E_l < 1 || n < 1 || n > kMaxChunks || !send_counts || !recv_counts || !send_off || !S ||
        !grp_rows || !grp_off || !src_off || !total_rows)
        return fail(nullptr, LANCET_ERR_ARG, "bad arguments");
    for (int i = 0; i < G * E_l * n; ++i)
        if (send_counts[i] < 0 || recv_counts[i] < 0) return fail(nullptr, LANCET_ERR_ARG, "negative count");
    plan_send(G * E_l, n, send_counts, S, send_off);
    *total_rows = plan_recv(G, E_l, n, recv_counts, grp_rows, grp_off, src_off);
    return LANCET_OK;
}

LANCET_API lancet_status lancet_workspace_bytes(const lancet_ctx* c, size_t* bytes)
{
    if (!c || !bytes) return fail(nullptr, LANCET_ERR_ARG, "null argument");
    size_t b = 0;
    for (const DevBuf& x : c->allocs) b += x.bytes;
    *bytes = b;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_nccl_registered(const lancet_ctx* c, int32_t* count)
{
    if (!c || !count) return fail(nullptr, LANCET_ERR_ARG, "null argument");
    *count = c->comm ? c->nccl_registered : 0;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_launch_counts(const lancet_ctx* c, int32_t* fwd, int32_t* bwd)
{
    if (!c) return fail(nullptr, LANCET_ERR_ARG, "ctx is NULL");
    if (fwd) *fwd = c->launches_fwd;
    if (bwd) *bwd = c->launches_bwd;
    return LANCET_OK;
}
