// block.cu -- C-ABI of the GPT-MoE block (include/lancet_block.h): the non-MoE part of the
// block (LN1, fused q|k|v projection, causal attention, output projection, residual + LN2) and
// Lancet's pre-MoE partition of it into the MoE layer's all-to-all pipeline.
//
// "if we partition non-MoE computations and integrate them into the computation-communication
// pipeline, we can create additional opportunities to overlap operations with the all-to-all
// communication" (fig:part_all).  Per chunk of whole sequences (the batch
// dimension, L252; R20) the block's stream runs LN1 -> QKV GEMM -> attention -> O GEMM ->
// residual + LN2 and hands the chunk's rows to the MoE layer, which gates them with the carried
// capacity state (L255) and exchanges / computes / combines them on its own streams
// (lancet::moe_forward_chunked) while the block's stream already works on the next chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/lancet_block.h"
#include "common.cuh"
#include "context.h"
#include "internal.h"
#include "kernels.h"

#define LANCET_API extern "C" __attribute__((visibility("default")))

struct lancet_block {
    lancet_ctx* moe = nullptr;
    int world = 1, rank = 0, device = 0, d = 0, H = 0, S = 0, max_tokens = 0;
    double cf_max = 0.0;
    cudaStream_t s_pre = nullptr;
    std::vector<void*> allocs;
    void *a1 = nullptr, *qkv = nullptr, *att = nullptr, *o = nullptr, *h = nullptr, *u = nullptr;
    float *mu1 = nullptr, *rs1 = nullptr, *mu2 = nullptr, *rs2 = nullptr, *lse = nullptr;
    int* tok_tab = nullptr;     // [2][kMaxChunks]: rows | first row of each chunk (projection GEMMs),
                                // then [2]: rows | first row of the whole batch (weight gradients)
    int T_last = 0;
    // backward workspace and the last forward's arguments (pointers only; the caller keeps them)
    void *du = nullptr, *dh = nullptr, *datt = nullptr, *dqkv = nullptr, *da1 = nullptr;
    float *Dbuf = nullptr, *ln_partial = nullptr;
    const void *x = nullptr, *w_qkv = nullptr, *w_o = nullptr;
    const float *ln1_g = nullptr, *ln2_g = nullptr;
    int n_last = 0;
    bool have_fwd = false;
    std::vector<cudaEvent_t> ev_out;   // [kMaxChunks]: chunk c of the last forward's out is stored
};

namespace {

using namespace lancet;

thread_local std::string g_block_err;

lancet_status bfail(lancet_block* b, lancet_status st, const std::string& msg)
{
    g_block_err = msg;
    return record_error(b ? b->moe : nullptr, st, msg);     // lancet_last_error(ctx or NULL)
}

#define BCK(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) return bfail(b, LANCET_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

__global__ void tok_tab_kernel(int* tab, int n, int Tc)
{
    pdl_wait();
    const int c = threadIdx.x;
    if (c < n) {
        tab[c] = Tc;
        tab[kMaxChunks + c] = c * Tc;
    }
    if (c == 0) {
        tab[2 * kMaxChunks] = n * Tc;
        tab[2 * kMaxChunks + 1] = 0;
    }
}

bool aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

LANCET_API lancet_status lancet_block_create_peer(lancet_block** out, int32_t world, int32_t rank, int32_t dev,
                                                  const lancet_block_config* cfg)
{
    if (!out || !cfg) return bfail(nullptr, LANCET_ERR_ARG, "out / cfg is NULL");
    *out = nullptr;
    const lancet_layer_config& m = cfg->moe;
    if (m.dtype != LANCET_BF16) return bfail(nullptr, LANCET_ERR_UNSUPPORTED, "the block runs in bf16");
    if (m.act == LANCET_ACT_IDENTITY_EXPERT) return bfail(nullptr, LANCET_ERR_UNSUPPORTED, "the block needs FFN experts");
    if (cfg->n_heads <= 0 || m.d_model != cfg->n_heads * 128)
        return bfail(nullptr, LANCET_ERR_UNSUPPORTED, "attention: d_model must be n_heads * 128 (head_dim 128)");
    if (m.d_model > 4096) return bfail(nullptr, LANCET_ERR_UNSUPPORTED, "LayerNorm: d_model <= 4096");
    if (cfg->seq_len <= 0 || cfg->seq_len % 128) return bfail(nullptr, LANCET_ERR_ARG, "seq_len must be a positive multiple of 128");
    if (m.max_tokens % cfg->seq_len) return bfail(nullptr, LANCET_ERR_ARG, "max_tokens must be a multiple of seq_len");
    if (!(cfg->max_capacity_factor > 0.0)) return bfail(nullptr, LANCET_ERR_ARG, "max_capacity_factor must be > 0");
    if (world < 1 || rank < 0 || rank >= world || m.n_experts % world)
        return bfail(nullptr, LANCET_ERR_ARG, "bad world / rank");
    lancet_layer_config mc = m;
    mc.flags |= LANCET_FLAG_PEER_PUSH;
    auto* b = new lancet_block();
    b->world = world; b->rank = rank; b->device = dev; b->d = m.d_model; b->H = cfg->n_heads; b->S = cfg->seq_len;
    b->max_tokens = m.max_tokens; b->cf_max = cfg->max_capacity_factor;
    // the experts' receive buffers hold every chunk group in place: E_l static regions of
    // world * C(max_tokens, cf_max) rows + 127 pad rows per chunk (moe_forward_chunked)
    const int E_l = m.n_experts / world;
    const long Cb = capacity_rows(m.max_tokens, m.max_k, m.n_experts, cfg->max_capacity_factor);
    const long min_rows = (long)E_l * round_up((int)std::min<long>((long)world * Cb + 127L * m.max_chunks, 1L << 28), kRowAlign);
    lancet_status st = create_peer_ctx(&b->moe, world, rank, dev, &mc, min_rows);
    if (st) {
        g_block_err = lancet_last_error(nullptr);
        delete b;
        return st;
    }
    const size_t T = m.max_tokens, d = m.d_model;
    auto al = [&](void** p, size_t bytes) -> bool {
        if (cudaMalloc(p, bytes) != cudaSuccess) return false;
        b->allocs.push_back(*p);
        return true;
    };
    bool ok = al(&b->a1, T * d * 2) && al(&b->qkv, T * 3 * d * 2) && al(&b->att, T * d * 2) && al(&b->o, T * d * 2) &&
              al(&b->h, T * d * 2) && al(&b->u, T * d * 2) && al((void**)&b->mu1, T * 4) && al((void**)&b->rs1, T * 4) &&
              al((void**)&b->mu2, T * 4) && al((void**)&b->rs2, T * 4) && al((void**)&b->lse, T * 4 * cfg->n_heads) &&
              al((void**)&b->tok_tab, sizeof(int) * (2 * kMaxChunks + 2)) && al(&b->du, T * d * 2) &&
              al(&b->dh, T * d * 2) && al(&b->datt, T * d * 2) && al(&b->dqkv, T * 3 * d * 2) && al(&b->da1, T * d * 2) &&
              al((void**)&b->Dbuf, T * 4 * cfg->n_heads) &&
              al((void**)&b->ln_partial, sizeof(float) * ln_bwd_partial_floats((int)T, (int)d));
    for (int i = 0; ok && i < kMaxChunks; ++i) {
        cudaEvent_t e;
        ok = cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        if (ok) b->ev_out.push_back(e);
    }
    if (!ok || cudaStreamCreateWithFlags(&b->s_pre, cudaStreamNonBlocking) != cudaSuccess) {
        lancet_block_destroy(b);
        return bfail(nullptr, LANCET_ERR_NOMEM, "block workspace allocation failed");
    }
    *out = b;
    return LANCET_OK;
}

LANCET_API lancet_ctx* lancet_block_moe(lancet_block* b) { return b ? b->moe : nullptr; }

LANCET_API lancet_status lancet_block_destroy(lancet_block* b)
{
    if (!b) return LANCET_OK;
    lancet_status st = LANCET_OK;
    if (b->moe) st = lancet_destroy(b->moe);
    cudaSetDevice(b->device);
    for (void* p : b->allocs) cudaFree(p);
    for (cudaEvent_t e : b->ev_out) cudaEventDestroy(e);
    if (b->s_pre) cudaStreamDestroy(b->s_pre);
    delete b;
    return st;
}

namespace {
// One block's forward.  ev_in (optional, [n]): chunk c's input rows are ready once ev_in[c] has
// fired (the previous block of a stack); the block's chunk-c output records b->ev_out[c]; join =
// false leaves the internal streams un-joined (the stack joins them at its end).
lancet_status block_forward_impl(lancet_block* b, const void* x, const float* ln1_g, const float* ln1_b,
                                 const void* w_qkv, const void* w_o, const float* ln2_g, const float* ln2_b,
                                 const float* wg, const void* w1, const void* w2, int32_t T, int32_t k, double cf,
                                 int32_t n, void* out, cudaStream_t s, const cudaEvent_t* ev_in, bool join)
{
    if (!b) return bfail(nullptr, LANCET_ERR_ARG, "block is NULL");
    lancet_ctx* c = b->moe;
    lancet_status st = ctx_ready(c);
    if (st) return st;
    const void* ptrs[] = {x, ln1_g, ln1_b, w_qkv, w_o, ln2_g, ln2_b, wg, w1, w2, out};
    for (const void* p : ptrs) {
        if (!p) return bfail(b, LANCET_ERR_ARG, "null required pointer");
        if (!aligned(p)) return bfail(b, LANCET_ERR_ARG, "every tensor must be 16-byte aligned (vector loads, TMA)");
    }
    if (T < b->S || T > b->max_tokens || T % b->S) return bfail(b, LANCET_ERR_ARG, "T must be n_seq * seq_len <= max_tokens");
    const int n_seq = T / b->S;
    if (n < 1 || n > c->cfg.max_chunks || n_seq % n) return bfail(b, LANCET_ERR_ARG, "n_chunks must divide the sequences (R20)");
    const int d = b->d, Tc = T / n, seq_c = n_seq / n;
    std::vector<int> bounds(n + 1);
    for (int ch = 0; ch <= n; ++ch) bounds[ch] = ch * Tc;
    // the projection GEMMs' group tables (on the caller's stream: every internal stream forks
    // from it after this)
    launch_k(tok_tab_kernel, 1, 64, 0, s, b->tok_tab, n, Tc);
    BCK(cudaGetLastError());
    const size_t row = (size_t)d * 2;
    int extra = 1;
    ChunkedInput in;
    in.n = n;
    in.bounds = bounds.data();
    in.resid = b->h;
    in.s_pre = b->s_pre;
    in.cf_max = b->cf_max;
    in.ev_in = ev_in;
    in.ev_out = b->ev_out.data();
    in.join = join;
    in.produce = [&](int ch, int t0, int t1, cudaStream_t sp) -> lancet_status {
        const int rows = t1 - t0;
        const int* tr = b->tok_tab + ch;
        const int* to = b->tok_tab + kMaxChunks + ch;
        const char* xs = (const char*)x + t0 * row;
        size_t op = op_begin(c, "ln1", 0, ch, sp);
        int r = launch_layer_norm(xs, nullptr, nullptr, ln1_g, ln1_b, (char*)b->a1 + t0 * row, b->mu1 + t0, b->rs1 + t0,
                                  rows, d, sp);
        op_end(c, op, sp);
        if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "LayerNorm shape");
        op = op_begin(c, "qkv_proj", 0, ch, sp);
        lancet_status e = dense_gemm(c, b->a1, T, w_qkv, 3 * d, d, b->qkv, T, tr, to, 1, Tc, sp, &extra);
        op_end(c, op, sp);
        if (e) return e;
        op = op_begin(c, "attention", 0, ch, sp);
        r = launch_attention_fwd(b->qkv, b->att, b->lse, t0, seq_c, b->S, b->H, d, T, sp);
        op_end(c, op, sp);
        if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "attention: unsupported shape or tensor-map encoding failed");
        op = op_begin(c, "o_proj", 0, ch, sp);
        e = dense_gemm(c, b->att, T, w_o, d, d, b->o, T, tr, to, 1, Tc, sp, &extra);
        op_end(c, op, sp);
        if (e) return e;
        op = op_begin(c, "ln2", 0, ch, sp);
        r = launch_layer_norm(xs, (const char*)b->o + t0 * row, (char*)b->h + t0 * row, ln2_g, ln2_b,
                              (char*)b->u + t0 * row, b->mu2 + t0, b->rs2 + t0, rows, d, sp);
        op_end(c, op, sp);
        if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "LayerNorm shape");
        extra += 3;
        cudaError_t ce = cudaGetLastError();
        if (ce != cudaSuccess) return bfail(b, LANCET_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(ce));
        return LANCET_OK;
    };
    b->have_fwd = false;
    st = moe_forward_chunked(c, b->u, wg, w1, w2, T, k, cf, out, in, s);
    if (st) return st;
    c->launches_fwd += extra;
    b->T_last = T;
    b->n_last = n;
    b->x = x; b->w_qkv = w_qkv; b->w_o = w_o; b->ln1_g = ln1_g; b->ln2_g = ln2_g;
    b->have_fwd = true;
    return LANCET_OK;
}
}  // namespace

LANCET_API lancet_status lancet_block_forward(lancet_block* b, const void* x, const float* ln1_g, const float* ln1_b,
                                              const void* w_qkv, const void* w_o, const float* ln2_g,
                                              const float* ln2_b, const float* wg, const void* w1, const void* w2,
                                              int32_t T, int32_t k, double cf, int32_t n, void* out,
                                              lancet_stream_t stream_)
{
    return block_forward_impl(b, x, ln1_g, ln1_b, w_qkv, w_o, ln2_g, ln2_b, wg, w1, w2, T, k, cf, n, out,
                              reinterpret_cast<cudaStream_t>(stream_), nullptr, true);
}

// A stack of L blocks (block l's output is block l+1's input) with the chunk pipeline running
// across the blocks: block l+1's LN1 / attention of chunk c starts as soon as block l has
// combined chunk c ("the non-MoE computation ... after (e.g., the following Transformer layer)
// the MoE layer", fig:part_after_gate + fig:part_all) instead of after
// block l's whole forward.  params: [L][9] device pointers in the order ln1_g, ln1_b, w_qkv,
// w_o, ln2_g, ln2_b, wg, w1, w2 (as lancet_block_forward); outs: [L] outputs [T][d].
LANCET_API lancet_status lancet_block_forward_stack(lancet_block* const* blocks, int32_t L, const void* x,
                                                    const void* const* params, int32_t T, int32_t k, double cf,
                                                    int32_t n, void* const* outs, lancet_stream_t stream_)
{
    if (!blocks || !params || !outs || L < 1) return bfail(nullptr, LANCET_ERR_ARG, "bad stack arguments");
    for (int l = 0; l < L; ++l)
        if (!blocks[l]) return bfail(nullptr, LANCET_ERR_ARG, "null block");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    for (int l = 0; l < L; ++l) {
        lancet_block* b = blocks[l];
        const void* const* p = params + 9 * l;
        const void* in = l == 0 ? x : outs[l - 1];
        lancet_status st = block_forward_impl(b, in, (const float*)p[0], (const float*)p[1], p[2], p[3],
                                              (const float*)p[4], (const float*)p[5], (const float*)p[6], p[7],
                                              p[8], T, k, cf, n, outs[l], s,
                                              l == 0 ? nullptr : blocks[l - 1]->ev_out.data(), false);
        if (st) return st;
    }
    for (int l = 0; l < L; ++l) {
        lancet_status st = moe_join(blocks[l]->moe, blocks[l]->s_pre, s);
        if (st) return st;
    }
    return LANCET_OK;
}

// Backward of the block (the chain rule of lancet_block.h's forward, R19), on the
// caller's stream after the MoE layer's own backward (which overlaps
// its all-to-alls with its dW GEMMs):
//   du = the MoE layer's input gradient (lancet_moe_backward of dy = dout)
//   dh = dout + LN2'(du);  dW_o = dh^T att;  datt = dh W_o;  dqkv = Attn'(datt)
//   dW_qkv = dqkv^T a1;  da1 = dqkv W_qkv;  dx = dh + LN1'(da1)
// The projection weight gradients run on the compute stream after their input-gradient GEMM
// (nothing downstream waits for them).
LANCET_API lancet_status lancet_block_backward(lancet_block* b, const void* dout, void* dx, float* dln1_g,
                                               float* dln1_b, float* dw_qkv, float* dw_o, float* dln2_g,
                                               float* dln2_b, float* dwg, float* dw1, float* dw2,
                                               lancet_stream_t stream_)
{
    if (!b) return bfail(nullptr, LANCET_ERR_ARG, "block is NULL");
    lancet_ctx* c = b->moe;
    lancet_status st = ctx_ready(c);
    if (st) return st;
    if (!b->have_fwd) return bfail(b, LANCET_ERR_STATE, "block backward without a block forward");
    const void* ptrs[] = {dout, dx, dln1_g, dln1_b, dw_qkv, dw_o, dln2_g, dln2_b, dwg, dw1, dw2};
    for (const void* p : ptrs) {
        if (!p) return bfail(b, LANCET_ERR_ARG, "null required pointer");
        if (!aligned(p)) return bfail(b, LANCET_ERR_ARG, "every tensor must be 16-byte aligned");
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
    const int T = b->T_last, d = b->d, H = b->H;
    st = moe_backward_into(c, dout, b->du, dwg, dw1, dw2, s);
    if (st) return st;
    b->have_fwd = false;
    int L = 0;
    const int* all_rows = b->tok_tab + 2 * kMaxChunks;
    const int* all_off = all_rows + 1;
    size_t op = op_begin(c, "ln2_bwd", 0, -1, s);
    int r = launch_layer_norm_bwd(b->du, b->h, b->mu2, b->rs2, b->ln2_g, dout, b->dh, b->ln_partial, dln2_g, dln2_b,
                                  T, d, s);
    op_end(c, op, s);
    if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "LayerNorm backward shape");
    L += r;
    op = op_begin(c, "o_proj_dx", 0, -1, s);
    st = dense_gemm_bmn(c, b->dh, T, b->w_o, d, d, b->datt, T, all_rows, all_off, 1, T, s, &L);
    op_end(c, op, s);
    if (st) return st;
    op = op_begin(c, "o_proj_dw", 0, -1, s);
    st = dense_wgrad(c, b->dh, d, b->att, d, d, d, T, all_rows, all_off, dw_o, s, &L);
    op_end(c, op, s);
    if (st) return st;
    op = op_begin(c, "attention_bwd", 0, -1, s);
    r = launch_attention_bwd(b->qkv, b->att, b->datt, b->lse, b->Dbuf, b->dqkv, 0, T / b->S, b->S, H, d, T, s);
    op_end(c, op, s);
    if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "attention backward: shape or tensor maps");
    L += r;
    op = op_begin(c, "qkv_proj_dx", 0, -1, s);
    st = dense_gemm_bmn(c, b->dqkv, T, b->w_qkv, d, 3 * d, b->da1, T, all_rows, all_off, 1, T, s, &L);
    op_end(c, op, s);
    if (st) return st;
    op = op_begin(c, "qkv_proj_dw", 0, -1, s);
    st = dense_wgrad(c, b->dqkv, 3 * d, b->a1, d, 3 * d, d, T, all_rows, all_off, dw_qkv, s, &L);
    op_end(c, op, s);
    if (st) return st;
    op = op_begin(c, "ln1_bwd", 0, -1, s);
    r = launch_layer_norm_bwd(b->da1, b->x, b->mu1, b->rs1, b->ln1_g, b->dh, dx, b->ln_partial, dln1_g, dln1_b, T, d,
                              s);
    op_end(c, op, s);
    if (r < 0) return bfail(b, LANCET_ERR_UNSUPPORTED, "LayerNorm backward shape");
    L += r;
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return bfail(b, LANCET_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(ce));
    c->launches_bwd += L;
    return LANCET_OK;
}

LANCET_API lancet_status lancet_block_debug_copy(lancet_block* b, int32_t which, void* host, size_t bytes)
{
    if (!b || !host) return bfail(b, LANCET_ERR_ARG, "null argument");
    const size_t T = b->T_last, d = b->d;
    const void* src = nullptr;
    size_t need = 0;
    switch (which) {
    case 0: src = b->h; need = T * d * 2; break;
    case 1: src = b->u; need = T * d * 2; break;
    case 2: src = b->att; need = T * d * 2; break;
    case 3: src = b->qkv; need = T * 3 * d * 2; break;
    case 4: src = b->a1; need = T * d * 2; break;
    case 5: src = b->lse; need = (size_t)b->H * T * 4; break;    // [H][T] of the last forward
    case 6: src = b->moe->idx; need = T * b->moe->k * 4; break;   // the MoE layer's routing
    case 7: src = b->moe->slot; need = T * b->moe->k * 4; break;
    case 8: src = b->dqkv; need = T * 3 * d * 2; break;          // the last backward's
    case 9: src = b->dh; need = T * d * 2; break;
    case 10: src = b->datt; need = T * d * 2; break;
    default: return bfail(b, LANCET_ERR_ARG, "bad `which`");
    }
    if (bytes != need) return bfail(b, LANCET_ERR_ARG, "bytes must match the buffer");
    if (cudaDeviceSynchronize() != cudaSuccess) return bfail(b, LANCET_ERR_CUDA, "synchronize");
    if (cudaMemcpy(host, src, need, cudaMemcpyDeviceToHost) != cudaSuccess) return bfail(b, LANCET_ERR_CUDA, "copy");
    return LANCET_OK;
}
