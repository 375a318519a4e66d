// kernels.h -- host launchers of the lancet_moe kernels (internal, C++).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

namespace lancet {

// Kernel launch with optional programmatic dependent launch (PDL): with g_pdl set, the kernel
// may start while its stream predecessor drains; every kernel of the library begins with
// pdl_wait() (common.cuh), so it observes the predecessor's writes before touching memory.
extern thread_local bool g_pdl;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- K1 / K2: routing (routing.cu) -------------------------------------------------------
struct RouteArgs {
    const void* x;        // [T][d] elt
    const float* wg;      // [d][E]
    int T, d, E, k, C, n_chunks, renorm;
    float* logits;        // [T][E]   out
    int* idx;             // [T][k]   out
    float* w;             // [T][k]   out
    int* slot;            // [T][k]   out
    int* hist;            // [n_tiles][E] scratch (zeroed here)
    int* S;               // [E][n+1] out: S[e][c] = min(C, P_e(t_c)) (capacity state)
    int* send_rows;       // [E]      out: admitted rows per expert
    int* send_off;        // [E]      out: 128-aligned packed row offset of expert e
    // Batch Prioritized Routing (R16; bpr != 0): scratch of the three-pass admission
    int bpr;
    double* score;        // [T]      importance score (fp64)
    int* list;            // [T*k]    pair ids grouped by expert, token order
    unsigned char* bpr_adm; // [T*k]  1 = admitted by priority
    int* hist2;           // [n_tiles][E] admitted pairs per token tile
    int* bpr_meta;        // [E]      pairs routed to e
    // Random gate (R18; random != 0): SplitMix64 draws instead of K1, x and Wg unused
    int random;
    unsigned long long seed;
    int t_base = 0;        // global index of token 0 of this launch (Random gate counters)
    // Capacity passing across separately gated chunks (the block's pre-MoE partition, PAPER.md
    // L255; carry_in != NULL): the launch covers one chunk `carry_chunk` of `carry_n`; pair
    // positions continue from carry_in[e] (pairs routed to e by earlier chunks), block 0 writes
    // carry_out[e] = carry_in[e] + this chunk's pairs, S[e][c], S[e][c+1] and the chunk's
    // admitted counts carry_counts[e * carry_n + c]; send_rows / send_off are not written.
    const int* carry_in = nullptr;
    int* carry_out = nullptr;
    int carry_chunk = 0, carry_n = 1;
    int* carry_counts = nullptr;
};
// Enqueues memset(hist) + K1 + K2 (K2 = three kernels under BPR).  Returns the number of kernels
// launched.
int launch_routing(const RouteArgs& a, bool is_bf16, cudaStream_t s);

// ---- K3..K6: dispatch / combine (dispatch.cu) --------------------------------------------
struct DispatchArgs {
    int T, k, d, E;
    const int* idx; const int* slot; const float* w;
    const int* send_off; const int* send_rows;
};
int launch_permute(const DispatchArgs& a, const void* x, void* xs, bool is_bf16, cudaStream_t s);
// K3 fused with the dispatch all-to-all over peer memory: tokens [t0, t1) of one chunk, row
// x[t] of choice (t, j) -> xe_ptrs[e / E_l] + (base[e] + slot) rows
int launch_permute_push(const DispatchArgs& a, const void* x, int t0, int t1, int E_l, const int* base,
                        char* const* xe_ptrs, bool is_bf16, cudaStream_t s);
// src_base / src_tab (fused combine exchange, optional): o rows read from src_tab[e / E_l] at
// rows src_base[e] + slot (the owners' expert outputs over peer memory) instead of comb
// resid (optional, [T][d]): y = resid + sum_j w_j o_j, the block's residual add (fp32 chain from resid)
int launch_combine(const DispatchArgs& a, const void* comb, void* y, int t0, int t1, bool is_bf16,
                   cudaStream_t s, const int* src_base = nullptr, const char* const* src_tab = nullptr,
                   int E_l = 1, const void* resid = nullptr);
// K5: also writes dlogit [T][E] (softmax Jacobian) and prow [T][k] (packed row or -1)
// push_base / push_dst (peer push, optional): the dO rows go to push_dst[e / E_l] at rows
// push_base[e] + slot instead of dcomb (backward all-to-all #1 fused into K5)
int launch_combine_bwd(const DispatchArgs& a, const void* dy, const void* comb, float* g,
                       void* dcomb, int t0, int t1, bool zero_pads, const float* logits, int renorm,
                       float* dlogit, int* prow, bool is_bf16, cudaStream_t s, const int* push_base = nullptr,
                       char* const* push_dst = nullptr, int E_l = 1, const char* const* src_tab = nullptr);
int launch_wg_transpose(const float* wg, int d, int E, float* wgT, cudaStream_t s);
bool gate_bwd_needs_wgT(int d, int E);   // true: the general K6 reads Wg^T (launch_wg_transpose)
// K6: dx_t = sum_j dX[prow_tj] + sum_e dlogit_te Wg[:, e]   (wg [d][E]; wgT = Wg transposed,
// [E][d], only read by the general path)
// src_tab (push mode, optional): prow holds (owner << kPeerRowBits) | row and the dX rows are
// read in place from src_tab[owner] (the owners' dX buffers over peer memory) instead of dxe
int launch_unpermute_gate_bwd(const DispatchArgs& a, const void* dxe, const int* prow,
                              const float* dlogit, const float* wg, const float* wgT, void* dx, int t0, int t1,
                              int num_sms, bool is_bf16, cudaStream_t s, const char* const* src_tab = nullptr);
// dWg = x^T dlogit (K7); partial: [ceil(T/64)][d][E] fp32 scratch
int launch_dwg(const void* x, const float* dlogit, int T, int d, int E, float* partial,
               float* dwg, bool is_bf16, int num_sms, cudaStream_t s);
size_t dwg_partial_floats(int T, int d, int E);
// K6 + K7 in one pass over all tokens (world 1; E <= 8, d % 256 == 0, d <= 2048, k <= 4):
// dx and dWg (partials + deterministic reduction).  Returns launches, or -1 if unsupported.
bool gate_bwd_fused_ok(int d, int E, int k);
int launch_gate_bwd_fused(const DispatchArgs& a, const void* dxe, const int* prow, const float* dlogit,
                          const float* wg, const void* x, void* dx, float* partial, float* dwg,
                          int num_sms, bool is_bf16, cudaStream_t s);
// zero rows [off_g + rows_g, off_g + round_up(rows_g, 128)) of a packed buffer
int launch_zero_pads(void* buf, int row_elems, const int* grp_off, const int* grp_rows,
                     int n_groups, int elt_bytes, cudaStream_t s);

// ---- the GPT-MoE block's non-MoE kernels (attention.cu) ----------------------------------
// Causal self-attention, head_dim 128, S % 128 == 0, d = H * 128: qkv [T_all][3d] (q | k | v),
// the n_seq sequences starting at token tok0; att [T_all][d] and lse [H][T_all] (log2 domain)
// written for those tokens.  Returns -1 if unsupported or the tensor maps fail.
int launch_attention_fwd(const void* qkv, void* att, float* lse, int tok0, int n_seq, int S, int H, int d,
                         int T_all, cudaStream_t s);
// LayerNorm over rows of d (d % 256 == 0, d <= 4096): y = (x - mean) rstd g + b, bf16; with
// resid != NULL the row is first h = bf16(a + resid), stored to hout.  mean / rstd [rows] out.
int launch_layer_norm(const void* a, const void* resid, void* hout, const float* g, const float* b, void* y,
                      float* mean, float* rstd, int rows, int d, cudaStream_t s);

// Backward of the causal attention (attention_bwd.cu): dqkv [T_all][3d] bf16 (dq | dk | dv) of
// the n_seq sequences starting at tok0, from qkv, att (= O), datt (= dO), lse (forward's, log2
// domain); Dbuf [H][T_all] fp32 scratch (D = rowsum(dO O)).  Returns launches or -1.
int launch_attention_bwd(const void* qkv, const void* att, const void* datt, const float* lse, float* Dbuf,
                         void* dqkv, int tok0, int n_seq, int S, int H, int d, int T_all, cudaStream_t s);
// LayerNorm backward: out = resid + dLN/dx (bf16), dg / db [d] fp32 (overwritten); x is the LN
// input (bf16), mean / rstd the forward's; partial: ln_bwd_partial_floats(rows, d) fp32 scratch.
int launch_layer_norm_bwd(const void* dy, const void* x, const float* mean, const float* rstd, const float* g,
                          const void* resid, void* out, float* partial, float* dg, float* db, int rows, int d,
                          cudaStream_t s);
size_t ln_bwd_partial_floats(int rows, int d);

// ---- grouped GEMMs (gemm_simt.cu, gemm_tc.cu) --------------------------------------------
enum GemmMode { GEMM_M_GROUPED = 0, GEMM_K_GROUPED = 1 };
enum GemmEpi { EPI_STORE = 0, EPI_ACT = 1, EPI_DACT = 2, EPI_F32 = 3 };

// Device-side chunk pipeline of one GEMM launch over all chunks (push mode).  Groups are in
// chunk-major table order (gpc groups per chunk).  wait_flags != NULL: before the first load of
// chunk c's tiles the TMA producer spins until every rank's flag wait_flags[c*stride + r]
// reaches seq[0] (then every row of chunk c has landed; the rows were written by a completed
// kernel and published by a flag kernel after it).  A wait that exceeds timeout_ns records
// err_code | chunk << 8 | rank in *err and gives up (the context is poisoned at its next call).
struct ChunkSync {
    int gpc = 0, ranks = 0;
    const uint32_t* wait_flags = nullptr;
    long wait_chunk_stride = 0;
    const uint32_t* seq = nullptr;
    unsigned long long timeout_ns = 0;
    uint32_t* err = nullptr;
    uint32_t err_code = 0;
};

struct GemmArgs {
    // A(m,k): A_MN ? A[(row0+k)*lda + m] : A[(row0+m)*lda + k]
    const void* A; long lda;
    // B(n,k): B_MN ? B[(krow0+k)*ldb + n] : B[n*ldb + k], B += (g / gpw) * b_group_stride
    const void* B; long ldb; long b_group_stride;
    // C(m,n): M-grouped C[(row0+m)*ldc + n];  K-grouped C[g*c_group_stride + m*ldc + n]
    void* C; long ldc; long c_group_stride;
    void* C2;             // EPI_ACT: act'(a) stored beside act(a) (same layout as C)
    const void* aux;      // EPI_DACT: act'(a) multiplied into the accumulator
    int M, N, K;          // M-grouped: N, K fixed, rows per group from the table;
                          // K-grouped: M, N fixed, K per group from the table
    int max_rows;         // M-grouped: upper bound of round_up(rows_g, 128) (grid sizing)
    int mode, n_groups, gpw;
    int n_weights;        // B group index = (g / gpw) % n_weights (groups of several chunks)
    const int* grp_rows;  // [n_groups] valid rows (M-grouped) / tokens (K-grouped)
    const int* grp_off;   // [n_groups] first row (128-aligned) in A / C (M) or A / B (K)
    int epi, act, accumulate;
    bool a_mn, b_mn;
    long a_rows, b_rows;  // outer extents of A and B viewed as 2D row-major tensors (TMA maps)
    long c_rows;          // outer extent of C / C2 / aux (M-grouped; TMA store maps)
    bool multicast;       // tcgen05: two CTA pairs share each A tile by TMA multicast
    ChunkSync cs;         // tcgen05, M-grouped: device-side chunk pipeline (push mode)
};
int launch_gemm_simt(const GemmArgs& a, bool is_bf16, cudaStream_t s);

// tcgen05 / TMEM / TMA grouped GEMM, bf16 in, fp32 accumulate (gemm_tc.cu).
// Returns <0 if the shape is unsupported (caller reports LANCET_ERR_UNSUPPORTED).
int launch_gemm_tc(const GemmArgs& a, int num_sms, cudaStream_t s);
bool gemm_tc_supported(const GemmArgs& a);

}  // namespace lancet
