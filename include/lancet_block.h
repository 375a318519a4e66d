/*
 * lancet_block.h -- C-ABI of the GPT-MoE block with Lancet's pre-MoE partition (SURVEY.md
 * §8(f) NEXT-1; BASELINE.json configs[3]).
 *
 * The operation (GPT-2 with MoE layers, Huggingface's pre-LN GPT2Block; DESIGN.md
 * R19-R22 where the paper is silent):
 *     a1 = LN1(x);  qkv = a1 W_qkv^T;  att = CausalMHA(qkv);  h = x + att W_o^T;
 *     u = LN2(h);   out = h + MoE(u)          (MoE = lancet_moe_forward's layer, include/lancet_moe.h)
 * LayerNorm: eps 1e-5, fp32 gain / bias; no projection biases; attention scale 1/sqrt(128).
 * Lancet's Opportunity 2 (L171-L173, fig:part_all, L252-L257): the batch is split into n_chunks
 * groups of whole sequences; each chunk's LN1 / attention / projections / LN2 and then its gate
 * run while the previous chunks' all-to-alls and experts are in flight, the gate of chunk c uses
 * the capacity left over by chunks 0..c-1 ("capacity passing", L255), so routing, drops and
 * results equal the unpartitioned block (L256).  Only gates that decide from partial batches
 * may be partitioned before the gate (Switch, Random; L271): Batch Prioritized Routing is
 * refused (LANCET_ERR_UNSUPPORTED, SPEC's UnsupportedGate).
 *
 * Conventions as in lancet_moe.h (device pointers, row-major, 16-byte aligned; status codes;
 * work ordered on the caller's stream).  The block's MoE layer always runs over the peer
 * transport in push mode (world 1 = a one-rank group), whose steps are device-driven.
 */
#ifndef LANCET_BLOCK_H_
#define LANCET_BLOCK_H_

#include "lancet_moe.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lancet_block lancet_block;   /* opaque, library-owned */

typedef struct {
    lancet_layer_config moe;      /* the block's MoE layer: dtype LANCET_BF16, act GELU-tanh or
                                     ReLU; LANCET_FLAG_PEER_PUSH is implied                     */
    int32_t n_heads;              /* H; head_dim = d_model / H must be 128                     */
    int32_t seq_len;              /* S: a multiple of 128; max_tokens a multiple of S          */
    double max_capacity_factor;   /* upper bound of the forwards' capacity factor: sizes the
                                     experts' receive regions (each chunk's rows must land in
                                     place before the later chunks are gated)                   */
} lancet_block_config;

/* Create rank `rank` of `world` (one process per GPU of one node, or several sharing one GPU).
 * Then set up the MoE layer's peer transport exactly as for lancet_create_peer: export the
 * blob of lancet_block_moe(b), all-gather, lancet_peer_import on it. */
lancet_status lancet_block_create_peer(lancet_block** out, int32_t world, int32_t rank, int32_t cuda_device,
                                       const lancet_block_config* cfg);
/* The block's MoE-layer context (owned by the block): peer export / import, flags, counts,
 * timeline (the block's ops are recorded in it), lancet_moe_backward of the last forward. */
lancet_ctx* lancet_block_moe(lancet_block* b);
/* Destroy (collective for world > 1, as lancet_destroy).  Safe on NULL. */
lancet_status lancet_block_destroy(lancet_block* b);

/* Forward of the block (collective when world > 1).
 *   x      [T][d]        bf16  in (caller-owned; valid until the MoE backward)
 *   ln1_g, ln1_b, ln2_g, ln2_b [d] fp32
 *   w_qkv  [3d][d]       bf16  (rows: q | k | v; head h at rows h*128.. of each)
 *   w_o    [d][d]        bf16
 *   wg     [d][E] fp32, w1 [E_l][f][d] bf16, w2 [E_l][d][f] bf16  (the MoE layer, as in
 *          lancet_moe_forward; valid until the MoE backward)
 *   T = n_seq * seq_len tokens of this rank, T <= max_tokens; k; capacity_factor in
 *   (0, max_capacity_factor]; n_chunks divides n_seq (chunks of whole sequences, R20)
 *   out    [T][d]        bf16  out
 * LANCET_FLAG_SERIAL on the MoE context: one stream, no overlap (the unoverlapped baseline).
 * Never blocks the host. */
lancet_status lancet_block_forward(lancet_block* b, const void* x, const float* ln1_g, const float* ln1_b,
                                   const void* w_qkv, const void* w_o, const float* ln2_g, const float* ln2_b,
                                   const float* wg, const void* w1, const void* w2, int32_t T, int32_t k,
                                   double capacity_factor, int32_t n_chunks, void* out, lancet_stream_t stream);

/* Forward of a stack of L blocks (collective when world > 1), block l's output feeding block
 * l+1, with the chunk pipeline running across the blocks: block l+1's LN1 / attention of chunk
 * c starts once block l has combined chunk c (the non-MoE computation after
 * the MoE layer -- the following Transformer layer -- joins the pipeline, fig:part_after_gate).
 *   blocks [L]; x [T][d] bf16 in; params [L][9] device pointers per block in the order ln1_g,
 *   ln1_b, w_qkv, w_o, ln2_g, ln2_b, wg, w1, w2 (as lancet_block_forward); outs [L] [T][d] bf16
 *   out (every block's output; each block's backward needs its own input = the previous out).
 *   The blocks must be distinct (own buffers) and share T, k, capacity_factor, n_chunks.
 * Results are bitwise those of L consecutive lancet_block_forward calls.  Never blocks. */
lancet_status lancet_block_forward_stack(lancet_block* const* blocks, int32_t L, const void* x,
                                         const void* const* params, int32_t T, int32_t k,
                                         double capacity_factor, int32_t n_chunks, void* const* outs,
                                         lancet_stream_t stream);

/* Backward of the last block forward (collective when world > 1): gradients of <dout, out>.
 *   dout [T][d] bf16 in;  dx [T][d] bf16 out;  dln1_g, dln1_b, dln2_g, dln2_b [d] fp32 out;
 *   dw_qkv [3d][d] fp32 out;  dw_o [d][d] fp32 out;  dwg [d][E] fp32 out (local, as
 *   lancet_moe_backward);  dw1 [E_l][f][d], dw2 [E_l][d][f] fp32 out.  All overwritten.
 * Runs the MoE layer's backward (its dW GEMMs overlap its all-to-alls),
 * then LN2', the output projection's gradients, the attention backward (dK/dV per key tile,
 * dQ per query tile, P recomputed from the forward's row normaliser), the q|k|v projection's
 * gradients and LN1'.  Never blocks the host.  LANCET_ERR_STATE without a preceding forward. */
lancet_status lancet_block_backward(lancet_block* b, const void* dout, void* dx, float* dln1_g, float* dln1_b,
                                    float* dw_qkv, float* dw_o, float* dln2_g, float* dln2_b, float* dwg,
                                    float* dw1, float* dw2, lancet_stream_t stream);

/* Copy an intermediate of the last forward to host (tests; synchronises).  which: 0 h [T][d],
 * 1 u = LN2(h) [T][d], 2 att [T][d], 3 qkv [T][3d], 4 a1 = LN1(x) [T][d] (all bf16), 5 lse
 * [H][T] fp32 (log2 of the attention row normaliser in the scaled log2 domain), 6 expert_idx
 * [T][k] int32, 7 slot [T][k] int32 (-1 = dropped); of the last backward: 8 dqkv [T][3d],
 * 9 dh [T][d], 10 datt [T][d] (bf16).  bytes must match. */
lancet_status lancet_block_debug_copy(lancet_block* b, int32_t which, void* host_dst, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* LANCET_BLOCK_H_ */
