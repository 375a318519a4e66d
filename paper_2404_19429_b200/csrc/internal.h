// internal.h -- C++ entry points of lancet.cu used by the GPT-MoE block (block.cu); not part of
// the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <string>

#include "context.h"

namespace lancet {

// The MoE input of the block arrives chunk by chunk (Lancet's pre-MoE partition, PAPER.md
// L252-L257, fig:part_all): `produce(ch, t0, t1, s)` enqueues on stream s everything that writes
// rows [t0, t1) of the MoE input x (and of `resid`); each chunk is then gated on its own with the
// capacity state carried over from the earlier chunks (L255), its sizes exchanged, its rows
// pushed to the owners, its experts run and its outputs combined -- while the producer already
// computes the next chunk.  y = resid + MoE(x) (resid may be NULL).
struct ChunkedInput {
    int n = 1;
    const int* bounds = nullptr;     // host [n + 1] token boundaries
    std::function<lancet_status(int ch, int t0, int t1, cudaStream_t s)> produce;
    const void* resid = nullptr;
    cudaStream_t s_pre = nullptr;    // the producer's stream
    double cf_max = 0.0;             // bound of the capacity factor (static receive regions)
    // chunk pipeline across consecutive layers (a stack of blocks): the producer of chunk c
    // first waits for ev_in[c] (the previous block's chunk-c output is stored), the combine of
    // chunk c records ev_out[c]; join = false leaves the internal streams un-joined to the
    // caller's stream (the stack joins every block at its end: moe_join)
    const cudaEvent_t* ev_in = nullptr;
    cudaEvent_t* ev_out = nullptr;
    bool join = true;
};
// make `s` wait for everything the context's streams (and `extra`) have enqueued
lancet_status moe_join(lancet_ctx* c, cudaStream_t extra, cudaStream_t s);
lancet_status moe_forward_chunked(lancet_ctx* c, const void* x, const float* wg, const void* w1, const void* w2,
                                  int T, int k, double cf, void* y, const ChunkedInput& in, cudaStream_t s);

// C[rows of each group] = A[rows] B^T on the tcgen05 GEMM; B [N][K] K-major; groups from device
// tables (rows / first row, 128-aligned); SMs reserved for the exchange kernels as for the
// expert GEMMs of the context.
lancet_status dense_gemm(lancet_ctx* c, const void* A, long a_rows, const void* B, int N, int K, void* C,
                         long c_rows, const int* grp_rows, const int* grp_off, int n_groups, int max_rows,
                         cudaStream_t s, int* launches);

// C[rows] = A[rows] B for B stored [K][N] row-major (read as an MN-major operand): the
// projections' input gradients dX = dY W
lancet_status dense_gemm_bmn(lancet_ctx* c, const void* A, long a_rows, const void* B, int N, int K, void* C,
                             long c_rows, const int* grp_rows, const int* grp_off, int n_groups, int max_rows,
                             cudaStream_t s, int* launches);
// C[M][N] (fp32, overwritten) = sum over the group's rows t of A[t][m] B[t][n] (K-grouped, one
// group): the projections' weight gradients dW = dY^T X
lancet_status dense_wgrad(lancet_ctx* c, const void* A, int lda, const void* B, int ldb, int M, int N, long rows_ext,
                          const int* grp_rows, const int* grp_off, float* C, cudaStream_t s, int* launches);
lancet_status moe_backward_into(lancet_ctx* c, const void* dy, void* dx, float* dwg, float* dw1, float* dw2,
                                cudaStream_t s);

// timeline records of the context (LANCET_FLAG_TIMELINE): begin returns a handle for end
size_t op_begin(lancet_ctx* c, const char* name, int lane, int chunk, cudaStream_t s);
void op_end(lancet_ctx* c, size_t h, cudaStream_t s);

lancet_status record_error(lancet_ctx* c, lancet_status st, const std::string& msg);
lancet_status ctx_ready(lancet_ctx* c);
// a peer-transport context whose expert-side buffers hold at least min_rows rows
lancet_status create_peer_ctx(lancet_ctx** out, int world, int rank, int device, const lancet_layer_config* cfg,
                              long min_rows);
int capacity_rows(int T, int k, int E, double cf);

}  // namespace lancet
