// context.h -- internal definition of lancet_ctx (the library-owned state behind the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/lancet_moe.h"
#include "kernels.h"

namespace lancet {

struct Transport;   // comm.cpp: NCCL or in-process local group

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool nccl = false;   // ncclMemAlloc (NCCL transport: registrable for zero-copy send/recv)
};

// Copy-engine peer transport (world > 1 without NCCL): every rank maps the pull sources of its
// peers (CUDA IPC) and copies the rows it needs into its own buffers with cudaMemcpyAsync on
// its comm stream (copy engines, no SMs); readiness and reuse are ordered by 32-bit sequence
// flags in device memory (stream wait-value / write-value operations).
// PK_PUSH: "my rows of chunk c are in your receive buffer" (push-dispatch, LANCET_FLAG_PEER_PUSH);
// PK_XEFREE: "my receive buffer may be written for this step" (its previous readers are done).
// PK_PUSH2 / PK_DOUTFREE: the same for the dO rows pushed by K5 into the owners' dout.
enum PeerKind { PK_XS = 0, PK_OUT, PK_DCOMB, PK_DXE, PK_COUNTS, PK_PUSH, PK_XEFREE, PK_PUSH2, PK_DOUTFREE,
                PK_N };
struct PeerLinks {
    int world = 0, n_max = 0;
    std::vector<char*> src[PK_DXE + 1];   // per peer: its pull-source buffers (self: local)
    std::vector<int*> counts;             // per peer: its count matrix [G][E][n]
    std::vector<char*> xe;                // per peer: its expert-side receive buffer (push-dispatch)
    char** d_xe = nullptr;                // device copy of `xe` [G]
    std::vector<char*> dout;              // per peer: its expert-side dO buffer (push, backward)
    char** d_dout = nullptr;              // device copy of `dout` [G]
    char** d_outsrc = nullptr;            // device copy of src[PK_OUT] [G] (fused combine reads)
    int* d_push_base = nullptr;           // [n_max][E] push row base per (chunk, expert)
    std::vector<uint32_t*> flags;         // per peer: its flag array
    int* my_counts = nullptr;             // [G][E][n_max] this rank's matrix
    uint32_t* my_flags = nullptr;         // [2][PK_N][n_max][G]: ready | consumed
    uint32_t seq = 0;                     // step counter (forward)
    std::vector<void*> opened;            // IPC mappings to close
    std::vector<int> matrix;              // host copy of the last count matrix [G][E][n]
    int* h_matrix = nullptr;              // pinned staging of the matrix
    // device-side protocol of the push mode (peer.cu dev_*): the step counter lives on the
    // device so flag values are never baked into the host's enqueue (graph-capturable), and
    // waits are kernels that give up after timeout_ns and record why in err (poison)
    uint32_t* d_seq = nullptr;            // [0] step (bumped by each forward), [1] step of the
                                          // last backward
    uint32_t** d_flag_tab = nullptr;      // [G] device copy of `flags`
    int** d_counts_tab = nullptr;         // [G] device copy of `counts`
    char** d_dxesrc = nullptr;            // [G] device copy of src[PK_DXE] (K6 reads in place)
    int* d_plan_scratch = nullptr;        // [2][E][n_max] owner group rows / offsets
    uint32_t* h_err = nullptr;            // mapped pinned word: 0, or the first failed wait
    uint32_t* d_err = nullptr;            //   (device alias of h_err)
    unsigned long long timeout_ns = 60ull * 1000 * 1000 * 1000;
    unsigned long long cfg_hash = 0;      // exported in the blob, checked by every importer
    int rows_cap = 0;                     // expert-side rows allocated (pushes are bounded by it)
    size_t flag_index(int consumed, int kind, int chunk, int r) const {
        return (((size_t)consumed * PK_N + kind) * n_max + chunk) * world + r;
    }
};

struct OpEvent {
    std::string name;
    int lane, chunk;
    cudaEvent_t beg, end;
};

}  // namespace lancet

struct lancet_ctx {
    // configuration
    int world = 1, rank = 0, device = 0, E_l = 0, num_sms = 0;
    bool ep = false;           // expert-parallel path (world > 1, or LANCET_FLAG_FORCE_EP)
    lancet_layer_config cfg{};
    bool bf16 = true;
    size_t elt = 2;

    // comm
    lancet::Transport* comm = nullptr;
    lancet::PeerLinks* peer = nullptr;   // copy-engine peer transport (instead of comm)
    bool peer_ready = false;             // peers imported
    bool push = false;                   // LANCET_FLAG_PEER_PUSH, fixed at creation

    // streams / events
    cudaStream_t s_comp = nullptr, s_comm = nullptr;
    cudaStream_t s_gate = nullptr;       // partitioned forward: the chunks' gates (producer stream)
    cudaStream_t s_comp2 = nullptr;      // push pipeline: odd chunks' fc2 / dfc1 launches, so one
                                         // chunk's tail wave overlaps the next chunk's GEMM
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_counts = nullptr, ev_tl_base = nullptr;
    std::vector<cudaEvent_t> ev_pool;                 // generic sync events
    std::vector<lancet::OpEvent> ops;                 // timeline of the last fwd+bwd
    std::vector<cudaEvent_t> tl_events;               // event pool for the timeline
    size_t tl_used = 0;
    bool tl_accumulate = false;

    // source-side workspace (rows_src = max_tokens*max_k + E*128)
    int rows_src = 0;
    float* logits = nullptr;  int* idx = nullptr;  float* w = nullptr;  int* slot = nullptr;
    int* hist = nullptr;  int* S = nullptr;  int* send_rows = nullptr;  int* send_off = nullptr;
    double* bpr_score = nullptr;  int* bpr_list = nullptr;  unsigned char* bpr_adm = nullptr;
    int* bpr_hist = nullptr;  int* bpr_meta = nullptr;   // Batch Prioritized Routing scratch (R16)
    void* xs = nullptr;        // [rows_src][d]  dispatch / send buffer
    void* comb = nullptr;      // [rows_src][d]  combined expert outputs (world > 1)
    void* dcomb = nullptr;     // [rows_src][d]  grad of expert outputs (source side)
    void* dxcomb = nullptr;    // [rows_src][d]  grad of expert inputs returned (world > 1)
    float* g = nullptr;  float* dlogit = nullptr;  float* dwg_partial = nullptr;
    float* wgT = nullptr;      // [E][d] transposed gate (backward, coalesced dx gate term)
    int* prow = nullptr;       // [T][k] packed source row of each choice (-1 dropped), from K5
    int* counts_dev = nullptr;   // [E][n] send counts, then [G][E_l][n] recv counts
    int* carry = nullptr;        // [max_chunks + 1][E] capacity state carried across separately
                                 // gated chunks (block mode): pairs routed to e before chunk c
    int* grp_dev = nullptr;      // expert-side group table: rows[n_groups] | off[n_groups]

    // expert-side workspace (rows_exp rows; == rows_src when world == 1)
    int rows_exp = 0;
    void* xe = nullptr;        // [rows_exp][d]  received tokens (world > 1; == xs at world 1)
    void* H = nullptr;         // [rows_exp][f]  act(a)
    void* Gp = nullptr;        // [rows_exp][f]  act'(a)
    void* out = nullptr;       // [rows_exp][d]  expert outputs
    void* dout = nullptr;      // [rows_exp][d]  received grads of expert outputs (world > 1)
    void* dA = nullptr;        // [rows_exp][f]
    void* dXe = nullptr;       // [rows_exp][d]

    // pinned host mirrors (world > 1)
    int* h_counts = nullptr;   // send [E][n] | recv [G][E_l][n]
    int* h_grp = nullptr;

    std::vector<lancet::DevBuf> allocs;
    bool nccl_mem = false;        // NCCL transport: allocate with ncclMemAlloc and register
    int nccl_registered = 0;      // buffers registered with the communicator

    // state of the last forward (pointers only; the caller keeps the tensors alive)
    bool have_fwd = false;
    const void* x = nullptr; const float* wg = nullptr; const void* w1 = nullptr; const void* w2 = nullptr;
    int T = 0, k = 0, n = 0, C = 0;
    double cf = 0.0;
    int n_groups = 0;          // expert-side GEMM groups of the last forward
    std::vector<int> host_send, host_recv, host_grp_rows, host_grp_off;  // world > 1
    int launches_fwd = 0, launches_bwd = 0;

    // cross-layer dW scheduling (LANCET_FLAG_DEFER_DW, R17)
    uint64_t gate_seed = 0;          // Random gate (LANCET_FLAG_GATE_RANDOM, R18)
    uint32_t bwd_seq = 0;             // peer: step (PeerLinks::seq) of the last backward
    bool out_consume_pending = false; // push: the owners' outputs read by K4 are not yet released
                                      // (K5 releases them; a forward without backward does)
    int dw_pending = 0;              // bit 0: dW1, bit 1: dW2 of the last backward not enqueued
    float* pend_dw1 = nullptr;  float* pend_dw2 = nullptr;
    cudaEvent_t ev_dw_ready = nullptr;   // after the last backward's dX GEMMs
    struct Filler { lancet_ctx* other; int which; int a2a; };
    std::vector<Filler> fillers;     // consumed by the next backward

    // errors
    bool poisoned = false;
    std::string err;
};
