/*
 * lancet_moe.h -- C-ABI of the B200-native expert-parallel MoE layer step
 * (Lancet, arXiv 2404.19429: "Accelerating Mixture-of-Experts Training via Whole Graph
 *  Computation-Communication Overlapping").
 *
 * Citations are PAPER.md line numbers (P:Lnnn) of /root/reference/PAPER.md and DESIGN.md
 * readings (Rn) where the paper is silent.
 *
 * The operation:
 *   Each of G ranks holds T tokens x[T][d] (data parallel) and E_l = E/G experts
 *   (expert parallel; expert e lives on rank e / E_l, "G = E / E_l").
 *   forward:  logit = x Wg (fp32, R1); top-k by logit (R2); combine weight
 *             w = softmax(logit)[idx] (R3); capacity C = max(1, min(T, ceil(cf*k*T/E))) per
 *             (rank, expert) (R4); token-major admission (R7) -- chunked routing
 *             equals unchunked routing, which is Lancet's capacity passing;
 *             dispatch all-to-all (irregular: P:L517-L526); expert FFN
 *             o = act(x W1^T) W2^T (R5); combine all-to-all; gather
 *             y_t = sum_{admitted j} w_tj o_tj (dropped -> 0, R6).
 *   The batch is split into n_chunks contiguous chunks (R9); the all-to-all of
 *   chunk c overlaps expert compute of other chunks, and in the backward the
 *   weight-gradient GEMMs are issued right after an all-to-all launch so they overlap it
 *   (P:L168-L169).
 *
 * Conventions
 *   - All tensor pointers are DEVICE pointers on the context's CUDA device unless marked
 *     (host).  Row-major, densely packed, 16-byte aligned.
 *   - "dtype" tensors are bf16 (LANCET_BF16) or fp32 (LANCET_FP32); the gate Wg, combine
 *     weights and all weight gradients are always fp32.
 *   - Every function returns a lancet_status; no C++ exception crosses the ABI.  Argument
 *     errors return LANCET_ERR_ARG before anything is enqueued.  CUDA / NCCL failures
 *     return LANCET_ERR_CUDA / LANCET_ERR_NCCL and poison the context (every later call
 *     returns LANCET_ERR_STATE).  lancet_last_error() gives the message.
 *   - Work is enqueued on the caller's `stream` (ordered after prior work on it); results
 *     are valid for later work on `stream`.  Internally the library forks to its own
 *     compute / comm streams and joins back with events.
 */
#ifndef LANCET_MOE_H_
#define LANCET_MOE_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LANCET_ABI_VERSION 2

typedef struct lancet_ctx lancet_ctx;                 /* opaque, library-owned */
typedef struct lancet_local_group lancet_local_group; /* opaque, library-owned */
typedef void* lancet_stream_t;                        /* a cudaStream_t (0 = legacy default) */

typedef enum {
    LANCET_OK = 0,
    LANCET_ERR_ARG = 1,          /* invalid argument; nothing was enqueued               */
    LANCET_ERR_CUDA = 2,         /* CUDA runtime / driver error; context poisoned        */
    LANCET_ERR_NCCL = 3,         /* NCCL error; context poisoned                         */
    LANCET_ERR_NOMEM = 4,        /* device or pinned allocation failed                   */
    LANCET_ERR_STATE = 5,        /* call out of order, or context poisoned               */
    LANCET_ERR_UNSUPPORTED = 6   /* valid request this build / device does not support   */
} lancet_status;

typedef enum { LANCET_BF16 = 0, LANCET_FP32 = 1 } lancet_dtype;

/* Expert activation (R5).  IDENTITY_EXPERT: o = x (no GEMMs; W1/W2 ignored and may be
 * NULL) -- the dispatch/combine test mode of the north star. */
typedef enum {
    LANCET_ACT_GELU_TANH = 0,
    LANCET_ACT_RELU = 1,
    LANCET_ACT_IDENTITY_EXPERT = 2
} lancet_act;

/* SMs (= NCCL CTAs) reserved for the all-to-all at world > 1 (see gemm_sms). */
#define LANCET_COMM_SMS 8

/* Behaviour flags (lancet_layer_config.flags, or lancet_set_flags). */
enum {
    LANCET_FLAG_RENORMALIZE = 1u << 0,  /* w = p[idx] / sum_j p[idx_j] (R3); default off     */
    LANCET_FLAG_TIMELINE    = 1u << 1,  /* record per-op events (lancet_last_timeline)       */
    LANCET_FLAG_SERIAL      = 1u << 2,  /* unoverlapped baseline: one stream, chunks merged,
                                           no dW reordering (the "unoverlapped a2a" of §8(d)) */
    LANCET_FLAG_SIMT_GEMM   = 1u << 3,  /* bf16: use the SIMT GEMM instead of tcgen05 (debug) */
    LANCET_FLAG_NO_DW_OVERLAP = 1u << 4,/* backward: dW GEMMs after all a2a (ablation)       */
    LANCET_FLAG_NO_SIDE_STREAM = 1u << 5,/* world 1 backward: K6/K7 on the caller stream, in
                                           line with the GEMMs (A/B of the side stream)      */
    LANCET_FLAG_GEMM_MULTICAST = 1u << 6,/* tcgen05 GEMMs: clusters of two CTA pairs sharing each
                                           A tile by TMA multicast.  Off by default: clusters
                                           of 4 fit on 132 of the 148 SMs, which costs more
                                           than the L2 traffic it saves (profiles/)          */
    LANCET_FLAG_UNFUSED_GATE_BWD = 1u << 7,/* world 1 with NO_SIDE_STREAM: K6 and K7 as two
                                           kernels even where the fused single pass applies  */
    LANCET_FLAG_NO_PDL = 1u << 8,       /* disable programmatic dependent launch (default on:
                                           each kernel may start while its stream predecessor
                                           drains; every kernel waits with griddepcontrol.wait
                                           before touching memory; ~1 % per step)            */
    LANCET_FLAG_FORCE_EP = 1u << 9,     /* run the expert-parallel path (chunked NCCL
                                           exchanges, S1/S2 scheduler) even at world 1, over a
                                           one-rank NCCL communicator (lancet_create needs an
                                           NCCL id); fixed at creation (lancet_set_flags keeps
                                           the creation bit).  Exercises the NCCL path on a
                                           single GPU                                         */
    LANCET_FLAG_TIMELINE_GEMM_ONLY = 1u << 10,/* with TIMELINE: events around the expert GEMM
                                           launches only (the least perturbing roofline pass) */
    LANCET_FLAG_GATE_BPR = 1u << 11,    /* Batch Prioritized Routing (DESIGN.md
                                           R16) instead of token-major admission: the pairs of
                                           each expert are admitted by the token's importance
                                           score s_t = sum_j p[t, idx_tj] (fp64; descending,
                                           ties to the lower token), so lower scores are dropped
                                           first; admitted pairs then take token-major slots.
                                           The gate sees the whole local batch and the chunks
                                           partition after it (fig:part_after_gate, L271), so
                                           chunked == unchunked as with the Switch gate.
                                           Costs two more routing kernels per forward        */
    LANCET_FLAG_DEFER_DW = 1u << 12,    /* backward: do not enqueue this layer's dW GEMMs; they
                                           stay pending (dW1 and dW2 separately) until
                                           lancet_moe_backward_dw or another context's filler
                                           slot enqueues them (cross-layer dW scheduling,
                                           PAPER.md L156, L348-L398; R17).  The next
                                           forward fails with LANCET_ERR_STATE while any are
                                           pending                                           */
    LANCET_FLAG_GATE_RANDOM = 1u << 13, /* Random gating (R18): token
                                           t's j-th expert is drawn by SplitMix64 from counter
                                           8t + j and the seed of lancet_set_gate_seed (distinct
                                           experts, uniform), combine weights 1/k, token-major
                                           admission.  No gate network: Wg is not read, logits
                                           are reported as 0, dwg is 0 and dx has no gate term.
                                           Exclusive with LANCET_FLAG_GATE_BPR (ERR_ARG)       */
    LANCET_FLAG_PEER_PUSH = 1u << 14,   /* peer transport: the dispatch all-to-all is fused into
                                           the permute kernel -- each admitted row is written
                                           straight into the owning rank's receive buffer (IPC-
                                           mapped peer memory; NVLink across GPUs) at its final
                                           row, one launch per chunk, readiness signalled per
                                           chunk by flags; no send buffer and no copy-engine
                                           pass.  Likewise the backward's first all-to-all:
                                           K5 writes its dO rows straight into the owners' dO
                                           buffers; and the combine: K4 / K5 read the expert
                                           outputs in place from the owners' buffers, and K6
                                           reads the dX rows in place from the owners' dX
                                           buffers (backward #2).  The exchange plan is built on
                                           the device from the gathered count matrix and every
                                           readiness flag is a kernel, so the step never waits on
                                           the host and can be captured in a CUDA graph.  The
                                           fused kernels run on the comm stream beside the
                                           expert GEMMs (which leave LANCET_COMM_SMS SMs free).
                                           Fixed at creation (lancet_set_flags keeps the creation
                                           bit); checked identical on every rank at
                                           lancet_peer_import                                   */
    LANCET_FLAG_CHUNK_LAUNCHES = 1u << 16,/* push mode: one expert-GEMM launch per chunk ordered
                                           by flag kernels on the host's enqueue (the A/B of the
                                           default: one launch over all chunks whose TMA producer
                                           waits for each chunk's rows on the device and whose
                                           epilogue publishes each chunk's outputs, with the dW
                                           GEMMs merged over the chunks)                         */
    LANCET_FLAG_NO_COMM = 1u << 15      /* TIMING ONLY (results are wrong): skip the data
                                           exchanges (NCCL / copy-engine: the C2 copies; push
                                           mode: the four fused exchange kernels) but keep every
                                           other op and wait -- T_step - T_step(NO_COMM) bounds
                                           the exposed exchange time from above  */
};

typedef struct {
    int32_t d_model;      /* d                                                         */
    int32_t d_ffn;        /* f                                                         */
    int32_t n_experts;    /* E (total over all ranks); E % world == 0                  */
    int32_t max_tokens;   /* upper bound on T per call (sizes the workspace)           */
    int32_t max_k;        /* upper bound on k                                          */
    int32_t max_chunks;   /* upper bound on n_chunks (<= 64)                           */
    int32_t dtype;        /* lancet_dtype                                              */
    int32_t act;          /* lancet_act                                                */
    uint32_t flags;       /* LANCET_FLAG_*                                             */
    int32_t gemm_sms;     /* SMs the persistent GEMMs may use.  0 = all SMs at world 1;
                             at world > 1 (NCCL) all but LANCET_COMM_SMS, which the NCCL
                             communicator is created to use (ncclConfig_t.maxCTAs), so the
                             all-to-all kernels always find free SMs beside the
                             persistent GEMMs and overlap them instead of queueing      */
} lancet_layer_config;

/* Per-op record of the last forward/backward (LANCET_FLAG_TIMELINE).  Times are
 * microseconds from the start event recorded on the caller's stream. */
typedef struct {
    char name[24];        /* e.g. "gate", "a2a_dispatch[2]", "expert_fc1[2]"          */
    int32_t lane;         /* 0 = compute stream, 1 = comm stream, 2 = side compute    */
    int32_t chunk;        /* chunk index or -1                                         */
    float start_us;
    float end_us;
} lancet_op_record;

int32_t lancet_abi_version(void);

/* Message for the last error of `ctx`, or of the calling thread if ctx == NULL. */
const char* lancet_last_error(const lancet_ctx* ctx);

/* Rank 0 creates the NCCL unique id (128 bytes, host); the caller broadcasts it. */
lancet_status lancet_nccl_unique_id(void* id_out /* host, 128 B */);

/* Create a context for `rank` of `world`.  world == 1: no communication (id ignored).
 * world > 1: NCCL communicator from `nccl_id` (host, 128 B); collective over all ranks,
 * each on its own device.  The config must be identical on every rank (checked). */
lancet_status lancet_create(lancet_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                            const void* nccl_id, const lancet_layer_config* cfg);

/* Simulated ranks in ONE process on ONE device (tests of the multi-rank data path without
 * several GPUs): the group is the transport; data all-to-alls become device-to-device
 * copies between the ranks' buffers, ordered with events exactly where NCCL would
 * synchronise.  Each rank's calls must be made from its own host thread (they block at the
 * exchange points like a collective). */
lancet_status lancet_local_group_create(lancet_local_group** out, int32_t world);
lancet_status lancet_local_group_destroy(lancet_local_group* group);
lancet_status lancet_create_local(lancet_ctx** out, lancet_local_group* group, int32_t rank,
                                  int32_t cuda_device, const lancet_layer_config* cfg);

/* Copy-engine peer transport (no NCCL; one process per rank, all ranks' devices reachable by
 * CUDA IPC -- one NVSwitch node, or several processes sharing one GPU).  Every rank maps its
 * peers' pull-source buffers and copies the rows it needs into its own buffers with
 * cudaMemcpyAsync on its comm stream (copy engines: no SMs taken from the expert GEMMs); the
 * chunk readiness / buffer reuse across processes is ordered by sequence flags in device
 * memory (stream wait-value / write-value operations).  Expert-side buffers are allocated at
 * their bound (world * max_tokens * max_k rows) at creation.  Setup:
 *   1. lancet_create_peer on every rank;
 *   2. lancet_peer_export: this rank's blob (lancet_peer_blob_bytes() bytes, host);
 *   3. the caller all-gathers the blobs (rank order) over its own channel;
 *   4. lancet_peer_import with the world blobs (host, world * blob bytes).
 * Then forward / backward as with NCCL (collective: every rank calls them in the same order).
 * The blob holds CUDA IPC handles; it is only meaningful to processes of the same node. */
lancet_status lancet_create_peer(lancet_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                                 const lancet_layer_config* cfg);
size_t lancet_peer_blob_bytes(void);
lancet_status lancet_peer_export(lancet_ctx* ctx, void* blob /* host, lancet_peer_blob_bytes() */);
lancet_status lancet_peer_import(lancet_ctx* ctx, const void* blobs /* host, world blobs */);
/* Import checks every blob's configuration hash (d_model, d_ffn, n_experts, max_tokens, max_k,
 * max_chunks, dtype, act, RENORMALIZE, PEER_PUSH, world) and rank: LANCET_ERR_CUDA with a
 * message naming the disagreeing rank otherwise.
 *
 * Failure handling of the peer transport.  Push mode (LANCET_FLAG_PEER_PUSH): every wait is
 * a kernel that gives up after the timeout (default 60 s, env LANCET_PEER_TIMEOUT_MS, or
 * lancet_set_peer_timeout_ms) and records which rank / flag it missed; the step's results are
 * then undefined and every later call on the context returns LANCET_ERR_STATE naming the
 * flag.  lancet_peer_abort (any mode, e.g. from a watchdog thread of the caller): sets every
 * flag of this rank so that all its pending waits -- stream wait-value operations of the
 * copy-engine mode included -- return, and poisons the context.  lancet_peer_status: the
 * context's asynchronous error state without blocking (LANCET_OK, or LANCET_ERR_STATE). */
lancet_status lancet_set_peer_timeout_ms(lancet_ctx* ctx, int64_t ms);
lancet_status lancet_peer_abort(lancet_ctx* ctx);
lancet_status lancet_peer_status(lancet_ctx* ctx);

/* Destroy; aborts the communicator if the context is poisoned.  Safe on NULL.  Peer
 * transport: collective -- peers read this rank's buffers over IPC, so destroy first waits
 * (bounded by the peer timeout) until every peer has signalled that it consumed this rank's
 * rows of the last step, then unmaps and frees; call it on every rank after the last step. */
lancet_status lancet_destroy(lancet_ctx* ctx);

lancet_status lancet_set_flags(lancet_ctx* ctx, uint32_t flags);

/* Seed of the Random gate (LANCET_FLAG_GATE_RANDOM) for the following forwards; default 0. */
lancet_status lancet_set_gate_seed(lancet_ctx* ctx, uint64_t seed);

/* Forward of the MoE layer (collective when world > 1).
 *   x   [T][d]      dtype   caller-owned; must stay valid and unmodified until backward
 *   wg  [d][E]      fp32    replicated gate
 *   w1  [E_l][f][d] dtype   this rank's experts e = rank*E_l + i; valid until backward
 *   w2  [E_l][d][f] dtype
 *   T in [1, max_tokens]; k in [1, min(E, max_k)]; capacity_factor > 0 (double: the
 *   capacity C = max(1, min(T, ceil(cf k T / E))) is evaluated in double, R4);
 *   n_chunks in [1, min(T, max_chunks)]
 *   y          [T][d] dtype  out
 *   expert_idx [T][k] int32  out or NULL   (rank order; idx[:,0] is the best expert)
 *   slot       [T][k] int32  out or NULL   (position in the expert's buffer; -1 = dropped)
 *   combine_w  [T][k] fp32   out or NULL
 * world > 1 over NCCL or the copy-engine peer transport: blocks the host once (the counts
 * exchange of P:L525 must reach the host to size the NCCL sends / the copies).  world == 1
 * and the push mode of the peer transport: never blocks (plan built on the device).
 * One outstanding forward per context: a second forward before backward is allowed (the
 * first is discarded); backward without forward returns LANCET_ERR_STATE. */
lancet_status lancet_moe_forward(lancet_ctx* ctx, const void* x, const float* wg,
                                 const void* w1, const void* w2, int32_t T, int32_t k,
                                 double capacity_factor, int32_t n_chunks, void* y,
                                 int32_t* expert_idx, int32_t* slot, float* combine_w,
                                 lancet_stream_t stream);

/* Forward with Lancet's partition BEFORE the gate (fig:part_all; the MoE
 * stage of lancet_block_forward, include/lancet_block.h): every chunk of the batch is gated on
 * its own, with the capacity left over by the earlier chunks ("capacity passing", L255), its
 * sizes exchanged (L525) and its rows pushed / computed / combined before later chunks are
 * gated.  Same arguments and results as lancet_moe_forward -- routing, drops and y equal the
 * unpartitioned layer (L256) -- plus resid [T][d] (optional): y = resid + MoE(x), the block's
 * residual fused into the combine.  Needs the peer transport in push mode; the experts'
 * receive buffers must hold E_l static regions of world * C(max_tokens) + 127 * n_chunks rows
 * (LANCET_ERR_ARG otherwise; lancet_block_create_peer sizes them).  Batch Prioritized Routing
 * needs the whole batch: LANCET_ERR_UNSUPPORTED (L270-L271).  lancet_moe_backward follows as
 * usual.  Never blocks the host. */
lancet_status lancet_moe_forward_partitioned(lancet_ctx* ctx, const void* x, const float* wg,
                                             const void* w1, const void* w2, int32_t T, int32_t k,
                                             double capacity_factor, int32_t n_chunks, const void* resid,
                                             void* y, int32_t* expert_idx, int32_t* slot, float* combine_w,
                                             lancet_stream_t stream);

/* Backward of the last forward (collective when world > 1).  Gradient of <dy, y>:
 *   dy  [T][d]      dtype  in
 *   dx  [T][d]      dtype  out (overwritten)
 *   dwg [d][E]      fp32   out (overwritten) -- LOCAL: the caller all-reduces it
 *   dw1 [E_l][f][d] fp32   out (overwritten; NULL allowed for identity experts)
 *   dw2 [E_l][d][f] fp32   out (overwritten; NULL allowed for identity experts)
 * Never blocks the host. */
lancet_status lancet_moe_backward(lancet_ctx* ctx, const void* dy, void* dx, float* dwg,
                                  float* dw1, float* dw2, lancet_stream_t stream);

/* Cross-layer dW scheduling (PAPER.md Opportunity 1, L156 "overlapped with any dWs in layer
 * N+k"; Alg. 1 placement L359 "placing them right after their overlapping all-to-all
 * instructions"; R17).
 *
 * lancet_moe_backward_dw: enqueue the pending dW GEMMs of `ctx`'s last backward (run with
 *   LANCET_FLAG_DEFER_DW) on `stream`, ordered after that backward's dX GEMMs by an event.
 *   which: bit 0 = dW1 (dA^T X), bit 1 = dW2 (dO^T H); both write the dw1 / dw2 pointers the
 *   backward was given (fp32, all chunks, in chunk order).  LANCET_ERR_STATE if a requested
 *   part is not pending.
 * lancet_set_dw_fillers: for the NEXT backward of `ctx` only -- right after that backward
 *   launches its all-to-all number a2a_index[i] (issue order: 0..n-1 = the per-chunk
 *   dispatch of dO to the experts, n..2n-1 = the per-chunk return of dX), enqueue the pending
 *   dW part which[i] of others[i] on the backward's compute stream.  An index the backward
 *   never reaches (e.g. world 1: no all-to-all) is served at its end.  others[i] may be ctx
 *   itself (its own dW placed under its own dX return).  Pointers are host arrays of n
 *   entries, copied.  The other contexts must outlive the call and keep their forward's
 *   buffers (no forward of theirs in between).
 * lancet_dw_schedule: Alg. 1 on any instruction DAG (host only, no device).  kind[i]: 0 other,
 *   1 all-to-all, 2 dW; cost[i] in any time unit; edges [n_edges][2] (src, dst) = dst
 *   consumes src.  assign[i] (out) = the all-to-all instruction dW i overlaps, else -1.
 *   Labelling: no directed path either way (L343); assignment: all-to-alls in program
 *   order, while unoverlapped time t_u > 0 take the unused eligible dW minimising
 *   |t_u - t_W| (ties -> lowest index).  LANCET_ERR_ARG on bad sizes / indices.
 * lancet_stack_dw_plan: the backward program of an L-layer stack of this layer (layers in
 *   forward order, backward runs L-1 first; per layer the per-chunk K5, dO a2a, dX GEMMs,
 *   then dW2, dW1, the per-chunk dX a2a, K6, K7 -- DESIGN.md R17) scheduled by Alg. 1.
 *   t_a2a [L][2n] (the layer's a2a in issue order), t_dw [L][2] (dW2, dW1).  Outputs per
 *   (layer, part) [L][2] (part 0 = dW2, 1 = dW1): host_layer = the layer whose backward
 *   carries it, host_a2a = the a2a index there, or -1 / -1 = unassigned (keep in place). */
lancet_status lancet_moe_backward_dw(lancet_ctx* ctx, int32_t which, lancet_stream_t stream);
lancet_status lancet_set_dw_fillers(lancet_ctx* ctx, int32_t n, lancet_ctx* const* others,
                                    const int32_t* which, const int32_t* a2a_index);
lancet_status lancet_dw_schedule(int32_t n_instr, const int32_t* kind, const double* cost,
                                 int32_t n_edges, const int32_t* edges, int32_t* assign);
lancet_status lancet_stack_dw_plan(int32_t L, int32_t n_chunks, const double* t_a2a,
                                   const double* t_dw, int32_t* host_layer, int32_t* host_a2a);

/* Chunk-count tuner (host only, no device): Lancet's partition-count
 * search reduced to one MoE layer.  The DP over partition ranges has a
 * single range here, so it is a scan over n = 1..max_chunks; each n is scored by the pipeline
 * scheduler of L488-L499 (stages of every chunk on a computation and a communication lane in
 * their scheduled order; an op starts at the later of its dependencies' end and its lane's
 * previous op; step = end of the last op), run on the schedule lancet.cu enqueues
 * (schedule 0: per-chunk launches of the copy-engine / NCCL paths; 1: the push pipeline).
 * Op costs come from a caching profiler (L322-L323): prof_us[i][op] = the op's duration per
 * chunk (per step for GATE, COUNTS, K7) measured with prof_n[i] chunks (n_prof >= 2, e.g. the
 * timeline of one step at n = 1, 2, 4).  Communication follows the cost model of L325-L328:
 * (bytes, us) points at the profiled message sizes bytes_full / prof_n[i], linearly
 * interpolated, and an n-partitioned exchange costs the model at bytes_full / n (the C/n
 * approximation); computation is interpolated linearly in 1/n.  bytes_full: bytes of one data
 * exchange at n = 1.  Outputs: pred_us[n-1] (step time), pred_exposed_us[n-1] (exposed
 * communication; may be NULL), *best_n.  LANCET_ERR_ARG on bad sizes. */
enum {
    LANCET_OP_GATE = 0,      /* once: routing (gate, slot scan; + permute on the pull / NCCL paths) */
    LANCET_OP_COUNTS,        /* once, comm: the size exchange                     */
    LANCET_OP_DISPATCH,      /* comm: dispatch exchange of a chunk (push: fused permute)   */
    LANCET_OP_FC1, LANCET_OP_FC2,
    LANCET_OP_COMBINE,       /* comm: combine exchange of a chunk (push: fused with K4)    */
    LANCET_OP_GATHER,        /* K4 (pull / NCCL)                                           */
    LANCET_OP_K5,            /* combine backward (pull / NCCL)                             */
    LANCET_OP_BWD_DISPATCH,  /* comm: dO rows to the experts (push: fused with K5)         */
    LANCET_OP_DFC2, LANCET_OP_DFC1,
    LANCET_OP_DW,            /* dW2 + dW1 (per chunk; push: merged, profiled as total / n) */
    LANCET_OP_BWD_COMBINE,   /* comm: dX rows back (push: fused with K6)                   */
    LANCET_OP_K6,            /* dispatch backward + gate term (pull / NCCL)                */
    LANCET_OP_K7,            /* once: dWg                                                  */
    LANCET_OP_N
};
typedef struct {
    int32_t schedule;
    int32_t n_prof;
    const int32_t* prof_n;   /* [n_prof]               */
    const double* prof_us;   /* [n_prof][LANCET_OP_N]  */
    double bytes_full;
    int32_t max_chunks;      /* 1..64                  */
} lancet_tune_input;
lancet_status lancet_tune_chunks(const lancet_tune_input* in, double* pred_us, double* pred_exposed_us,
                                 int32_t* best_n);

/* Routing sizes of the last forward (host arrays; synchronises with the forward):
 *   send_counts [E][n_chunks]         rows this rank admitted per expert per chunk
 *   recv_counts [G][E_l][n_chunks]    rows this rank's experts receive per source rank
 *   capacity    C of the last forward  (out or NULL) */
lancet_status lancet_get_counts(lancet_ctx* ctx, int32_t* send_counts, int32_t* recv_counts,
                                int32_t* capacity);

/* Start accumulating the timeline (LANCET_FLAG_TIMELINE) of every following forward and
 * backward until the next call; times are relative to an event recorded on `stream` now.
 * Without it, each forward starts a fresh timeline. */
lancet_status lancet_timeline_begin(lancet_ctx* ctx, lancet_stream_t stream);

/* Timeline of the last forward+backward, or of everything since lancet_timeline_begin
 * (LANCET_FLAG_TIMELINE); synchronises the device. */
lancet_status lancet_last_timeline(lancet_ctx* ctx, lancet_op_record* out, int32_t cap,
                                   int32_t* n_out);

/* Copy an internal buffer of the last forward to host (tests and diagnostics; synchronises).
 * which: 0 = gate logits [T][E] fp32 (R1 chain). */
lancet_status lancet_debug_copy(lancet_ctx* ctx, int32_t which, void* host_dst, size_t bytes);

/* Host-side plan of the expert-parallel exchange (no device; the scheduler posts every NCCL
 * send/recv from exactly this layout).  Inputs (host):
 *   send_counts [E][n]        rows this rank admitted per expert (E = G*E_l) per chunk
 *   recv_counts [G][E_l][n]   rows this rank's experts receive per source rank, local expert,
 *                             chunk (the result of the size all-to-all)
 * Outputs (host, caller-allocated):
 *   send_off [E], S [E][n+1]  chunk c of expert e is packed send rows
 *                             [send_off[e] + S[e][c], send_off[e] + S[e][c+1])
 *   grp_rows [n][E_l], grp_off [n][E_l]   rows and first (128-aligned) row of each
 *                             (chunk, local expert) GEMM group in the receive buffer; the
 *                             buffer holds the groups expert-major (e_l, c)
 *   src_off [G][E_l][n]       row offset of each source's rows inside its group (R12)
 *   total_rows                receive-buffer rows
 * Errors: LANCET_ERR_ARG for null pointers, non-positive sizes or negative counts. */
lancet_status lancet_plan_exchange(int32_t G, int32_t E_l, int32_t n, const int32_t* send_counts,
                                   const int32_t* recv_counts, int32_t* send_off, int32_t* S,
                                   int32_t* grp_rows, int32_t* grp_off, int32_t* src_off,
                                   int32_t* total_rows);

/* Bytes of device workspace the context owns. */
lancet_status lancet_workspace_bytes(const lancet_ctx* ctx, size_t* bytes);

/* NCCL transport (lancet_create with world > 1 or LANCET_FLAG_FORCE_EP): the context's device
 * buffers come from ncclMemAlloc and are registered with the communicator (ncclCommRegister),
 * so the grouped send/recv of the exchanges can move rows between registered buffers directly
 * (NCCL user-buffer registration) instead of staging them through NCCL's own buffers.  *count =
 * buffers currently registered (0 for the other transports, or where NCCL declined -- the
 * exchanges then run unregistered).  Environment LANCET_NCCL_REGISTER=0 at creation: plain
 * cudaMalloc buffers, nothing registered (the A/B). */
lancet_status lancet_nccl_registered(const lancet_ctx* ctx, int32_t* count);

/* Number of this library's kernel launches enqueued by the last forward / backward. */
lancet_status lancet_launch_counts(const lancet_ctx* ctx, int32_t* fwd, int32_t* bwd);

#ifdef __cplusplus
}
#endif

#endif /* LANCET_MOE_H_ */
