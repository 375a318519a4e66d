// peer.h -- copy-engine peer transport (peer.cu): CUDA IPC mappings + stream memory-op flags.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "kernels.h"

struct lancet_ctx;

namespace lancet {

// one pull: `bytes` from offset `src_off` of rank `peer`'s source buffer of the exchange's kind
// into the local pointer `dst`
struct PeerCopy {
    int peer;
    size_t src_off;
    void* dst;
    size_t bytes;
};

int peer_init(lancet_ctx* c, std::string& err);
int peer_flag_words(int world, int n_max);          // after the workspace is allocated
size_t peer_blob_bytes();                                 // per rank
int peer_export(lancet_ctx* c, void* blob, std::string& err);
int peer_import(lancet_ctx* c, const void* blobs, std::string& err);   // world blobs, rank order
void peer_destroy(lancet_ctx* c);
int peer_signal(lancet_ctx* c, int consumed, int kind, int chunk, cudaStream_t s);
int peer_wait_consumed(lancet_ctx* c, cudaStream_t s, bool push = false, bool prev_backward = true);
int peer_wait_all(lancet_ctx* c, int kind, int chunk, cudaStream_t s);
int peer_pull(lancet_ctx* c, int kind, int chunk, const std::vector<PeerCopy>& copies, bool last,
              cudaStream_t s, std::string& err);
int peer_counts(lancet_ctx* c, const int* d_send, int n, cudaStream_t s, std::string& err);
// this rank's flags all set to a value every wait accepts, and the error word set: every
// stream-memop and kernel wait on this rank returns (lancet_peer_abort)
int peer_poison(lancet_ctx* c, uint32_t code);
int peer_quiesce(lancet_ctx* c);   // 0: peers done with this rank's buffers; 1: timed out

// ---- device-side protocol (push mode, LANCET_FLAG_PEER_PUSH) ------------------------------
// Flags carry the step number read from the device counter (d_seq), waits are single-warp
// kernels that spin with ld.acquire.sys and give up after timeout_ns (recording the failed
// flag in the error word, which poisons the context at its next call).  No value is baked
// into the host's enqueue, so a step can be captured in a CUDA graph and replayed.
enum WaitTarget { TGT_STEP = 0, TGT_PREV = 1, TGT_LAST_BWD = 2 };
int dev_seq_bump(lancet_ctx* c, cudaStream_t s);
// this rank's flag (consumed?, kind, chunk) := step in every peer's array; mark_bwd also
// records the step as "last backward" (d_seq[1])
int dev_signal(lancet_ctx* c, int consumed, int kind, int chunk, cudaStream_t s, bool mark_bwd = false);
// wait until every rank's flag (consumed?, kind, chunk) in this rank's array reaches the target
int dev_wait(lancet_ctx* c, int consumed, int kind, int chunk, int target, cudaStream_t s);
// count matrix all-gather ([G][E][n], this rank's row written into every peer's) + wait
int dev_counts(lancet_ctx* c, const int* d_send, int n, cudaStream_t s);
// expert-side group table (c->grp_dev, [n][E_l] rows | offsets) and the push row bases
// [n][E] of this rank, from the gathered matrix
int dev_plan(lancet_ctx* c, int n, cudaStream_t s);
// block mode (every chunk gated on its own): the size exchange of chunk ch (column ch of the
// [E][n] counts) + wait, and the plan of chunk ch in the static-region layout (peer.cu)
int dev_counts_chunk(lancet_ctx* c, const int* d_counts, int n, int ch, cudaStream_t s);
int dev_plan_chunk(lancet_ctx* c, int n, int ch, int region, cudaStream_t s);
uint32_t peer_error(const lancet_ctx* c);      // 0 or the error word
// ChunkSync of a GEMM over all chunks: its TMA producer waits for kind `wait_kind` per chunk
ChunkSync chunk_sync(lancet_ctx* c, int wait_kind);
std::string peer_error_text(uint32_t code);

}  // namespace lancet
