// peer.h -- copy-engine peer transport (peer.cu): CUDA IPC mappings + stream memory-op flags.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

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

int peer_init(lancet_ctx* c, std::string& err);          // after the workspace is allocated
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

}  // namespace lancet
