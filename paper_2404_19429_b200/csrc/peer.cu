// peer.cu -- copy-engine peer transport of the irregular all-to-all (world > 1, no NCCL).
//
// The all-to-all of the MoE layer moves large contiguous row blocks (a chunk's rows for one
// (source rank, expert) pair are one range on both sides), which is what
// the copy engines do best over NVLink / NVSwitch -- and they leave every SM to the expert
// GEMMs, where an NCCL all-to-all needs SMs of its own.  Pull model: every rank maps its
// peers' pull-source buffers once (CUDA IPC) and copies the rows it needs into its own buffers
// with cudaMemcpyAsync on its comm stream.  Ordering across processes uses 32-bit sequence
// flags in device memory (stream write-value / wait-value operations), one per (kind, chunk,
// rank):
//   ready[kind][chunk][p]    = s  once rank p has produced step s's rows of `kind` / chunk;
//   consumed[kind][chunk][q] = s  once rank q has pulled them (p may then overwrite them).
// The count matrix [G][E][n] (rows rank g admitted to expert e in chunk c) is all-gathered the
// same way: each rank writes its row into every peer's matrix, so every rank can compute every
// peer's send and receive layout (the remote offsets of its pulls).
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "comm.h"
#include "common.cuh"
#include "context.h"
#include "kernels.h"
#include "peer.h"

namespace lancet {

namespace {

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct MemOps {
    WaitValueFn wait = nullptr;
    WriteValueFn write = nullptr;
};

const MemOps& memops()
{
    static MemOps ops;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.wait = reinterpret_cast<WaitValueFn>(p);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            ops.write = reinterpret_cast<WriteValueFn>(p);
    });
    return ops;
}

constexpr int kBufs = 8;   // exported: xs, out-source, dcomb, dXe-source, counts, flags, xe, dout

}  // namespace

int peer_flag_words(int world, int n_max) { return 2 * PK_N * n_max * world; }

int peer_init(lancet_ctx* c, std::string& err)
{
    if (!memops().wait || !memops().write) {
        err = "stream memory operations (cuStreamWaitValue32 / cuStreamWriteValue32) unavailable";
        return 1;
    }
    auto* pl = new PeerLinks();
    c->peer = pl;
    pl->world = c->world;
    pl->n_max = c->cfg.max_chunks;
    const int G = c->world, E = c->cfg.n_experts;
    if (cudaMalloc(&pl->my_counts, sizeof(int) * (size_t)G * E * pl->n_max) != cudaSuccess ||
        cudaMalloc(&pl->my_flags, sizeof(uint32_t) * peer_flag_words(G, pl->n_max)) != cudaSuccess) {
        err = "cudaMalloc (peer flags / counts)";
        return 1;
    }
    cudaMemset(pl->my_counts, 0, sizeof(int) * (size_t)G * E * pl->n_max);
    if (cudaMallocHost(&pl->h_matrix, sizeof(int) * (size_t)G * E * pl->n_max) != cudaSuccess) {
        err = "cudaMallocHost (peer counts)";
        return 1;
    }
    cudaMemset(pl->my_flags, 0, sizeof(uint32_t) * peer_flag_words(G, pl->n_max));
    if (cudaMalloc(&pl->d_xe, sizeof(char*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_dout, sizeof(char*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_outsrc, sizeof(char*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_push_base, sizeof(int) * (size_t)pl->n_max * E) != cudaSuccess) {
        err = "cudaMalloc (push tables)";
        return 1;
    }
    pl->xe.assign(G, nullptr);
    pl->dout.assign(G, nullptr);
    for (int k = 0; k <= PK_DXE; ++k) pl->src[k].assign(G, nullptr);
    pl->counts.assign(G, nullptr);
    pl->flags.assign(G, nullptr);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : (err = "cudaDeviceSynchronize", 1);
}

static void* local_src(lancet_ctx* c, int kind)
{
    const bool ident = c->cfg.act == LANCET_ACT_IDENTITY_EXPERT;
    switch (kind) {
    case PK_XS: return c->xs;
    case PK_OUT: return ident ? c->xe : c->out;
    case PK_DCOMB: return c->dcomb;
    default: return ident ? c->dout : c->dXe;
    }
}

size_t peer_blob_bytes() { return kBufs * sizeof(cudaIpcMemHandle_t); }

int peer_export(lancet_ctx* c, void* blob, std::string& err)
{
    PeerLinks* pl = c->peer;
    void* bufs[kBufs] = {local_src(c, PK_XS), local_src(c, PK_OUT), local_src(c, PK_DCOMB),
                         local_src(c, PK_DXE), pl->my_counts, pl->my_flags, c->xe, c->dout};
    auto* h = reinterpret_cast<cudaIpcMemHandle_t*>(blob);
    for (int i = 0; i < kBufs; ++i)
        if (cudaIpcGetMemHandle(&h[i], bufs[i]) != cudaSuccess) {
            err = "cudaIpcGetMemHandle";
            return 1;
        }
    return 0;
}

int peer_import(lancet_ctx* c, const void* blobs, std::string& err)
{
    PeerLinks* pl = c->peer;
    const int G = c->world;
    for (int p = 0; p < G; ++p) {
        void* m[kBufs];
        if (p == c->rank) {
            for (int k = 0; k <= PK_DXE; ++k) m[k] = local_src(c, k);
            m[4] = pl->my_counts;
            m[5] = pl->my_flags;
            m[6] = c->xe;
            m[7] = c->dout;
        } else {
            const auto* h = reinterpret_cast<const cudaIpcMemHandle_t*>(
                reinterpret_cast<const char*>(blobs) + (size_t)p * peer_blob_bytes());
            for (int i = 0; i < kBufs; ++i) {
                if (cudaIpcOpenMemHandle(&m[i], h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    err = "cudaIpcOpenMemHandle (peer " + std::to_string(p) + ")";
                    return 1;
                }
                pl->opened.push_back(m[i]);
            }
        }
        for (int k = 0; k <= PK_DXE; ++k) pl->src[k][p] = reinterpret_cast<char*>(m[k]);
        pl->counts[p] = reinterpret_cast<int*>(m[4]);
        pl->flags[p] = reinterpret_cast<uint32_t*>(m[5]);
        pl->xe[p] = reinterpret_cast<char*>(m[6]);
        pl->dout[p] = reinterpret_cast<char*>(m[7]);
    }
    if (cudaMemcpy(pl->d_xe, pl->xe.data(), sizeof(char*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_dout, pl->dout.data(), sizeof(char*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_outsrc, pl->src[PK_OUT].data(), sizeof(char*) * G, cudaMemcpyHostToDevice) != cudaSuccess) {
        err = "cudaMemcpy (peer receive-buffer table)";
        return 1;
    }
    return 0;
}

void peer_destroy(lancet_ctx* c)
{
    PeerLinks* pl = c->peer;
    if (!pl) return;
    for (void* p : pl->opened) cudaIpcCloseMemHandle(p);
    if (pl->my_counts) cudaFree(pl->my_counts);
    if (pl->my_flags) cudaFree(pl->my_flags);
    if (pl->d_xe) cudaFree(pl->d_xe);
    if (pl->d_dout) cudaFree(pl->d_dout);
    if (pl->d_outsrc) cudaFree(pl->d_outsrc);
    if (pl->d_push_base) cudaFree(pl->d_push_base);
    if (pl->h_matrix) cudaFreeHost(pl->h_matrix);
    delete pl;
    c->peer = nullptr;
}

// this rank's flag (consumed?, kind, chunk) := seq in every peer's array (self included)
int peer_signal(lancet_ctx* c, int consumed, int kind, int chunk, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    for (int p = 0; p < pl->world; ++p) {
        uint32_t* f = pl->flags[p] + pl->flag_index(consumed, kind, chunk, c->rank);
        if (memops().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(f), pl->seq,
                           CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return 1;
    }
    return 0;
}

// wait until rank r's flag (consumed?, kind, chunk) in this rank's array reaches `value`
int peer_wait(lancet_ctx* c, int consumed, int kind, int chunk, int r, uint32_t value, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    uint32_t* f = pl->my_flags + pl->flag_index(consumed, kind, chunk, r);
    return memops().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(f), value,
                         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS;
}

// before this step overwrites any pull source: every peer has pulled the previous step's rows
// of every kind
int peer_wait_consumed(lancet_ctx* c, cudaStream_t s, bool push, bool prev_backward)
{
    PeerLinks* pl = c->peer;
    if (pl->seq <= 1) return 0;
    for (int kind = 0; kind <= PK_DXE; ++kind) {
        if (push && (kind == PK_XS || kind == PK_DCOMB)) continue;   // pushed, never pulled
        // a forward that was not followed by a backward produced no backward rows to consume
        if (!prev_backward && (kind == PK_DCOMB || kind == PK_DXE)) continue;
        for (int r = 0; r < pl->world; ++r)
            if (peer_wait(c, 1, kind, 0, r, pl->seq - 1, s)) return 1;
    }
    return 0;
}

// push-dispatch: wait until every peer's receive buffer is free for this step, and (after the
// push of chunk `chunk`) until every peer's rows of chunk `chunk` have landed in ours
int peer_wait_all(lancet_ctx* c, int kind, int chunk, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    for (int r = 0; r < pl->world; ++r)
        if (peer_wait(c, 0, kind, chunk, r, pl->seq, s)) return 1;
    return 0;
}

int peer_pull(lancet_ctx* c, int kind, int chunk, const std::vector<PeerCopy>& copies, bool last,
              cudaStream_t s, std::string& err)
{
    PeerLinks* pl = c->peer;
    std::vector<bool> from(pl->world, false);
    for (const PeerCopy& cp : copies) from[cp.peer] = true;
    for (int p = 0; p < pl->world; ++p)
        if (from[p] && peer_wait(c, 0, kind, chunk, p, pl->seq, s)) { err = "cuStreamWaitValue32"; return 1; }
    for (const PeerCopy& cp : copies) {
        if (!cp.bytes) continue;
        if (cudaMemcpyAsync(cp.dst, pl->src[kind][cp.peer] + cp.src_off, cp.bytes, cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess) {
            err = "cudaMemcpyAsync (peer pull)";
            return 1;
        }
    }
    // after the step's last pull of this kind: tell every source its rows may be reused (the
    // pulls are in order on this stream, so this covers all chunks; slot 0)
    if (last && peer_signal(c, 1, kind, 0, s)) { err = "cuStreamWriteValue32"; return 1; }
    return 0;
}

// all-gather of the count matrix: this rank's row [E][n] into every peer's matrix, then ready
int peer_counts(lancet_ctx* c, const int* d_send, int n, cudaStream_t s, std::string& err)
{
    PeerLinks* pl = c->peer;
    const int E = c->cfg.n_experts;
    const size_t row = sizeof(int) * (size_t)E * n;
    for (int p = 0; p < pl->world; ++p)
        if (cudaMemcpyAsync(reinterpret_cast<char*>(pl->counts[p]) + row * c->rank, d_send, row,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
            err = "cudaMemcpyAsync (peer counts)";
            return 1;
        }
    if (peer_signal(c, 0, PK_COUNTS, 0, s)) { err = "cuStreamWriteValue32"; return 1; }
    for (int r = 0; r < pl->world; ++r)
        if (peer_wait(c, 0, PK_COUNTS, 0, r, pl->seq, s)) { err = "cuStreamWaitValue32"; return 1; }
    return 0;
}

}  // namespace lancet
