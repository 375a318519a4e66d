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

#include <chrono>
#include <cstdlib>
#include <thread>
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

// blob: kBufs IPC handles, then the exporter's configuration hash (checked by every importer)
struct BlobTail {
    unsigned long long cfg_hash;
    int32_t rank, world;
};

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
    if (cudaMalloc(&pl->d_seq, sizeof(uint32_t) * 2) != cudaSuccess ||
        cudaMalloc(&pl->d_flag_tab, sizeof(uint32_t*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_counts_tab, sizeof(int*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_dxesrc, sizeof(char*) * G) != cudaSuccess ||
        cudaMalloc(&pl->d_plan_scratch, sizeof(int) * 2 * (size_t)E * pl->n_max) != cudaSuccess) {
        err = "cudaMalloc (device protocol state)";
        return 1;
    }
    cudaMemset(pl->d_seq, 0, sizeof(uint32_t) * 2);
    if (cudaHostAlloc(&pl->h_err, sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&pl->d_err, pl->h_err, 0) != cudaSuccess) {
        err = "cudaHostAlloc (mapped error word)";
        return 1;
    }
    *pl->h_err = 0;
    if (const char* t = getenv("LANCET_PEER_TIMEOUT_MS")) {
        const long long ms = atoll(t);
        if (ms > 0) pl->timeout_ns = (unsigned long long)ms * 1000000ull;
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

size_t peer_blob_bytes() { return kBufs * sizeof(cudaIpcMemHandle_t) + sizeof(BlobTail); }

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
    BlobTail tail{pl->cfg_hash, c->rank, c->world};
    memcpy(reinterpret_cast<char*>(blob) + kBufs * sizeof(cudaIpcMemHandle_t), &tail, sizeof(tail));
    return 0;
}

int peer_import(lancet_ctx* c, const void* blobs, std::string& err)
{
    PeerLinks* pl = c->peer;
    const int G = c->world;
    // every rank must run the same layer configuration (and the same push mode): the flag
    // slots, the receive-buffer bounds and the protocol depend on it
    for (int p = 0; p < G; ++p) {
        BlobTail tail;
        memcpy(&tail, reinterpret_cast<const char*>(blobs) + (size_t)p * peer_blob_bytes() +
                          kBufs * sizeof(cudaIpcMemHandle_t), sizeof(tail));
        if (tail.rank != p || tail.world != G) {
            err = "peer blob " + std::to_string(p) + " is rank " + std::to_string(tail.rank) + " of " +
                  std::to_string(tail.world) + " (blobs must be all-gathered in rank order)";
            return 1;
        }
        if (tail.cfg_hash != pl->cfg_hash) {
            err = "layer configuration differs between rank " + std::to_string(c->rank) + " and rank " +
                  std::to_string(p) + " (d_model, d_ffn, n_experts, max_tokens, max_k, max_chunks, dtype, act, "
                  "RENORMALIZE and PEER_PUSH must agree)";
            return 1;
        }
    }
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
        cudaMemcpy(pl->d_outsrc, pl->src[PK_OUT].data(), sizeof(char*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_dxesrc, pl->src[PK_DXE].data(), sizeof(char*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_flag_tab, pl->flags.data(), sizeof(uint32_t*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(pl->d_counts_tab, pl->counts.data(), sizeof(int*) * G, cudaMemcpyHostToDevice) != cudaSuccess) {
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
    for (void* p : {(void*)pl->d_seq, (void*)pl->d_flag_tab, (void*)pl->d_counts_tab, (void*)pl->d_dxesrc,
                    (void*)pl->d_plan_scratch})
        if (p) cudaFree(p);
    if (pl->h_err) cudaFreeHost(pl->h_err);
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

// destroy: wait (host polling, bounded by the timeout) until every peer has signalled that it
// consumed this rank's rows of the last step -- the kinds peers read from this rank: pull
// sources (copy-engine mode) or the expert outputs and dX rows read in place (push mode)
int peer_quiesce(lancet_ctx* c)
{
    PeerLinks* pl = c->peer;
    if (!pl || pl->seq == 0 || peer_error(c)) return 0;
    const int words = peer_flag_words(pl->world, pl->n_max);
    std::vector<uint32_t> f(words);
    const bool had_bwd = c->bwd_seq == pl->seq;
    std::vector<int> kinds;
    if (c->push) {
        if (had_bwd) kinds = {PK_OUT, PK_DXE};   // a forward-only last step: its outputs are
                                                  // released by the next forward, which never comes
    } else {
        kinds = {PK_XS, PK_OUT};
        if (had_bwd) { kinds.push_back(PK_DCOMB); kinds.push_back(PK_DXE); }
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        if (cudaMemcpy(f.data(), pl->my_flags, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
        bool done = true;
        for (int k : kinds)
            for (int r = 0; r < pl->world; ++r)
                if (f[pl->flag_index(1, k, 0, r)] < pl->seq) done = false;
        if (done) return 0;
        const double ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
        if (ns > (double)pl->timeout_ns) return 1;
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

int peer_poison(lancet_ctx* c, uint32_t code)
{
    PeerLinks* pl = c->peer;
    if (!pl) return 0;
    if (pl->h_err && *reinterpret_cast<volatile uint32_t*>(pl->h_err) == 0) *pl->h_err = code;
    // on a stream of its own: the context's streams may be blocked on the very flags
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return 1;
    const int r = cudaMemsetAsync(pl->my_flags, 0xFF, sizeof(uint32_t) * peer_flag_words(pl->world, pl->n_max), st) !=
                  cudaSuccess;
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    return r;
}

// ============================ device-side protocol (push mode) ============================
namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void seq_bump_kernel(uint32_t* seq)
{
    pdl_wait();
    seq[0] += 1;
}

// every write of the preceding kernels (stream order) before the flag: a system-scope fence,
// then the release store of the step number into rank p's array (thread p)
__global__ void signal_kernel(uint32_t* const* tab, int G, size_t idx, const uint32_t* seq, uint32_t* mark)
{
    pdl_wait();
    __threadfence_system();
    const uint32_t v = seq[0];
    for (int p = threadIdx.x; p < G; p += blockDim.x) st_release_sys(tab[p] + idx, v);
    if (mark && threadIdx.x == 0) mark[0] = v;
}

// lane r spins on rank r's flag until it reaches the target (unsigned >=, as the stream
// wait-value GEQ); after timeout_ns it records (code | r) in the error word and returns, and
// every later wait returns at once (the step's results are then undefined; the context is
// poisoned at its next call)
__global__ void wait_kernel(const uint32_t* flags, size_t idx0, int G, const uint32_t* seq, int target,
                            unsigned long long timeout_ns, uint32_t* err, uint32_t code)
{
    pdl_wait();
    const uint32_t want = target == TGT_STEP ? seq[0] : target == TGT_PREV ? seq[0] - 1u : seq[1];
    const unsigned long long t0 = globaltimer();
    for (int r = threadIdx.x; r < G; r += blockDim.x) {
        unsigned ns = 32;
        while (ld_acquire_sys(flags + idx0 + r) < want) {
            if (*reinterpret_cast<volatile uint32_t*>(err) != 0) return;
            if (globaltimer() - t0 > timeout_ns) {
                atomicCAS(err, 0u, code | (uint32_t)r);
                return;
            }
            __nanosleep(ns);
            if (ns < 1024) ns *= 2;
        }
    }
    __syncwarp();
}

// count-matrix all-gather: this rank's row (E*n ints) into row `rank` of every peer's matrix,
// then the PK_COUNTS flag in every peer's array
__global__ void counts_allgather_kernel(const int* __restrict__ row, int len, int* const* mats, int G, int rank,
                                        uint32_t* const* tab, size_t idx, const uint32_t* seq)
{
    pdl_wait();
    for (int p = 0; p < G; ++p)
        for (int i = threadIdx.x; i < len; i += blockDim.x) mats[p][(size_t)rank * len + i] = row[i];
    __threadfence_system();
    __syncthreads();
    const uint32_t v = seq[0];
    for (int p = threadIdx.x; p < G; p += blockDim.x) st_release_sys(tab[p] + idx, v);
}

// The exchange plan of this rank from the count matrix M [G][E][n] (rows rank g admitted to
// expert e in chunk c), the same layout as the host Plan / GlobalPlan in lancet.cu:
//   owner p's receive buffer holds groups (e_l, c) in expert-major order, 128-row aligned,
//   rows of a group ordered by source rank (R12);
//   grp_rows / grp_off [n][E_l]: this rank's groups (chunk-major table);
//   base [n][E]: row of this rank's chunk-c rows for expert e in the owner's buffer, minus
//   S[e][c] (so row = base + slot).
__global__ void plan_kernel(const int* __restrict__ M, int G, int E, int E_l, int n, int me, int* grp_rows,
                            int* grp_off, int* base, int* R, int* OFF, int rows_cap, uint32_t* err, uint32_t code,
                            int* merged)
{
    pdl_wait();
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int q = tid; q < E * n; q += nt) {              // q = (p E_l + e_l) n + c = e n + c
        const int e = q / n, ch = q % n;
        int s = 0;
        for (int src = 0; src < G; ++src) s += M[((size_t)src * E + e) * n + ch];
        R[q] = s;
    }
    __syncthreads();
    for (int p = tid; p < G; p += nt) {
        int run = 0;
        for (int i = 0; i < E_l * n; ++i) {
            const int q = p * E_l * n + i;
            OFF[q] = run;
            run += round_up(R[q], kRowAlign);
        }
        if (run > rows_cap) atomicCAS(err, 0u, code | (uint32_t)p);
    }
    __syncthreads();
    for (int q = tid; q < n * E_l; q += nt) {
        const int ch = q / E_l, el = q % E_l;
        const int i = (me * E_l + el) * n + ch;
        grp_rows[q] = R[i];
        grp_off[q] = OFF[i];
    }
    // merged dW tables [E_l] rows | offsets: expert e_l's rows of every chunk as one K range
    // (its groups are consecutive in the buffer; the pads between them are zero rows)
    for (int el = tid; el < E_l; el += nt) {
        const int i0 = (me * E_l + el) * n, i1 = i0 + n - 1;
        merged[el] = OFF[i1] + R[i1] - OFF[i0];
        merged[E_l + el] = OFF[i0];
    }
    for (int q = tid; q < n * E; q += nt) {
        const int ch = q / E, e = q % E;
        int src_off = 0, S = 0;
        for (int src = 0; src < me; ++src) src_off += M[((size_t)src * E + e) * n + ch];
        for (int c2 = 0; c2 < ch; ++c2) S += M[((size_t)me * E + e) * n + c2];
        base[q] = OFF[e * n + ch] + src_off - S;
    }
}

// Per-chunk size exchange of the block's pre-MoE partition (each chunk is gated separately,
// PAPER.md L255-L257): column `ch` of this rank's count row ([E][n]) into row `rank` of every
// peer's matrix, then the PK_COUNTS flag of chunk ch in every peer's array.
__global__ void counts_col_kernel(const int* __restrict__ counts, int E, int n, int ch, int* const* mats, int G,
                                  int rank, uint32_t* const* tab, size_t idx, const uint32_t* seq)
{
    pdl_wait();
    for (int p = 0; p < G; ++p)
        for (int e = threadIdx.x; e < E; e += blockDim.x)
            mats[p][((size_t)rank * E + e) * n + ch] = counts[e * n + ch];
    __threadfence_system();
    __syncthreads();
    const uint32_t v = seq[0];
    for (int p = threadIdx.x; p < G; p += blockDim.x) st_release_sys(tab[p] + idx, v);
}

// The exchange plan of chunk ch when every chunk is gated on its own (block mode): owner p's
// receive buffer gives local expert e_l a static region of `region` rows starting at
// e_l * region; inside it the groups (e_l, 0), (e_l, 1), ... follow each other 128-row aligned
// (so an expert's rows over all chunks stay one K range for the merged dW GEMM), rows of a
// group ordered by source rank (R12).  Only the columns 0..ch of M are read: chunk ch's plan is
// final before any later chunk is gated.  Writes this rank's group ch (grp_rows / grp_off
// [n][E_l]), its push bases of chunk ch (base[ch][e] = row of its first chunk-ch row in the
// owner's group minus S[e][ch], so row = base + slot) and, at the last chunk, the merged dW table.
__global__ void plan_chunk_kernel(const int* __restrict__ M, int G, int E, int E_l, int n, int me, int ch,
                                  int region, int* grp_rows, int* grp_off, int* base, uint32_t* err, uint32_t code,
                                  int* merged)
{
    pdl_wait();
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int p = e / E_l, el = e % E_l;
        int off = el * region;
        int R = 0;
        for (int c = 0; c <= ch; ++c) {
            R = 0;
            for (int src = 0; src < G; ++src) R += M[((size_t)src * E + e) * n + c];
            if (c < ch) off += round_up(R, kRowAlign);
        }
        if (off + round_up(R, kRowAlign) > (el + 1) * region) atomicCAS(err, 0u, code | (uint32_t)p);
        int src_off = 0, Sme = 0;
        for (int src = 0; src < me; ++src) src_off += M[((size_t)src * E + e) * n + ch];
        for (int c = 0; c < ch; ++c) Sme += M[((size_t)me * E + e) * n + c];
        base[ch * E + e] = off + src_off - Sme;
        if (p == me) {
            grp_rows[ch * E_l + el] = R;
            grp_off[ch * E_l + el] = off;
            if (ch == n - 1) {
                merged[el] = off + R - el * region;
                merged[E_l + el] = el * region;
            }
        }
    }
}

constexpr uint32_t kErrBit = 0x80000000u;
uint32_t wait_code(int consumed, int kind, int chunk)
{
    return kErrBit | ((uint32_t)(consumed & 1) << 30) | ((uint32_t)(kind & 63) << 24) | ((uint32_t)(chunk & 0xFFFF) << 8);
}
constexpr int kPlanKind = 63;

}  // namespace

std::string peer_error_text(uint32_t code)
{
    if (!code) return "";
    const int consumed = (code >> 30) & 1, kind = (code >> 24) & 63, chunk = (code >> 8) & 0xFFFF, r = code & 0xFF;
    if (code == 0xFFFFFFFFu) return "peer transport aborted (lancet_peer_abort)";
    if (kind == kPlanKind)
        return "expert-side receive buffer of rank " + std::to_string(r) + " too small for the step's rows";
    static const char* names[] = {"xs", "out", "dcomb", "dXe", "counts", "push", "xe-free", "push2", "dout-free"};
    return std::string("peer wait timed out: rank ") + std::to_string(r) + " never signalled " +
           (consumed ? "consumed " : "ready ") + (kind < PK_N ? names[kind] : "?") + " of chunk " + std::to_string(chunk);
}

uint32_t peer_error(const lancet_ctx* c)
{
    return (c->peer && c->peer->h_err) ? *reinterpret_cast<volatile uint32_t*>(c->peer->h_err) : 0u;
}

ChunkSync chunk_sync(lancet_ctx* c, int wait_kind)
{
    PeerLinks* pl = c->peer;
    ChunkSync cs;
    cs.gpc = c->E_l;
    cs.ranks = pl->world;
    cs.wait_flags = pl->my_flags + pl->flag_index(0, wait_kind, 0, 0);
    cs.wait_chunk_stride = pl->world;
    cs.seq = pl->d_seq;
    cs.timeout_ns = pl->timeout_ns;
    cs.err = pl->d_err;
    cs.err_code = wait_code(0, wait_kind, 0);
    return cs;
}

int dev_seq_bump(lancet_ctx* c, cudaStream_t s)
{
    launch_k(seq_bump_kernel, 1, 1, 0, s, c->peer->d_seq);
    return cudaGetLastError() != cudaSuccess;
}

int dev_signal(lancet_ctx* c, int consumed, int kind, int chunk, cudaStream_t s, bool mark_bwd)
{
    PeerLinks* pl = c->peer;
    launch_k(signal_kernel, 1, 32, 0, s, pl->d_flag_tab, pl->world, pl->flag_index(consumed, kind, chunk, c->rank),
             (const uint32_t*)pl->d_seq, mark_bwd ? pl->d_seq + 1 : (uint32_t*)nullptr);
    return cudaGetLastError() != cudaSuccess;
}

int dev_wait(lancet_ctx* c, int consumed, int kind, int chunk, int target, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    launch_k(wait_kernel, 1, 32, 0, s, (const uint32_t*)pl->my_flags, pl->flag_index(consumed, kind, chunk, 0),
             pl->world, (const uint32_t*)pl->d_seq, target, pl->timeout_ns, pl->d_err, wait_code(consumed, kind, chunk));
    return cudaGetLastError() != cudaSuccess;
}

int dev_counts(lancet_ctx* c, const int* d_send, int n, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    const int E = c->cfg.n_experts;
    launch_k(counts_allgather_kernel, 1, 256, 0, s, d_send, E * n, pl->d_counts_tab, pl->world, c->rank,
             pl->d_flag_tab, pl->flag_index(0, PK_COUNTS, 0, c->rank), (const uint32_t*)pl->d_seq);
    if (cudaGetLastError() != cudaSuccess) return 1;
    return dev_wait(c, 0, PK_COUNTS, 0, TGT_STEP, s);
}

int dev_plan(lancet_ctx* c, int n, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    const int E = c->cfg.n_experts;
    int* R = pl->d_plan_scratch;
    int* OFF = R + (size_t)E * pl->n_max;
    launch_k(plan_kernel, 1, 256, 0, s, (const int*)pl->my_counts, pl->world, E, c->E_l, n, c->rank, c->grp_dev,
             c->grp_dev + n * c->E_l, pl->d_push_base, R, OFF, pl->rows_cap, pl->d_err,
             wait_code(0, kPlanKind, 0), c->grp_dev + 2 * kMaxChunks * c->E_l);
    return cudaGetLastError() != cudaSuccess;
}

int dev_counts_chunk(lancet_ctx* c, const int* d_counts, int n, int ch, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    const int E = c->cfg.n_experts;
    launch_k(counts_col_kernel, 1, 256, 0, s, d_counts, E, n, ch, pl->d_counts_tab, pl->world, c->rank, pl->d_flag_tab,
             pl->flag_index(0, PK_COUNTS, ch, c->rank), (const uint32_t*)pl->d_seq);
    if (cudaGetLastError() != cudaSuccess) return 1;
    return dev_wait(c, 0, PK_COUNTS, ch, TGT_STEP, s);
}

int dev_plan_chunk(lancet_ctx* c, int n, int ch, int region, cudaStream_t s)
{
    PeerLinks* pl = c->peer;
    const int E = c->cfg.n_experts;
    launch_k(plan_chunk_kernel, 1, 256, 0, s, (const int*)pl->my_counts, pl->world, E, c->E_l, n, c->rank, ch, region,
             c->grp_dev, c->grp_dev + n * c->E_l, pl->d_push_base, pl->d_err, wait_code(0, kPlanKind, ch),
             c->grp_dev + 2 * kMaxChunks * c->E_l);
    return cudaGetLastError() != cudaSuccess;
}

}  // namespace lancet
