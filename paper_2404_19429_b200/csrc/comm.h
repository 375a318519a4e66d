// comm.h -- transports of the irregular all-to-all (PAPER.md L517-L526,
// fig:irregular_implementations): "a first all-to-all is performed to exchange the amount of
// data to be sent and received across devices, followed by a second all-to-all only sending
// and receiving the required amount of data ... implemented via a grouped NCCL
// communication consisting of NCCLSends and NCCLRecvs."
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace lancet {

struct P2P {
    int peer;
    void* buf;
    size_t bytes;
};

struct Transport {
    int world = 1, rank = 0;
    virtual ~Transport() {}
    // One grouped exchange enqueued on `s`: every send to peer p is matched, in order, with a
    // recv posted by p from this rank (NCCL group semantics).  Zero-byte entries may be
    // omitted by both sides.  Returns 0, or nonzero with `err` set (context is poisoned).
    virtual int exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs,
                         cudaStream_t s, std::string& err) = 0;
    // Host-side check that every rank passed the same 64-bit value (config hash).
    virtual int check_same(unsigned long long v, cudaStream_t s, std::string& err) = 0;
    virtual void abort() {}
    virtual bool is_nccl() const { return false; }
    // NCCL user-buffer registration (ncclCommRegister) of a buffer the exchanges use: send /
    // recv over NVLink then move the rows between the registered buffers directly instead of
    // staging them through NCCL's internal buffers.  Returns 0 if registered, nonzero if the
    // transport or the buffer does not support it (the exchange still works unregistered).
    virtual int register_buffer(void* /*p*/, size_t /*bytes*/) { return 1; }
    virtual void deregister_buffer(void* /*p*/) {}
};

// ncclMemAlloc / ncclMemFree (cuMem-backed, the allocation NCCL can register for zero-copy
// point-to-point); nullptr if unavailable
void* nccl_mem_alloc(size_t bytes);
void nccl_mem_free(void* p);

// NCCL (one process per GPU).  `id` is the 128-byte ncclUniqueId.
// max_ctas > 0: the communicator's kernels use at most that many CTAs (ncclConfig_t.maxCTAs)
Transport* make_nccl_transport(int world, int rank, const void* id, int max_ctas, std::string& err);
int nccl_unique_id(void* out, std::string& err);

// In-process simulated ranks on one device.
struct LocalGroupImpl;
LocalGroupImpl* local_group_create(int world);
void local_group_destroy(LocalGroupImpl* g);
Transport* make_local_transport(LocalGroupImpl* g, int rank, std::string& err);

}  // namespace lancet
