// comm.cpp -- NCCL and local (in-process) transports of the irregular all-to-all.
#include "comm.h"

#include <nccl.h>

#include <condition_variable>
#include <mutex>

namespace lancet {

// ---------------------------------------------------------------------------- NCCL -------

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    int* d_scratch = nullptr;
    std::vector<std::pair<void*, void*>> regs;   // (buffer, registration handle)

    ~NcclTransport() override {
        if (comm) {
            for (auto& r : regs) ncclCommDeregister(comm, r.second);
            ncclCommDestroy(comm);
        }
        if (d_scratch) cudaFree(d_scratch);
    }
    bool is_nccl() const override { return true; }
    void abort() override {
        if (comm) { ncclCommAbort(comm); comm = nullptr; }
        regs.clear();
    }
    int register_buffer(void* p, size_t bytes) override {
        if (!comm || !p) return 1;
        void* h = nullptr;
        if (ncclCommRegister(comm, p, bytes, &h) != ncclSuccess || !h) return 1;
        regs.push_back({p, h});
        return 0;
    }
    void deregister_buffer(void* p) override {
        for (size_t i = 0; i < regs.size(); ++i)
            if (regs[i].first == p) {
                if (comm) ncclCommDeregister(comm, regs[i].second);
                regs.erase(regs.begin() + i);
                return;
            }
    }
    int exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s,
                 std::string& err) override {
        ncclResult_t r = ncclGroupStart();
        for (const P2P& p : sends)
            if (r == ncclSuccess && p.bytes)
                r = ncclSend(p.buf, p.bytes, ncclUint8, p.peer, comm, s);
        for (const P2P& p : recvs)
            if (r == ncclSuccess && p.bytes)
                r = ncclRecv(p.buf, p.bytes, ncclUint8, p.peer, comm, s);
        ncclResult_t r2 = ncclGroupEnd();
        if (r == ncclSuccess) r = r2;
        if (r != ncclSuccess) {
            err = std::string("NCCL grouped send/recv failed: ") + ncclGetErrorString(r);
            return 1;
        }
        return 0;
    }
    int check_same(unsigned long long v, cudaStream_t s, std::string& err) override {
        // all-reduce max and min of the value; equal iff every rank passed v
        unsigned long long h[2] = {v, ~v};
        if (!d_scratch && cudaMalloc(&d_scratch, 16) != cudaSuccess) { err = "cudaMalloc"; return 1; }
        cudaMemcpyAsync(d_scratch, h, 16, cudaMemcpyHostToDevice, s);
        ncclResult_t r = ncclAllReduce(d_scratch, d_scratch, 2, ncclUint64, ncclMax, comm, s);
        if (r != ncclSuccess) { err = ncclGetErrorString(r); return 1; }
        unsigned long long o[2];
        cudaMemcpyAsync(o, d_scratch, 16, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) { err = "cudaStreamSynchronize"; return 1; }
        if (o[0] != v || o[1] != ~v) {
            err = "layer configuration differs between ranks";
            return 1;
        }
        return 0;
    }
};

void* nccl_mem_alloc(size_t bytes)
{
    void* p = nullptr;
    if (ncclMemAlloc(&p, bytes) != ncclSuccess) return nullptr;
    return p;
}
void nccl_mem_free(void* p)
{
    if (p) ncclMemFree(p);
}

int nccl_unique_id(void* out, std::string& err)
{
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclResult_t r = ncclGetUniqueId(reinterpret_cast<ncclUniqueId*>(out));
    if (r != ncclSuccess) { err = ncclGetErrorString(r); return 1; }
    return 0;
}

Transport* make_nccl_transport(int world, int rank, const void* id, int max_ctas, std::string& err)
{
    auto* t = new NcclTransport();
    t->world = world;
    t->rank = rank;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 1;
    if (max_ctas > 0) cfg.maxCTAs = max_ctas;
    ncclResult_t r = ncclCommInitRankConfig(&t->comm, world, uid, rank, &cfg);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        t->comm = nullptr;
        delete t;
        return nullptr;
    }
    return t;
}

// ---------------------------------------------------------------------------- local ------
// G ranks driven by G host threads of one process on one device.  An exchange is a
// rendezvous: each rank publishes its send list and an event recorded after the work that
// produced the send buffers; after all ranks arrived, each rank copies what it receives
// (device-to-device, on its own stream, after waiting on the sender's event) and records a
// "done" event; senders then make their stream wait on every peer's "done" (a grouped NCCL
// send/recv likewise completes on the sender's stream only when the peers have received).

struct LocalGroupImpl {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<std::vector<P2P>> posted;
    std::vector<cudaEvent_t> ready, done;
    std::vector<unsigned long long> vals;
    explicit LocalGroupImpl(int w) : world(w), posted(w), ready(w), done(w), vals(w) {
        for (int i = 0; i < w; ++i) {
            cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
        }
    }
    ~LocalGroupImpl() {
        for (int i = 0; i < world; ++i) {
            cudaEventDestroy(ready[i]);
            cudaEventDestroy(done[i]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

LocalGroupImpl* local_group_create(int world) { return new LocalGroupImpl(world); }
void local_group_destroy(LocalGroupImpl* g) { delete g; }

struct LocalTransport : Transport {
    LocalGroupImpl* g;
    explicit LocalTransport(LocalGroupImpl* grp) : g(grp) {}
    int exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, cudaStream_t s,
                 std::string& err) override {
        cudaEventRecord(g->ready[rank], s);
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->posted[rank] = sends;
        }
        g->barrier();                                   // all send lists published
        std::vector<size_t> next(world, 0);             // per-peer match cursor
        std::vector<bool> waited(world, false);
        for (const P2P& r : recvs) {
            if (!r.bytes) continue;
            const std::vector<P2P>& ps = g->posted[r.peer];
            size_t& i = next[r.peer];
            while (i < ps.size() && (ps[i].peer != rank || ps[i].bytes == 0)) ++i;
            if (i >= ps.size() || ps[i].bytes != r.bytes) {
                err = "local transport: unmatched send/recv sizes";
                g->barrier();
                return 1;
            }
            if (!waited[r.peer]) {
                cudaStreamWaitEvent(s, g->ready[r.peer], 0);
                waited[r.peer] = true;
            }
            cudaMemcpyAsync(r.buf, ps[i].buf, r.bytes, cudaMemcpyDeviceToDevice, s);
            ++i;
        }
        cudaEventRecord(g->done[rank], s);
        g->barrier();                                   // all copies enqueued
        for (int p = 0; p < world; ++p)
            if (p != rank) cudaStreamWaitEvent(s, g->done[p], 0);
        g->barrier();                                   // posted lists may be reused
        return cudaGetLastError() == cudaSuccess ? 0 : (err = "local transport CUDA error", 1);
    }
    int check_same(unsigned long long v, cudaStream_t, std::string& err) override {
        g->vals[rank] = v;
        g->barrier();
        bool same = true;
        for (int p = 0; p < world; ++p) same &= g->vals[p] == v;
        g->barrier();
        if (!same) { err = "layer configuration differs between ranks"; return 1; }
        return 0;
    }
};

Transport* make_local_transport(LocalGroupImpl* g, int rank, std::string& err)
{
    if (!g || rank < 0 || rank >= g->world) { err = "bad local group / rank"; return nullptr; }
    auto* t = new LocalTransport(g);
    t->world = g->world;
    t->rank = rank;
    return t;
}

}  // namespace lancet
