// TEST-ONLY in-process transport with NCCL's interface, for testing the
// multi-GPU code path of this library on ONE GPU (HMG_TRANSPORT=local).  It is
// NOT part of the product library: build.py compiles it into its own
// libhmg_localtx.so, which libhmg.so dlopens only when HMG_TRANSPORT=local
// (tests/test_dist_local.py).
//
// Every rank is a host thread of the same process, all on the same device,
// each enqueuing its work on its own stream.  The collectives the library uses
// (grouped ncclSend/ncclRecv for the halo exchange, ncclAllReduce of the CG
// dots, ncclAllGather of the coarse gather) are implemented with host-side
// rendezvous (mutex + condition variable) and device-side copies ordered by
// CUDA events: no kernel ever waits for another rank (the B200 profiling guide
// forbids kernels that spin on each other on one GPU); a rank's stream only
// waits on events the other ranks have recorded.  Sums run in rank order, so
// every rank gets the same bits (as NCCL's deterministic ring would not
// guarantee -- the tests compare the distributed V-cycle bitwise against the
// 1-GPU one, and the PCG iteration count).
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "nccl_dyn.h"

namespace hmg {
namespace {

__global__ void k_sum_ranks(const double* __restrict__ stage, double* __restrict__ out, size_t count, int nranks) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    double s = stage[i];
    for (int q = 1; q < nranks; ++q) s = s + stage[(size_t)q * count + i];
    out[i] = s;
}

struct Msg {
    const void* ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;   // recorded on the sender's stream at send time
    cudaEvent_t done = nullptr;    // recorded on the receiver's stream after its copy
    bool copied = false;
};

struct Group {
    int nranks = 0;
    std::mutex m;
    std::condition_variable cv;
    std::map<std::tuple<int, int, uint64_t>, std::shared_ptr<Msg>> box;   // (src, dst, seq)
    std::vector<uint64_t> sseq, rseq;                                       // [src * nranks + dst]
    // collectives
    uint64_t bar_gen = 0;
    int bar_count = 0;
    std::vector<const void*> cptr;
    std::vector<cudaEvent_t> cev, ccp;
    void barrier() {
        std::unique_lock<std::mutex> l(m);
        const uint64_t g = bar_gen;
        if (++bar_count == nranks) {
            bar_count = 0;
            ++bar_gen;
            cv.notify_all();
        } else {
            cv.wait(l, [&] { return bar_gen != g; });
        }
    }
};

struct Comm {
    Group* g = nullptr;
    int rank = 0;
    cudaEvent_t ready = nullptr, cp = nullptr;
    double* stage = nullptr;
    size_t stage_count = 0;
};

std::mutex g_reg_m;
std::map<std::string, Group*> g_registry;

struct PendingOp {
    bool send;
    const void* sbuf;
    void* rbuf;
    size_t bytes;
    int peer;
    Comm* comm;
    cudaStream_t stream;
};
thread_local std::vector<PendingOp> t_pending;
thread_local int t_group_depth = 0;

cudaEvent_t new_event() {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

int run_p2p(std::vector<PendingOp>& ops) {
    std::vector<std::shared_ptr<Msg>> sent;
    // 1. post every send (data ready once the sender's stream reaches this point)
    for (auto& op : ops) {
        if (!op.send) continue;
        Group* G = op.comm->g;
        auto msg = std::make_shared<Msg>();
        msg->ptr = op.sbuf;
        msg->bytes = op.bytes;
        msg->ready = new_event();
        msg->done = new_event();
        cudaEventRecord(msg->ready, op.stream);
        {
            std::lock_guard<std::mutex> l(G->m);
            const int src = op.comm->rank, dst = op.peer;
            G->box[{src, dst, G->sseq[src * G->nranks + dst]++}] = msg;
        }
        G->cv.notify_all();
        sent.push_back(msg);
    }
    // 2. serve every receive: wait for the matching send, copy after its event
    for (auto& op : ops) {
        if (op.send) continue;
        Group* G = op.comm->g;
        const int src = op.peer, dst = op.comm->rank;
        std::shared_ptr<Msg> msg;
        {
            std::unique_lock<std::mutex> l(G->m);
            const auto key = std::make_tuple(src, dst, G->rseq[src * G->nranks + dst]++);
            G->cv.wait(l, [&] { return G->box.count(key) != 0; });
            msg = G->box[key];
            G->box.erase(key);
        }
        if (msg->bytes != op.bytes) return 5;   // mismatched send/recv sizes
        cudaStreamWaitEvent(op.stream, msg->ready, 0);
        cudaMemcpyAsync(op.rbuf, msg->ptr, op.bytes, cudaMemcpyDeviceToDevice, op.stream);
        cudaEventRecord(msg->done, op.stream);
        {
            std::lock_guard<std::mutex> l(G->m);
            msg->copied = true;
        }
        G->cv.notify_all();
    }
    // 3. the sender's later work must not overwrite a buffer before it was copied
    size_t i = 0;
    for (auto& op : ops) {
        if (!op.send) continue;
        Group* G = op.comm->g;
        auto& msg = sent[i++];
        {
            std::unique_lock<std::mutex> l(G->m);
            G->cv.wait(l, [&] { return msg->copied; });
        }
        cudaStreamWaitEvent(op.stream, msg->done, 0);
        cudaEventDestroy(msg->ready);   // destruction is deferred until pending work completes
        cudaEventDestroy(msg->done);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int l_get_unique_id(NcclUniqueId* id) {
    std::random_device rd;
    std::memset(id->internal, 0, sizeof(id->internal));
    const std::string tag = "hmg-local-" + std::to_string(rd()) + "-" + std::to_string(rd());
    std::memcpy(id->internal, tag.c_str(), tag.size());
    return 0;
}

int l_comm_init_rank(ncclComm_t* comm, int nranks, NcclUniqueId id, int rank) {
    const std::string key(id.internal, strnlen(id.internal, sizeof(id.internal)));
    Group* G = nullptr;
    {
        std::lock_guard<std::mutex> l(g_reg_m);
        auto it = g_registry.find(key);
        if (it == g_registry.end()) {
            G = new Group();
            G->nranks = nranks;
            G->sseq.assign((size_t)nranks * nranks, 0);
            G->rseq.assign((size_t)nranks * nranks, 0);
            G->cptr.assign(nranks, nullptr);
            G->cev.assign(nranks, nullptr);
            G->ccp.assign(nranks, nullptr);
            g_registry[key] = G;
        } else {
            G = it->second;
        }
    }
    if (G->nranks != nranks || rank < 0 || rank >= nranks) return 4;
    Comm* C = new Comm();
    C->g = G;
    C->rank = rank;
    C->ready = new_event();
    C->cp = new_event();
    *comm = reinterpret_cast<ncclComm_t>(C);
    return 0;
}

int l_comm_destroy(ncclComm_t comm) {
    Comm* C = reinterpret_cast<Comm*>(comm);
    if (!C) return 0;
    cudaEventDestroy(C->ready);
    cudaEventDestroy(C->cp);
    if (C->stage) cudaFree(C->stage);
    delete C;   // the group stays registered (other ranks may still use it)
    return 0;
}

// Gather all ranks' buffers into `dst` (rank q's `count` doubles at dst + q count)
// on this rank's stream, then make the stream wait until every rank has copied
// from this rank's buffer.
int gather_all(Comm* C, const void* src, double* dst, size_t count, cudaStream_t s) {
    Group* G = C->g;
    cudaEventRecord(C->ready, s);
    G->cptr[C->rank] = src;
    G->cev[C->rank] = C->ready;
    G->barrier();
    for (int q = 0; q < G->nranks; ++q) {
        cudaStreamWaitEvent(s, G->cev[q], 0);
        cudaMemcpyAsync(dst + (size_t)q * count, G->cptr[q], count * sizeof(double), cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(C->cp, s);
    G->ccp[C->rank] = C->cp;
    G->barrier();
    for (int q = 0; q < G->nranks; ++q) cudaStreamWaitEvent(s, G->ccp[q], 0);
    G->barrier();   // slots may be reused by the next collective
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int l_all_reduce(const void* send, void* recv, size_t count, int dtype, int op, ncclComm_t comm, cudaStream_t s) {
    if (dtype != kNcclFloat64 || op != kNcclSum) return 5;
    Comm* C = reinterpret_cast<Comm*>(comm);
    const size_t need = count * (size_t)C->g->nranks;
    if (C->stage_count < need) {
        if (C->stage) cudaFree(C->stage);
        if (cudaMalloc(&C->stage, need * sizeof(double)) != cudaSuccess) return 1;
        C->stage_count = need;
    }
    const int r = gather_all(C, send, C->stage, count, s);
    if (r) return r;
    k_sum_ranks<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(C->stage, static_cast<double*>(recv), count,
                                                               C->g->nranks);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int l_all_gather(const void* send, void* recv, size_t count, int dtype, ncclComm_t comm, cudaStream_t s) {
    if (dtype != kNcclFloat64) return 5;
    return gather_all(reinterpret_cast<Comm*>(comm), send, static_cast<double*>(recv), count, s);
}

int flush_if_ungrouped() {
    if (t_group_depth > 0) return 0;
    std::vector<PendingOp> ops;
    ops.swap(t_pending);
    return run_p2p(ops);
}

int l_send(const void* buf, size_t count, int dtype, int peer, ncclComm_t comm, cudaStream_t s) {
    if (dtype != kNcclFloat64) return 5;
    t_pending.push_back({true, buf, nullptr, count * sizeof(double), peer, reinterpret_cast<Comm*>(comm), s});
    return flush_if_ungrouped();
}

int l_recv(void* buf, size_t count, int dtype, int peer, ncclComm_t comm, cudaStream_t s) {
    if (dtype != kNcclFloat64) return 5;
    t_pending.push_back({false, nullptr, buf, count * sizeof(double), peer, reinterpret_cast<Comm*>(comm), s});
    return flush_if_ungrouped();
}

int l_group_start() {
    ++t_group_depth;
    return 0;
}

int l_group_end() {
    if (--t_group_depth > 0) return 0;
    std::vector<PendingOp> ops;
    ops.swap(t_pending);
    return run_p2p(ops);
}

const char* l_error_string(int r) {
    switch (r) {
        case 0: return "success";
        case 4: return "local transport: inconsistent communicator";
        case 5: return "local transport: unsupported type/op or mismatched send/recv";
        default: return "local transport: CUDA error";
    }
}

}  // namespace

}  // namespace hmg

extern "C" const void* hmg_local_transport_table() {
    using namespace hmg;
    static Nccl t;
    t.GetUniqueId = l_get_unique_id;
    t.CommInitRank = l_comm_init_rank;
    t.CommDestroy = l_comm_destroy;
    t.AllReduce = l_all_reduce;
    t.AllGather = l_all_gather;
    t.Send = l_send;
    t.Recv = l_recv;
    t.GroupStart = l_group_start;
    t.GroupEnd = l_group_end;
    t.GetErrorString = l_error_string;
    return &t;
}
