// Collectives for angle sharding.  Two transports behind one interface:
//  * NCCL, loaded with dlopen("libnccl.so.2") so the library has no link-time NCCL
//    dependency and shares whatever NCCL the process already loaded (e.g. torch's);
//  * caller callbacks (ctk_comm_callbacks), e.g. torch.distributed from Python.
// Scalars are all-gathered and summed in rank order, so every rank computes bitwise the
// same sum independent of the collective algorithm.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctk_internal.h"

namespace ctkb {
namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.CommDestroy;
        if (!api.ok) api.err = "libnccl.so.2 lacks required symbols";
    });
    if (!api.ok) fail(CTK_E_UNSUPPORTED, api.err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(CTK_E_CUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

struct NcclState {
    ncclComm_t comm = nullptr;
    bool owned = true;  // false: adopted from the caller (ctk_comm_adopt_nccl), not destroyed here
    cudaStream_t stream = nullptr;
    double* d_scalars = nullptr;  // [nranks] gather target + [1] send
    double* h_scalars = nullptr;
};

int nccl_allreduce_cb(void* buf, size_t count, int dtype, void* stream, void* user) {
    auto* st = static_cast<NcclState*>(user);
    nccl_check(nccl().AllReduce(buf, buf, count, dtype == 1 ? ncclFloat64 : ncclFloat32, ncclSum, st->comm,
                                static_cast<cudaStream_t>(stream)),
               "ncclAllReduce");
    return 0;
}

}  // namespace

void comm_allreduce(Comm* c, void* d_buf, size_t count, int dtype, cudaStream_t s) {
    if (!c || c->cb.nranks <= 1) return;
    if (!c->cb.allreduce_sum) fail(CTK_E_PARAMETER, "communicator lacks allreduce_sum");
    if (c->cb.allreduce_sum(d_buf, count, dtype, s, c->cb.user) != 0) fail(CTK_E_CUDA, "allreduce_sum callback failed");
}

namespace {
// every rank's value, in rank order
std::vector<double> comm_gather_scalar(Comm* c, double v) {
    std::vector<double> all(size_t(c->cb.nranks), 0.0);
    if (c->nccl_comm) {
        auto* st = static_cast<NcclState*>(c->nccl_comm);
        CTK_CUDA(cudaMemcpyAsync(st->d_scalars, &v, sizeof(double), cudaMemcpyHostToDevice, st->stream));
        nccl_check(nccl().AllGather(st->d_scalars, st->d_scalars + 1, 1, ncclFloat64, st->comm, st->stream),
                   "ncclAllGather");
        CTK_CUDA(cudaMemcpyAsync(all.data(), st->d_scalars + 1, sizeof(double) * all.size(), cudaMemcpyDeviceToHost,
                                 st->stream));
        CTK_CUDA(cudaStreamSynchronize(st->stream));
    } else {
        if (!c->cb.allgather_f64) fail(CTK_E_PARAMETER, "communicator lacks allgather_f64");
        if (c->cb.allgather_f64(v, all.data(), c->cb.user) != 0) fail(CTK_E_CUDA, "allgather_f64 callback failed");
    }
    return all;
}
}  // namespace

// Point-to-point exchange of the band-sharded range (bands.cpp): NCCL grouped Send/Recv on
// the library's stream, or the caller's exchange callback.
void comm_exchange(Comm* c, const std::vector<ctk_p2p_op>& ops, int dtype, cudaStream_t s) {
    if (!c || c->cb.nranks <= 1 || ops.empty()) return;
    if (c->nccl_comm) {
        auto& api = nccl();
        if (!api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd)
            fail(CTK_E_UNSUPPORTED, "libnccl.so.2 lacks ncclSend/ncclRecv");
        auto* st = static_cast<NcclState*>(c->nccl_comm);
        const ncclDataType_t dt = dtype == 1 ? ncclFloat64 : ncclFloat32;
        nccl_check(api.GroupStart(), "ncclGroupStart");
        for (const ctk_p2p_op& o : ops) {
            if (o.is_send) nccl_check(api.Send(o.d_buf, o.count, dt, o.peer, st->comm, s), "ncclSend");
            else nccl_check(api.Recv(o.d_buf, o.count, dt, o.peer, st->comm, s), "ncclRecv");
        }
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
        return;
    }
    if (!c->cb.exchange) fail(CTK_E_PARAMETER, "communicator lacks the exchange callback (band-sharded range)");
    if (c->cb.exchange(ops.data(), int(ops.size()), dtype, s, c->cb.user) != 0) fail(CTK_E_CUDA, "exchange callback failed");
}

std::vector<double> comm_allgather_scalar(Comm* c, double v) {
    if (!c || c->cb.nranks <= 1) return {v};
    return comm_gather_scalar(c, v);
}

double comm_sum_scalar(Comm* c, double v) {
    if (!c || c->cb.nranks <= 1) return v;
    double s = 0.0;
    for (double x : comm_gather_scalar(c, v)) s += x;  // rank order
    return s;
}

void comm_sum_vector(Comm* c, double* d_v, int m, cudaStream_t s) {
    if (!c || c->cb.nranks <= 1 || m <= 0) return;
    const size_t R = size_t(c->cb.nranks), M = size_t(m);
    c->gather.ensure(sizeof(double) * R * M);
    double* gb = c->gather.as<double>();
    if (c->nccl_comm) {
        auto* st = static_cast<NcclState*>(c->nccl_comm);
        nccl_check(nccl().AllGather(d_v, gb, M, ncclFloat64, st->comm, s), "ncclAllGather");
    } else {
        // callback transport: a sum-allreduce of a zeroed [nranks][m] buffer in which each
        // rank fills its own row -- one nonzero term per entry, so the gather is exact
        CTK_CUDA(cudaMemsetAsync(gb, 0, sizeof(double) * R * M, s));
        CTK_CUDA(cudaMemcpyAsync(gb + size_t(c->cb.rank) * M, d_v, sizeof(double) * M, cudaMemcpyDeviceToDevice, s));
        comm_allreduce(c, gb, R * M, 1, s);
    }
    rank_sum(gb, int(R), m, d_v, s);
}

double comm_max_scalar(Comm* c, double v) {
    if (!c || c->cb.nranks <= 1) return v;
    double m = v;
    for (double x : comm_gather_scalar(c, v)) m = std::max(m, x);
    return m;
}

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, 128);
}

Comm* comm_create_nccl(const void* id128, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(CTK_E_PARAMETER, "invalid rank / nranks");
    auto* st = new NcclState();
    try {
        ncclUniqueId id;
        std::memcpy(&id, id128, 128);
        nccl_check(nccl().CommInitRank(&st->comm, nranks, id, rank), "ncclCommInitRank");
        CTK_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
        CTK_CUDA(cudaMalloc(&st->d_scalars, sizeof(double) * (size_t(nranks) + 1)));
    } catch (...) {
        delete st;
        throw;
    }
    auto* c = new Comm();
    c->cb.rank = rank;
    c->cb.nranks = nranks;
    c->cb.allreduce_sum = nccl_allreduce_cb;
    c->cb.allgather_f64 = nullptr;
    c->cb.user = st;
    c->nccl_comm = st;
    return c;
}

// Adopt a communicator the caller already initialised (e.g. torch.distributed's NCCL
// process group); the caller keeps ownership and must outlive the ctk_comm.
Comm* comm_adopt_nccl(void* nccl_comm, int nranks, int rank) {
    if (!nccl_comm) fail(CTK_E_PARAMETER, "null ncclComm_t");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(CTK_E_PARAMETER, "invalid rank / nranks");
    (void)nccl();  // the NCCL entry points must resolve in this process
    auto* st = new NcclState();
    st->comm = static_cast<ncclComm_t>(nccl_comm);
    st->owned = false;
    try {
        CTK_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
        CTK_CUDA(cudaMalloc(&st->d_scalars, sizeof(double) * (size_t(nranks) + 1)));
    } catch (...) {
        if (st->stream) cudaStreamDestroy(st->stream);
        delete st;
        throw;
    }
    auto* c = new Comm();
    c->cb.rank = rank;
    c->cb.nranks = nranks;
    c->cb.allreduce_sum = nccl_allreduce_cb;
    c->cb.allgather_f64 = nullptr;
    c->cb.user = st;
    c->nccl_comm = st;
    return c;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->nccl_comm) {
        auto* st = static_cast<NcclState*>(c->nccl_comm);
        if (st->comm && st->owned) nccl().CommDestroy(st->comm);
        if (st->d_scalars) cudaFree(st->d_scalars);
        if (st->stream) cudaStreamDestroy(st->stream);
        delete st;
    }
    delete c;
}

}  // namespace ctkb
