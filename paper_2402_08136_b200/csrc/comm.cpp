// NCCL (2.28, torch-bundled libnccl.so.2) loaded at run time. See comm.h.
#include "comm.h"

#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "nccl.h"

namespace hhlsv {

namespace {
struct NcclApi {
    void *h = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    decltype(&ncclCommGetAsyncError) asyncError = nullptr;
    decltype(&ncclCommAbort) commAbort = nullptr;
    std::string why;
    bool ok = false;
};

NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *env = getenv("HHLSV_NCCL_LIB");
        const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            if (!nm) continue;
            a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) {
            a.why = std::string("cannot dlopen libnccl.so.2 (set HHLSV_NCCL_LIB): ") + dlerror();
            return;
        }
#define LOAD(field, sym)                                                  \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(a.h, #sym));      \
    if (!a.field) {                                                       \
        a.why = "libnccl lacks " #sym;                                    \
        return;                                                           \
    }
        LOAD(getUniqueId, ncclGetUniqueId)
        LOAD(commInitRank, ncclCommInitRank)
        LOAD(commDestroy, ncclCommDestroy)
        LOAD(send, ncclSend)
        LOAD(recv, ncclRecv)
        LOAD(groupStart, ncclGroupStart)
        LOAD(groupEnd, ncclGroupEnd)
        LOAD(allReduce, ncclAllReduce)
        LOAD(errStr, ncclGetErrorString)
        LOAD(asyncError, ncclCommGetAsyncError)
        LOAD(commAbort, ncclCommAbort)
#undef LOAD
        a.ok = true;
    });
    return a;
}

thread_local std::string g_err;

int check(ncclResult_t r) {
    if (r == ncclSuccess) return 0;
    g_err = api().errStr ? api().errStr(r) : "nccl error";
    return (int)r;
}
}  // namespace

bool nccl_available(const char **why) {
    NcclApi &a = api();
    if (why) *why = a.why.c_str();
    return a.ok;
}

const char *nccl_last_error() { return g_err.c_str(); }

int nccl_unique_id(unsigned char out[128]) {
    if (!api().ok) {
        g_err = api().why;
        return -1;
    }
    ncclUniqueId id;
    int rc = check(api().getUniqueId(&id));
    if (rc == 0) std::memcpy(out, &id, sizeof(id));
    return rc;
}

int nccl_init(Comm &c, int world, int rank, const unsigned char idb[128]) {
    if (!api().ok) {
        g_err = api().why;
        return -1;
    }
    ncclUniqueId id;
    std::memcpy(&id, idb, sizeof(id));
    ncclComm_t comm = nullptr;
    int rc = check(api().commInitRank(&comm, world, id, rank));
    if (rc) return rc;
    c.comm = comm;
    c.world = world;
    c.rank = rank;
    return 0;
}

void nccl_destroy(Comm &c) {
    if (c.comm && api().ok) api().commDestroy((ncclComm_t)c.comm);
    c.comm = nullptr;
}

int nccl_sendrecv(Comm &c, const double *sendbuf, double *recvbuf, size_t count, int peer, cudaStream_t s) {
    NcclApi &a = api();
    int rc = check(a.groupStart());
    if (rc) return rc;
    rc = check(a.send(sendbuf, count, ncclDouble, peer, (ncclComm_t)c.comm, s));
    int rc2 = check(a.recv(recvbuf, count, ncclDouble, peer, (ncclComm_t)c.comm, s));
    int rc3 = check(a.groupEnd());
    return rc ? rc : (rc2 ? rc2 : rc3);
}

int nccl_alltoall_pairs(Comm &c, const double *const *sendbufs, double *const *recvbufs, const int *peers, int npeers,
                        size_t count, cudaStream_t s) {
    NcclApi &a = api();
    int rc = check(a.groupStart());
    if (rc) return rc;
    for (int i = 0; i < npeers && !rc; i++) {
        rc = check(a.send(sendbufs[i], count, ncclDouble, peers[i], (ncclComm_t)c.comm, s));
        if (!rc) rc = check(a.recv(recvbufs[i], count, ncclDouble, peers[i], (ncclComm_t)c.comm, s));
    }
    const int rc2 = check(a.groupEnd());
    return rc ? rc : rc2;
}

int nccl_wait(Comm &c, cudaStream_t s, double timeout_s) {
    // Poll the stream and the communicator's asynchronous error state; abort the communicator when
    // NCCL reports an error or the collective does not finish in time (a lost peer would otherwise
    // hang the caller forever). SURVEY §5 failure detection.
    NcclApi &a = api();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return 0;
        if (q != cudaErrorNotReady) {
            g_err = std::string("CUDA error while waiting for NCCL: ") + cudaGetErrorString(q);
            return -1;
        }
        ncclResult_t ae = ncclSuccess;
        if (c.comm && a.asyncError((ncclComm_t)c.comm, &ae) == ncclSuccess && ae != ncclSuccess &&
            ae != ncclInProgress) {
            g_err = std::string("NCCL asynchronous error: ") + a.errStr(ae);
            a.commAbort((ncclComm_t)c.comm);
            c.comm = nullptr;
            return (int)ae;
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > timeout_s) {
            g_err = "NCCL operation timed out after " + std::to_string(timeout_s) + " s (peer lost?)";
            if (c.comm) a.commAbort((ncclComm_t)c.comm);
            c.comm = nullptr;
            return -2;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

int nccl_allreduce_sum(Comm &c, double *buf, size_t count, cudaStream_t s) {
    return check(api().allReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)c.comm, s));
}

}  // namespace hhlsv
