// Multi-GPU transport for global-qubit swaps and readout reductions.
// NCCL is loaded with dlopen the first time a sharded state is created, so single-GPU
// use of the library has no NCCL dependency. The library creates its own communicator
// from the 128-byte ncclUniqueId the caller broadcast (e.g. with torch.distributed).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace hhlsv {

struct Comm {
    void *comm = nullptr;   // ncclComm_t
    int world = 1, rank = 0;
};

bool nccl_available(const char **why);
int nccl_unique_id(unsigned char out[128]);                               // 0 on success
int nccl_init(Comm &c, int world, int rank, const unsigned char id[128]);  // 0 on success
void nccl_destroy(Comm &c);
// Grouped pairwise exchange: send `count` doubles from sendbuf to peer, receive `count` into recvbuf.
int nccl_sendrecv(Comm &c, const double *sendbuf, double *recvbuf, size_t count, int peer, cudaStream_t s);
// Grouped all-to-all over explicit peers: send `count` doubles from sendbufs[i] to peers[i] and
// receive `count` from the same peer into recvbufs[i] (one ncclGroupStart/End).
int nccl_alltoall_pairs(Comm &c, const double *const *sendbufs, double *const *recvbufs, const int *peers, int npeers,
                        size_t count, cudaStream_t s);
// Wait for the stream's NCCL work with failure detection: polls ncclCommGetAsyncError and aborts the
// communicator on an asynchronous error or after timeout_s (0 on success).
int nccl_wait(Comm &c, cudaStream_t s, double timeout_s);
// In-place sum all-reduce of `count` doubles.
int nccl_allreduce_sum(Comm &c, double *buf, size_t count, cudaStream_t s);
const char *nccl_last_error();

}  // namespace hhlsv
