// comm.hpp -- halo exchange and gradient all-reduce between ranks (internal).
//
// Two backends behind one interface:
//   NCCL      one process per GPU; libnccl.so.2 is opened at run time (the copy PyTorch already
//             loaded), grouped ncclSend/ncclRecv for the neighbour halos, ncclAllReduce (sum,
//             fp32) for the weight gradient and the head's pooled features.
//   loopback  several ranks as host threads of one process on one GPU (tests of the sharded
//             engine on a single B200): device-to-device copies ordered by events + host barriers.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <vector>

namespace lrcnn {

struct XferBuf {
    int peer;
    int send;       // 1 = this rank sends ptr[0, bytes) to peer; 0 = receives into it
    void *ptr;
    size_t bytes;
};

struct Comm;
int comm_rank(const Comm *c);
int comm_world(const Comm *c);
bool comm_graph_safe(const Comm *c);   // may the calls be captured into a CUDA graph
// grouped point-to-point transfers, ordered on `st`; returns 0 on success
int comm_exchange(Comm *c, const std::vector<XferBuf> &xs, cudaStream_t st, const char **err);
// in-place sum over ranks of n floats, ordered on `st`
int comm_allreduce_f32(Comm *c, float *buf, size_t n, cudaStream_t st, const char **err);
// in-place sum over ranks of n doubles (NCCL, loopback; host-staged: an all-gather through the exchange
// callback and a rank-ordered sum on the host)
int comm_allreduce_f64(Comm *c, double *buf, size_t n, cudaStream_t st, const char **err);

}  // namespace lrcnn
