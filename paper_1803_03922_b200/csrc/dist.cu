// dist.cu -- NCCL plumbing for the one-worker-per-process engine (NVLink 5 /
// NVSwitch inside one box).  The reference simulates these collectives in
// memory (comm.py:75-197); here they are real:
//   delegate masks  : ncclAllGather of d/8 bytes, OR-folded by phase_finish
//                     (NCCL has no bitwise-OR reduction)
//   normal records  : grouped ncclSend/ncclRecv alltoallv of 8-byte records
//   build           : ncclAllReduce(sum) of degrees, alltoallv of edges
#include <nccl.h>

#include "internal.h"

namespace dbfs {

#define DBFS_NCCL(call)                                                                            \
    do {                                                                                           \
        ncclResult_t _r = (call);                                                                  \
        if (_r != ncclSuccess)                                                                     \
            throw ::dbfs::Error(DBFS_ENCCL, std::string(#call) + ": " + ncclGetErrorString(_r));   \
    } while (0)

static ncclComm_t comm_of(Ctx &ctx) {
    DBFS_CHECK(ctx.comm != nullptr, DBFS_EINVAL, "context has no NCCL communicator");
    return (ncclComm_t)ctx.comm;
}

void nccl_unique_id(uint8_t *out) {
    ncclUniqueId id;
    DBFS_NCCL(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof(id));
}

void nccl_init(Ctx &ctx, const uint8_t *uid, int nranks, int rank) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    DBFS_CUDA(cudaSetDevice(ctx.device));
    ncclComm_t c;
    DBFS_NCCL(ncclCommInitRank(&c, nranks, id, rank));
    ctx.comm = c;
    ctx.nranks = nranks;
    ctx.rank = rank;
}

// Another rank failed: unblock this rank's pending collectives (NCCL kernels
// see the abort flag and exit); the communicator is unusable afterwards.
void nccl_abort(Ctx &ctx) {
    if (ctx.comm) ncclCommAbort((ncclComm_t)ctx.comm);
    ctx.comm = nullptr;
}

void nccl_destroy(Ctx &ctx) {
    if (ctx.comm) ncclCommDestroy((ncclComm_t)ctx.comm);
    ctx.comm = nullptr;
}

void nccl_allreduce_u32_sum(Ctx &ctx, uint32_t *dbuf, int64_t count) {
    if (count <= 0) return;
    DBFS_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclUint32, ncclSum, comm_of(ctx), ctx.stream));
}

void nccl_allreduce_i32_min(Ctx &ctx, int32_t *dbuf, int64_t count) {
    if (count <= 0) return;
    DBFS_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclInt32, ncclMin, comm_of(ctx), ctx.stream));
}

void nccl_allreduce_i64(Ctx &ctx, int64_t *dbuf, int64_t count, int op) {  // 0 sum, 1 min, 2 max
    if (count <= 0) return;
    DBFS_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclInt64, op == 2 ? ncclMax : (op ? ncclMin : ncclSum),
                            comm_of(ctx), ctx.stream));
}

void nccl_allreduce_f64_max(Ctx &ctx, double *dbuf, int64_t count) {
    if (count <= 0) return;
    DBFS_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclFloat64, ncclMax, comm_of(ctx), ctx.stream));
}

void nccl_allreduce_u8_max(Ctx &ctx, uint8_t *dbuf, int64_t count) {
    if (count <= 0) return;
    DBFS_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclUint8, ncclMax, comm_of(ctx), ctx.stream));
}

void nccl_allgather_bytes(Ctx &ctx, const void *send, void *recv, int64_t bytes) {
    DBFS_NCCL(ncclAllGather(send, recv, (size_t)bytes, ncclChar, comm_of(ctx), ctx.stream));
}

void nccl_alltoallv_bytes(Ctx &ctx, const void *send, const int64_t *send_off, const int64_t *send_bytes,
                          void *recv, const int64_t *recv_off, const int64_t *recv_bytes) {
    ncclComm_t c = comm_of(ctx);
    DBFS_NCCL(ncclGroupStart());
    for (int o = 0; o < ctx.nranks; o++) {
        if (send_bytes[o] > 0)
            DBFS_NCCL(ncclSend((const char *)send + send_off[o], (size_t)send_bytes[o], ncclChar, o, c, ctx.stream));
        if (recv_bytes[o] > 0)
            DBFS_NCCL(ncclRecv((char *)recv + recv_off[o], (size_t)recv_bytes[o], ncclChar, o, c, ctx.stream));
    }
    DBFS_NCCL(ncclGroupEnd());
}

// Device-side barrier: an all-reduce of one word enqueued on the context
// stream, no host wait (later work on the stream runs after every rank got here).
void nccl_allreduce_async(Ctx &ctx, void *word) {
    DBFS_NCCL(ncclAllReduce(word, word, 1, ncclInt32, ncclSum, comm_of(ctx), ctx.stream));
}

void nccl_barrier(Ctx &ctx) {
    void *p = ctx.ensure_scratch(64);
    DBFS_NCCL(ncclAllReduce(p, p, 1, ncclInt32, ncclSum, comm_of(ctx), ctx.stream));
    DBFS_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace dbfs
