// comm.cu -- G6: the error-count allreduce over NCCL for callers of the C ABI.
//
// The multi-GPU BER sweep's only collective is one sum of int64[4] = {bit errors,
// failures, iterations, frames} per Eb/N0 point (channel.py:123-135 folds exactly
// these); the Python package does it with torch.distributed.  A non-Python host
// (C, Go via cgo, ...) gets the same through these entry points.  NCCL is loaded on
// first use with dlopen("libnccl.so.2") -- if torch already loaded its NCCL in this
// process, that library is reused -- so the decoder itself never depends on NCCL.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include <nccl.h>

#include "common.cuh"

struct ldpc_comm {
    ncclComm_t comm = nullptr;
    int device = 0;
};

namespace {

struct Nccl {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};

const Nccl *nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy && n.error_string;
    });
    return n.ok ? &n : nullptr;
}

int nccl_fail(const Nccl *n, ncclResult_t r, const char *what) {
    ldpc::set_error("%s: %s", what, n->error_string(r));
    return LDPC_ECUDA;
}

}  // namespace

using namespace ldpc;

extern "C" int ldpc_comm_unique_id(uint8_t *id_out) {
    LDPC_ARG_CHECK(id_out != nullptr, "NULL argument");
    const Nccl *n = nccl();
    LDPC_ARG_CHECK(n != nullptr, "NCCL (libnccl.so.2) could not be loaded");
    static_assert(sizeof(ncclUniqueId) == LDPC_COMM_ID_BYTES, "unique id size");
    ncclUniqueId id;
    const ncclResult_t r = n->get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
    return LDPC_OK;
}

extern "C" int ldpc_comm_create(int32_t nranks, int32_t rank, const uint8_t *id, ldpc_comm **out) {
    LDPC_ARG_CHECK(id != nullptr && out != nullptr, "NULL argument");
    LDPC_ARG_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "rank %d outside 0..%d", rank, nranks - 1);
    const Nccl *n = nccl();
    LDPC_ARG_CHECK(n != nullptr, "NCCL (libnccl.so.2) could not be loaded");
    *out = nullptr;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto *c = new ldpc_comm();
    LDPC_CUDA_TRY(cudaGetDevice(&c->device));
    const ncclResult_t r = n->comm_init_rank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(n, r, "ncclCommInitRank");
    }
    *out = c;
    return LDPC_OK;
}

extern "C" int ldpc_allreduce_counts_i64(ldpc_comm *c, int64_t *counts_dev, int32_t count, void *stream) {
    LDPC_ARG_CHECK(c != nullptr && counts_dev != nullptr, "NULL argument");
    LDPC_ARG_CHECK(count >= 1, "count must be at least 1");
    const Nccl *n = nccl();
    DeviceGuard dg(c->device);
    const ncclResult_t r = n->all_reduce(counts_dev, counts_dev, (size_t)count, ncclInt64, ncclSum, c->comm,
                                         (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclAllReduce");
    return LDPC_OK;
}

extern "C" void ldpc_comm_destroy(ldpc_comm *c) {
    if (!c) return;
    if (const Nccl *n = nccl()) n->comm_destroy(c->comm);
    delete c;
}
