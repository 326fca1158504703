// comm.cu -- the one collective of the batched-pairs path:
// an NCCL communicator per rank and the all-gather of the per-pair results
// (plus the MIN all-reduce that agrees on the first illegal residue), issued
// on the library's caller stream so PyTorch only supplies buffers.
//
// NCCL is bound at run time (dlopen "libnccl.so.2", RTLD_NOLOAD first): a
// process that already loaded PyTorch's NCCL shares that instance, so the
// library has no link-time NCCL dependency and never mixes two NCCL copies.
// Reference: overlap.py:110-152 is the per-pair call whose results are
// gathered; the reference itself is single-process.
#include <dlfcn.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace saix {

namespace {
constexpr int kIdBytes = 128;  // NCCL_UNIQUE_ID_BYTES
struct NcclId {
    char internal[kIdBytes];
};
using ncclComm_t = void *;
using ncclResult_t = int;
constexpr int kNcclInt64 = 4, kNcclMin = 3;  // ncclDataType_t / ncclRedOp_t values (nccl.h)

struct NcclApi {
    ncclResult_t (*get_unique_id)(NcclId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, NcclId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.all_reduce;
    });
    return api;
}

int nccl_fail(const char *what, ncclResult_t r) {
    NcclApi &a = nccl();
    set_error("%s: NCCL error %d (%s)", what, r, a.error_string ? a.error_string(r) : "?");
    return SAIX_ENCCL;
}
int need_nccl(const char *what) {
    if (nccl().ok) return SAIX_OK;
    set_error("%s: libnccl.so.2 not loadable", what);
    return SAIX_ENCCL;
}
}  // namespace

}  // namespace saix

using namespace saix;

extern "C" int saix_comm_unique_id(uint8_t *out) {
    if (!out) {
        set_error("saix_comm_unique_id: null output");
        return SAIX_EINVAL;
    }
    SAIX_TRY(need_nccl("saix_comm_unique_id"));
    NcclId id;
    ncclResult_t r = nccl().get_unique_id(&id);
    if (r) return nccl_fail("ncclGetUniqueId", r);
    memcpy(out, id.internal, kIdBytes);
    return SAIX_OK;
}

extern "C" int saix_comm_init(void **comm, int nranks, const uint8_t *id, int rank, int device) {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("saix_comm_init: invalid arguments");
        return SAIX_EINVAL;
    }
    SAIX_TRY(need_nccl("saix_comm_init"));
    SAIX_CUDA(cudaSetDevice(device));
    NcclId nid;
    memcpy(nid.internal, id, kIdBytes);
    ncclComm_t c = nullptr;
    ncclResult_t r = nccl().comm_init_rank(&c, nranks, nid, rank);
    if (r) return nccl_fail("ncclCommInitRank", r);
    *comm = c;
    return SAIX_OK;
}

extern "C" int saix_comm_destroy(void *comm) {
    if (!comm) return SAIX_OK;
    SAIX_TRY(need_nccl("saix_comm_destroy"));
    ncclResult_t r = nccl().comm_destroy(comm);
    if (r) return nccl_fail("ncclCommDestroy", r);
    return SAIX_OK;
}

extern "C" int saix_comm_allgather_i64(void *comm, const int64_t *send, int64_t count, int64_t *recv, void *stream) {
    if (!comm || count < 0 || (count > 0 && (!send || !recv))) {
        set_error("saix_comm_allgather_i64: invalid arguments");
        return SAIX_EINVAL;
    }
    SAIX_TRY(need_nccl("saix_comm_allgather_i64"));
    Prof prof_("comm.allgather", 8.0 * (double)count, (cudaStream_t)stream);
    ncclResult_t r = nccl().all_gather(send, recv, (size_t)count, kNcclInt64, comm, (cudaStream_t)stream);
    if (r) return nccl_fail("ncclAllGather", r);
    return SAIX_OK;
}

extern "C" int saix_comm_allreduce_min_i64(void *comm, const int64_t *send, int64_t *recv, int64_t count,
                                           void *stream) {
    if (!comm || count < 0 || (count > 0 && (!send || !recv))) {
        set_error("saix_comm_allreduce_min_i64: invalid arguments");
        return SAIX_EINVAL;
    }
    SAIX_TRY(need_nccl("saix_comm_allreduce_min_i64"));
    ncclResult_t r = nccl().all_reduce(send, recv, (size_t)count, kNcclInt64, kNcclMin, comm, (cudaStream_t)stream);
    if (r) return nccl_fail("ncclAllReduce", r);
    return SAIX_OK;
}
