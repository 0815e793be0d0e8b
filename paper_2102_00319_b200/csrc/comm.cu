// comm.cu -- logit-ciphertext gather over NCCL (the only collective on the
// path).  Every rank evaluates its own image batch with replicated keys; the output
// logit ciphertexts (out, 2, k, N) of all ranks are all-gathered so rank 0 (or any
// rank) can hand them to the client.  Raw residues travel unchanged, so the gathered
// words are bit-identical to each rank's own result.
//
// NCCL is bound at run time (dlopen of libnccl.so.2, preferring a copy the process has
// already loaded, e.g. PyTorch's), so the library carries no link-time NCCL dependency
// and never mixes two NCCL builds in one process.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace {
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *);
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    const char *(*error_string)(ncclResult_t);
    const char *why = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
        if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_gather || !api.error_string)
            api.why = "libnccl.so.2 lacks an entry point";
    });
    return api;
}

int nccl_fail(const char *what, ncclResult_t r) {
    return fail(HEB_ECUDA, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "nccl error");
}
}  // namespace

struct heb_comm {
    ncclComm_t comm;
    int rank, nranks;
};

extern "C" int heb_comm_unique_id(uint8_t *out) {
    if (!out) return fail(HEB_EINVAL, "heb_comm_unique_id: null output");
    const NcclApi &api = nccl();
    if (api.why) return fail(HEB_EUNSUP, "heb_comm_unique_id: %s", api.why);
    ncclUniqueId id;
    const ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return HEB_OK;
}

extern "C" int heb_comm_init(heb_comm **out, const uint8_t *id, int nranks, int rank, int device) {
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(HEB_EINVAL, "heb_comm_init: bad args");
    const NcclApi &api = nccl();
    if (api.why) return fail(HEB_EUNSUP, "heb_comm_init: %s", api.why);
    CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId uid;
    memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm;
    const ncclResult_t r = api.comm_init_rank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
    *out = new heb_comm{comm, rank, nranks};
    return HEB_OK;
}

extern "C" int heb_comm_destroy(heb_comm *c) {
    if (!c) return HEB_OK;
    const ncclResult_t r = nccl().comm_destroy(c->comm);
    delete c;
    return r == ncclSuccess ? HEB_OK : nccl_fail("ncclCommDestroy", r);
}

extern "C" int heb_gather_logits(heb_comm *c, const uint64_t *send, uint64_t *recv, int64_t words, void *stream) {
    if (!c || !send || !recv || words < 0) return fail(HEB_EINVAL, "heb_gather_logits: bad args");
    if (words == 0) return HEB_OK;
    const ncclResult_t r =
        nccl().all_gather(send, recv, (size_t)words, ncclUint64, c->comm, (cudaStream_t)stream);
    return r == ncclSuccess ? HEB_OK : nccl_fail("ncclAllGather", r);
}
