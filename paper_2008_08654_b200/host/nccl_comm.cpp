// nccl_comm.cpp -- the multi-GPU merge of the boundary (SURVEY 8b entry 6,
// 8e): one in-place NCCL allreduce of a t x m counter table over NVLink /
// NVSwitch, the distributed form of CountSketch::merge (reference
// sketch.cpp:182-193: counter-wise wrapping u64 add).
//
// NCCL is bound at run time (dlopen of libnccl.so.2) rather than at link time:
// inside a PyTorch process the library torch already loaded is reused
// (RTLD_NOLOAD), so a communicator created by torch and one created here come
// from the same NCCL; a plain C++ caller gets the system libnccl.  The types
// and enum values come from <nccl.h> (stable across NCCL 2.x).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <type_traits>
#include <string>

#include "../../include/mersenne_b200.h"
#include "../csrc/mb200_capi_util.h"

namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetVersion) get_version = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string load_error;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // the NCCL already in the process (torch's) first, then the loader's search path
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            a.handle = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
            if (a.handle) break;
        }
        if (!a.handle)
            for (const char* nm : names) {
                a.handle = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
                if (a.handle) break;
            }
        if (!a.handle) {
            const char* e = dlerror();
            a.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.handle, name));
            if (!fn && a.load_error.empty()) a.load_error = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(a.get_version, "ncclGetVersion");
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.comm_count, "ncclCommCount");
        sym(a.all_reduce, "ncclAllReduce");
        sym(a.error_string, "ncclGetErrorString");
    });
    return a;
}

int need_api() {
    const NcclApi& a = api();
    if (!a.load_error.empty()) return mb200::fail(MB200_UNSUPPORTED, a.load_error);
    return MB200_OK;
}

int nccl_fail(ncclResult_t r, const char* where) {
    return mb200::fail(MB200_CUDA_ERROR, std::string(where) + ": " + api().error_string(r));
}

}  // namespace

extern "C" {

int mb200_nccl_version(int* version) {
    if (int rc = need_api()) return rc;
    if (!version) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    ncclResult_t r = api().get_version(version);
    return r == ncclSuccess ? MB200_OK : nccl_fail(r, "ncclGetVersion");
}

int mb200_nccl_unique_id(uint8_t out[MB200_NCCL_UNIQUE_ID_BYTES]) {
    if (int rc = need_api()) return rc;
    if (!out) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    ncclUniqueId id;
    ncclResult_t r = api().get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == MB200_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
    return MB200_OK;
}

int mb200_nccl_comm_init(int nranks, const uint8_t id[MB200_NCCL_UNIQUE_ID_BYTES], int rank, void** comm) {
    if (int rc = need_api()) return rc;
    if (!id || !comm) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return mb200::fail(MB200_INVALID_ARGUMENT, "rank out of range");
    *comm = nullptr;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    ncclResult_t r = api().comm_init_rank(&c, nranks, uid, rank);  // collective over the ranks
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return MB200_OK;
}

int mb200_nccl_comm_destroy(void* comm) {
    if (!comm) return MB200_OK;
    if (int rc = need_api()) return rc;
    ncclResult_t r = api().comm_destroy(static_cast<ncclComm_t>(comm));
    return r == ncclSuccess ? MB200_OK : nccl_fail(r, "ncclCommDestroy");
}

int mb200_nccl_comm_size(void* comm, int* nranks) {
    if (int rc = need_api()) return rc;
    if (!comm || !nranks) return mb200::fail(MB200_INVALID_ARGUMENT, "null argument");
    ncclResult_t r = api().comm_count(static_cast<ncclComm_t>(comm), nranks);
    return r == ncclSuccess ? MB200_OK : nccl_fail(r, "ncclCommCount");
}

// In-place sum of the rank-local tables.  The counters travel as ncclUint64:
// unsigned addition wraps exactly like the reference's merge, which adds the
// u64 images of the i64 counters (sketch.cpp:189-191).
int mb200_cs_allreduce(int64_t* d_counters, uint64_t count, void* nccl_comm, void* stream) {
    if (int rc = need_api()) return rc;
    if (!nccl_comm) return mb200::fail(MB200_INVALID_ARGUMENT, "null communicator");
    if (count == 0) return MB200_OK;
    if (!d_counters) return mb200::fail(MB200_INVALID_ARGUMENT, "null counters");
    ncclResult_t r = api().all_reduce(d_counters, d_counters, size_t(count), ncclUint64, ncclSum,
                                      static_cast<ncclComm_t>(nccl_comm), static_cast<cudaStream_t>(stream));
    return r == ncclSuccess ? MB200_OK : nccl_fail(r, "ncclAllReduce");
}

}  // extern "C"
