// The run's only collective: samples are sharded over the
// GPUs of one box with the weights replicated, every rank runs its own verify
// loop to completion, and the per-sample outputs are all-gathered at the end
// over NCCL (NVLink 5 / NVSwitch).  This gives C++ hosts that exchange without
// Python: an NCCL communicator bootstrapped from a 128-byte unique id that the
// host ships between its ranks out of band, and the all-gather.
//
// libnccl.so.2 is opened at first use (dlopen; an already loaded copy, e.g.
// torch's, is reused), so the library itself carries no link-time NCCL
// dependency and everything else works where NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "handles.h"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
        api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
        api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
        api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
        api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    });
    SD_CHECK(api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather, sdb::INTERNAL,
             "NCCL unavailable: " + (err.empty() ? std::string("missing symbols in libnccl.so.2") : err));
    return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw sdb::Error(sdb::INTERNAL, std::string("nccl: ") + what + ": " +
                                            (nccl().error_string ? nccl().error_string(r) : std::to_string((int)r)));
}

thread_local std::string g_comm_err;

template <class F>
int cguard(F&& f) {
    try {
        f();
        return sdb::OK;
    } catch (const sdb::Error& e) {
        g_comm_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_comm_err = e.what();
        return sdb::INTERNAL;
    }
}

}  // namespace

struct sd_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    cudaStream_t st = nullptr;
    ~sd_comm() {
        if (comm) nccl().comm_destroy(comm);
        if (st) cudaStreamDestroy(st);
    }
};

extern "C" {

const char* sd_comm_last_error(void) { return g_comm_err.c_str(); }

int sd_nccl_unique_id(uint8_t* id) {
    return cguard([&] {
        ncclUniqueId u;
        nccl_ok(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int sd_comm_init(const uint8_t* id, int world, int rank, int device, sd_comm** out) {
    return cguard([&] {
        SD_CHECK(world >= 1 && rank >= 0 && rank < world, sdb::CONFIG, "rank outside the world");
        sdb::set_device(device);
        auto* c = new sd_comm();
        try {
            c->world = world;
            c->rank = rank;
            c->device = device;
            ncclUniqueId u;
            std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
            nccl_ok(nccl().comm_init_rank(&c->comm, world, u, rank), "ncclCommInitRank");
            CUDA_OK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int sd_comm_size(const sd_comm* c, int* world, int* rank) {
    return cguard([&] {
        *world = c->world;
        *rank = c->rank;
    });
}

void sd_comm_destroy(sd_comm* c) {
    if (c) {
        cudaSetDevice(c->device);
        delete c;
    }
}

// Every rank contributes `count` int32 (the same count on all ranks); every
// rank receives world * count in rank order.  Host buffers in and out.
int sd_comm_allgather_i32(sd_comm* c, const int32_t* local, int64_t count, int32_t* all) {
    return cguard([&] {
        SD_CHECK(count >= 0, sdb::CONTRACT, "negative element count");
        sdb::set_device(c->device);
        const size_t n = (size_t)count, bytes = 4 * n;
        int32_t* d = (int32_t*)sdb::dmalloc(bytes * (size_t)(c->world + 1));
        try {
            int32_t* send = d + n * (size_t)c->world;
            CUDA_OK(cudaMemcpyAsync(send, local, bytes, cudaMemcpyHostToDevice, c->st));
            nccl_ok(nccl().all_gather(send, d, n, ncclInt32, c->comm, c->st), "ncclAllGather");
            CUDA_OK(cudaMemcpyAsync(all, d, bytes * (size_t)c->world, cudaMemcpyDeviceToHost, c->st));
            CUDA_OK(cudaStreamSynchronize(c->st));
        } catch (...) {
            sdb::dfree(d);
            throw;
        }
        sdb::dfree(d);
    });
}

}  // extern "C"
