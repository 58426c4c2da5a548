// NCCL bound at run time (dlopen) instead of link time: the process may
// already carry another libnccl.so.2 (e.g. torch's bundled 2.28 next to the
// system 2.27), and two copies of the same soname in one process break the
// one loaded second. An already-loaded libnccl is reused (RTLD_NOLOAD);
// otherwise $SPD_NCCL_LIB, then the system libnccl.so.2.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

#include "host.hpp"

namespace spd {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static NcclApi& get() {
        static NcclApi api = load();
        return api;
    }

private:
    static NcclApi load() {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("SPD_NCCL_LIB");
            if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) internal_error("NcclError", std::string("cannot load libnccl.so.2: ") + dlerror());
        NcclApi a;
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) internal_error("NcclError", std::string("libnccl lacks ") + n);
            return p;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        return a;
    }
};

#define SPD_NCCL(x)                                                                          \
    do {                                                                                     \
        ncclResult_t r_ = (x);                                                               \
        if (r_ != ncclSuccess)                                                               \
            ::spd::internal_error("NcclError",                                               \
                                  std::string(#x) + ": " + NcclApi::get().GetErrorString(r_)); \
    } while (0)

}  // namespace spd
