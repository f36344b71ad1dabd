#include "nccl_dyn.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace hmg {

namespace {

// HMG_TRANSPORT=local (tests only): every rank a thread of this process on one
// GPU, collectives through the test transport of local_transport.cu, which is
// built into its own libhmg_localtx.so next to this library (not part of it).
const Nccl* local_transport(std::string* err) {
    static const Nccl* table = nullptr;
    static std::string load_err;
    static std::once_flag once;
    std::call_once(once, [] {
        Dl_info info{};
        std::string dir = ".";
        if (dladdr(reinterpret_cast<void*>(&local_transport), &info) && info.dli_fname) {
            dir = info.dli_fname;
            const size_t slash = dir.rfind('/');
            dir = slash == std::string::npos ? "." : dir.substr(0, slash);
        }
        const std::string path = dir + "/libhmg_localtx.so";
        void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            load_err = "HMG_TRANSPORT=local: cannot load " + path + " (test-only transport; build.py builds it)";
            return;
        }
        auto fn = reinterpret_cast<const void* (*)()>(dlsym(h, "hmg_local_transport_table"));
        if (!fn) {
            load_err = path + " lacks hmg_local_transport_table";
            return;
        }
        table = static_cast<const Nccl*>(fn());
    });
    if (!table && err) *err = load_err;
    return table;
}

}  // namespace

const Nccl* nccl(std::string* err) {
    static const bool local = [] {
        const char* e = std::getenv("HMG_TRANSPORT");
        return e && std::string(e) == "local";
    }();
    if (local) return local_transport(err);
    static Nccl table;
    static bool ok = false;
    static std::string load_err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (const char* p = std::getenv("HMG_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // the copy torch loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            load_err = "cannot load libnccl.so.2 (set HMG_NCCL_LIB)";
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        table.GetUniqueId = reinterpret_cast<decltype(table.GetUniqueId)>(sym("ncclGetUniqueId"));
        table.CommInitRank = reinterpret_cast<decltype(table.CommInitRank)>(sym("ncclCommInitRank"));
        table.CommDestroy = reinterpret_cast<decltype(table.CommDestroy)>(sym("ncclCommDestroy"));
        table.AllReduce = reinterpret_cast<decltype(table.AllReduce)>(sym("ncclAllReduce"));
        table.AllGather = reinterpret_cast<decltype(table.AllGather)>(sym("ncclAllGather"));
        table.Send = reinterpret_cast<decltype(table.Send)>(sym("ncclSend"));
        table.Recv = reinterpret_cast<decltype(table.Recv)>(sym("ncclRecv"));
        table.GroupStart = reinterpret_cast<decltype(table.GroupStart)>(sym("ncclGroupStart"));
        table.GroupEnd = reinterpret_cast<decltype(table.GroupEnd)>(sym("ncclGroupEnd"));
        table.GetErrorString = reinterpret_cast<decltype(table.GetErrorString)>(sym("ncclGetErrorString"));
        ok = table.GetUniqueId && table.CommInitRank && table.CommDestroy && table.AllReduce && table.AllGather &&
             table.Send && table.Recv && table.GroupStart && table.GroupEnd && table.GetErrorString;
        if (!ok) load_err = "libnccl.so.2 lacks a required symbol";
    });
    if (!ok) {
        if (err) *err = load_err;
        return nullptr;
    }
    return &table;
}

}  // namespace hmg
