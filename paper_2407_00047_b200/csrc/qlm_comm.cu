// qlm_comm.cu -- the NCCL communicator behind the C ABI (a8 cross-GPU min-loc,
// a12 MC combine; SURVEY.md 8(b) qlm_comm_unique_id / qlm_comm_attach).
//
// NCCL is resolved at run time with dlopen: a process that already loaded
// NCCL (torch does) shares that copy, so the library and torch.distributed
// never run two NCCL builds side by side, and libqlm.so has no link-time
// NCCL dependency (it builds and loads on a box without NCCL; the comm calls
// then fail with QLM_ENCCL).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "qlm_comm.h"
#include "qlm_launch.h"

namespace qlm {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*GetVersion)(int *);
    bool ok = false;
    std::string why;
};

NcclApi &api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded, if any
        if (!h) {
            const char *path = getenv("QLM_NCCL_PATH");
            h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) {
            a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
#define QLM_SYM(field, name)                                                  \
    *reinterpret_cast<void **>(&a.field) = dlsym(h, name);                    \
    if (!a.field) {                                                           \
        a.why = std::string("libnccl.so.2 has no symbol ") + name;            \
        return;                                                               \
    }
        QLM_SYM(GetUniqueId, "ncclGetUniqueId");
        QLM_SYM(CommInitRank, "ncclCommInitRank");
        QLM_SYM(CommDestroy, "ncclCommDestroy");
        QLM_SYM(AllGather, "ncclAllGather");
        QLM_SYM(AllReduce, "ncclAllReduce");
        QLM_SYM(GetErrorString, "ncclGetErrorString");
        QLM_SYM(GetVersion, "ncclGetVersion");
#undef QLM_SYM
        a.ok = true;
    });
    return a;
}

bool nccl_ok(ncclResult_t r, const char *what, std::string &err) {
    if (r == ncclSuccess) return true;
    err = std::string(what) + ": " + api().GetErrorString(r);
    return false;
}

}  // namespace

struct Comm {
    ncclComm_t c = nullptr;
    int rank = 0, world = 1;
};

bool comm_unique_id(uint8_t id[kCommIdBytes], std::string &err) {
    static_assert(sizeof(ncclUniqueId) == kCommIdBytes, "ncclUniqueId is 128 bytes");
    NcclApi &a = api();
    if (!a.ok) { err = a.why; return false; }
    ncclUniqueId u;
    if (!nccl_ok(a.GetUniqueId(&u), "ncclGetUniqueId", err)) return false;
    memcpy(id, &u, kCommIdBytes);
    return true;
}

Comm *comm_init(const uint8_t id[kCommIdBytes], int rank, int world, std::string &err) {
    NcclApi &a = api();
    if (!a.ok) { err = a.why; return nullptr; }
    ncclUniqueId u;
    memcpy(&u, id, kCommIdBytes);
    Comm *c = new Comm;
    c->rank = rank;
    c->world = world;
    if (!nccl_ok(a.CommInitRank(&c->c, world, u, rank), "ncclCommInitRank", err)) {
        delete c;
        return nullptr;
    }
    return c;
}

void comm_destroy(Comm *c) {
    if (!c) return;
    if (c->c) api().CommDestroy(c->c);
    delete c;
}

int comm_rank(const Comm *c) { return c ? c->rank : 0; }
int comm_world(const Comm *c) { return c ? c->world : 1; }

bool comm_allgather_bytes(Comm *c, const void *send, void *recv, size_t bytes, cudaStream_t st,
                          std::string &err) {
    nvtxRangePushA("qlm_nccl_allgather");
    qlog(1, "ncclAllGather %zu B x %d ranks", bytes, c->world);
    const bool ok = nccl_ok(api().AllGather(send, recv, bytes, ncclUint8, c->c, st), "ncclAllGather", err);
    nvtxRangePop();
    return ok;
}

bool comm_allreduce_sum_u32(Comm *c, uint32_t *buf, size_t n, cudaStream_t st, std::string &err) {
    nvtxRangePushA("qlm_nccl_allreduce_sum");
    qlog(1, "ncclAllReduce(sum, u32) n=%zu", n);
    const bool ok = nccl_ok(api().AllReduce(buf, buf, n, ncclUint32, ncclSum, c->c, st), "ncclAllReduce(sum)", err);
    nvtxRangePop();
    return ok;
}

bool comm_allreduce_max_i32(Comm *c, int32_t *buf, size_t n, cudaStream_t st, std::string &err) {
    nvtxRangePushA("qlm_nccl_allreduce_max");
    qlog(1, "ncclAllReduce(max, i32) n=%zu", n);
    const bool ok = nccl_ok(api().AllReduce(buf, buf, n, ncclInt32, ncclMax, c->c, st), "ncclAllReduce(max)", err);
    nvtxRangePop();
    return ok;
}

int comm_nccl_version() {
    NcclApi &a = api();
    int v = 0;
    if (a.ok) a.GetVersion(&v);
    return v;
}

}  // namespace qlm
