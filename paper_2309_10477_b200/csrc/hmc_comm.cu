// hmc_comm.cu -- the cross-rank exchange of the multi-GPU engine, owned by
// libhmc (include/hmc.h "multi-process"): one process per GPU, NCCL over
// NVLink / NVSwitch.
//
// Reference counterpart: the thread fan-out + ordered fsum of
// engine.py:104-116 (workers on disjoint path ranges, partials combined in
// path order).  Here every rank simulates a contiguous, chunk-aligned slice
// of the path axis (hmc_slice_chunks -- the same rule as
// paper_2309_10477_b200.parallel.shard), and hmc_comm_gather_chunks places
// every rank's chunk partials into the global [run][chunk][HMC_NW] array in
// path order on every rank.  hmc_reduce_chunks then reduces it with the
// fixed-shape tree, so the result is bit-identical for any number of GPUs.
//
// The exchange is one ncclAllGather straight into place when every rank
// holds the same number of chunks and there is one run (the bench job:
// 1024 chunks over 1/2/4/8 GPUs), else world grouped ncclBroadcasts (rank q
// the root of its own exact-sized slice; no padding), into place for one run
// and through a private scratch + one 2-D copy per rank for several.  Payload:
// n_chunks * n_runs * 112 B (115 KB for the 2^24-path bench job) --
// latency-bound, a few microseconds over NVSwitch.
//
// NCCL is opened with dlopen on first use (the torch-bundled libnccl.so.2,
// usually already mapped into the process by torch): libhmc itself loads
// and runs single-GPU jobs without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hmc_host.h"

#ifndef HMC_NCCL_LIB_DIR
#define HMC_NCCL_LIB_DIR ""
#endif

using namespace hmc_host;

struct hmc_comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, world = 1, device = 0;
};

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

std::once_flag g_nccl_once;
NcclApi g_nccl;

void load_nccl() {
    const std::string dir = HMC_NCCL_LIB_DIR;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h && !dir.empty()) h = dlopen((dir + "/libnccl.so.2").c_str(), RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_nccl.error = std::string("cannot open libnccl.so.2: ") + dlerror();
        return;
    }
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p && g_nccl.error.empty()) g_nccl.error = std::string("libnccl.so.2 lacks ") + name;
        return p;
    };
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))sym("ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))sym("ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
    g_nccl.Broadcast = (decltype(g_nccl.Broadcast))sym("ncclBroadcast");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))sym("ncclAllReduce");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))sym("ncclAllGather");
    g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
    g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
}

int nccl_ready() {
    std::call_once(g_nccl_once, load_nccl);
    if (!g_nccl.error.empty()) return fail(HMC_E_CUDA, g_nccl.error);
    return HMC_OK;
}

#define HMC_NCCL(expr)                                                                         \
    do {                                                                                       \
        ncclResult_t r_ = (expr);                                                              \
        if (r_ != ncclSuccess)                                                                 \
            return fail(HMC_E_CUDA, std::string(#expr) + ": " + g_nccl.GetErrorString(r_));   \
    } while (0)

// parallel.shard: chunks dealt as evenly as possible, the first C % world
// ranks get one more
void slice_of(long long n_chunks, int rank, int world, long long* lo, long long* hi) {
    const long long base = n_chunks / world, extra = n_chunks % world;
    *lo = rank * base + (rank < extra ? rank : extra);
    *hi = *lo + base + (rank < extra ? 1 : 0);
}

int check_comm(const hmc_comm* c) {
    if (!c || !c->nccl) return fail(HMC_E_INVALID, "communicator is NULL or destroyed");
    return HMC_OK;
}

}  // namespace

extern "C" {

int hmc_slice_chunks(int64_t n_paths, int32_t rank, int32_t world, int64_t* chunk_lo,
                     int64_t* chunk_hi) {
    if (n_paths < 1 || world < 1 || rank < 0 || rank >= world || !chunk_lo || !chunk_hi)
        return fail(HMC_E_INVALID, "need n_paths >= 1 and 0 <= rank < world");
    long long lo, hi;
    slice_of(n_chunks_of(n_paths), rank, world, &lo, &hi);
    *chunk_lo = lo;
    *chunk_hi = hi;
    return HMC_OK;
}

int hmc_comm_unique_id(uint8_t* id_out) {
    if (!id_out) return fail(HMC_E_INVALID, "id_out is NULL");
    int rc = nccl_ready();
    if (rc) return rc;
    ncclUniqueId id;
    HMC_NCCL(g_nccl.GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == HMC_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return HMC_OK;
}

int hmc_comm_init(const uint8_t* id, int32_t rank, int32_t world, int32_t device, hmc_comm** out) {
    if (!id || !out) return fail(HMC_E_INVALID, "id / out is NULL");
    if (world < 1 || rank < 0 || rank >= world) return fail(HMC_E_INVALID, "need 0 <= rank < world");
    int rc = nccl_ready();
    if (rc) return rc;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    hmc_comm* c = new hmc_comm();
    c->rank = rank;
    c->world = world;
    c->device = device;
    const ncclResult_t r = g_nccl.CommInitRank(&c->nccl, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(HMC_E_CUDA, std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r));
    }
    *out = c;
    return HMC_OK;
}

int hmc_comm_destroy(hmc_comm* comm) {
    if (!comm) return HMC_OK;
    ncclResult_t r = ncclSuccess;
    if (comm->nccl) r = g_nccl.CommDestroy(comm->nccl);
    delete comm;
    if (r != ncclSuccess) return fail(HMC_E_CUDA, std::string("ncclCommDestroy: ") + g_nccl.GetErrorString(r));
    return HMC_OK;
}

int hmc_comm_gather_chunks(hmc_comm* comm, const double* d_local, int32_t n_runs, int64_t n_paths,
                           double* d_full, void* stream) {
    int rc = check_comm(comm);
    if (rc) return rc;
    if (!d_full || n_runs < 1 || n_paths < 1) return fail(HMC_E_INVALID, "bad gather arguments");
    const long long C = n_chunks_of(n_paths), R = n_runs;
    const size_t row = (size_t)HMC_NW * sizeof(double);
    long long my_lo, my_hi;
    slice_of(C, comm->rank, comm->world, &my_lo, &my_hi);
    if (my_hi > my_lo && !d_local) return fail(HMC_E_INVALID, "d_local is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(comm->device));
    if (R == 1 && C % comm->world == 0) {
        // equal slices, rank-major = path order: one all-gather straight into place
        HMC_NCCL(g_nccl.AllGather(d_local, d_full, (size_t)(C / comm->world) * HMC_NW, ncclDouble, comm->nccl,
                                  st));
        return HMC_OK;
    }
    if (R == 1) {  // slices are contiguous in the global array: broadcast into place
        HMC_NCCL(g_nccl.GroupStart());
        for (int q = 0; q < comm->world; ++q) {
            long long lo, hi;
            slice_of(C, q, comm->world, &lo, &hi);
            if (hi <= lo) continue;
            const void* send = q == comm->rank ? (const void*)d_local : nullptr;
            ncclResult_t r = g_nccl.Broadcast(send, d_full + lo * HMC_NW, (size_t)(hi - lo) * HMC_NW,
                                              ncclDouble, q, comm->nccl, st);
            if (r != ncclSuccess) {
                g_nccl.GroupEnd();
                return fail(HMC_E_CUDA, std::string("ncclBroadcast: ") + g_nccl.GetErrorString(r));
            }
        }
        HMC_NCCL(g_nccl.GroupEnd());
        return HMC_OK;
    }
    // several runs: rank slices [run][nc_q][HMC_NW] land back to back in a
    // scratch buffer, then one 2-D copy per rank interleaves them by run
    char* scratch = nullptr;
    HMC_CK(pool_alloc(comm->device, (void**)&scratch, (size_t)R * C * row, st));
    std::vector<long long> off((size_t)comm->world + 1, 0);
    for (int q = 0; q < comm->world; ++q) {
        long long lo, hi;
        slice_of(C, q, comm->world, &lo, &hi);
        off[q + 1] = off[q] + R * (hi - lo);
    }
    ncclResult_t r = g_nccl.GroupStart();
    for (int q = 0; q < comm->world && r == ncclSuccess; ++q) {
        if (off[q + 1] == off[q]) continue;
        const void* send = q == comm->rank ? (const void*)d_local : nullptr;
        r = g_nccl.Broadcast(send, scratch + off[q] * row, (size_t)(off[q + 1] - off[q]) * HMC_NW, ncclDouble,
                             q, comm->nccl, st);
    }
    const ncclResult_t r_end = g_nccl.GroupEnd();
    if (r == ncclSuccess) r = r_end;
    cudaError_t e = cudaSuccess;
    for (int q = 0; q < comm->world && r == ncclSuccess && e == cudaSuccess; ++q) {
        long long lo, hi;
        slice_of(C, q, comm->world, &lo, &hi);
        if (hi <= lo) continue;
        e = cudaMemcpy2DAsync(d_full + lo * HMC_NW, (size_t)C * row, scratch + off[q] * row,
                              (size_t)(hi - lo) * row, (size_t)(hi - lo) * row, (size_t)R,
                              cudaMemcpyDeviceToDevice, st);
    }
    cudaFreeAsync(scratch, st);
    if (r != ncclSuccess) return fail(HMC_E_CUDA, std::string("ncclBroadcast: ") + g_nccl.GetErrorString(r));
    HMC_CK(e);
    return HMC_OK;
}

int hmc_comm_allreduce_sum(hmc_comm* comm, void* d_buf, int64_t count, int32_t dtype, void* stream) {
    int rc = check_comm(comm);
    if (rc) return rc;
    if (!d_buf || count < 0) return fail(HMC_E_INVALID, "bad allreduce arguments");
    ncclDataType_t t;
    switch (dtype) {
        case HMC_DTYPE_I64: t = ncclInt64; break;
        case HMC_DTYPE_F64: t = ncclFloat64; break;
        default: return fail(HMC_E_INVALID, "dtype must be HMC_DTYPE_I64 or HMC_DTYPE_F64");
    }
    if (count == 0) return HMC_OK;
    const DeviceGuard keep_device;
    HMC_CK(cudaSetDevice(comm->device));
    HMC_NCCL(g_nccl.AllReduce(d_buf, d_buf, (size_t)count, t, ncclSum, comm->nccl, (cudaStream_t)stream));
    return HMC_OK;
}

}  // extern "C"
