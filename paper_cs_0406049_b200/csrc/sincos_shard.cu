// sincos_shard.cu -- the single-process multi-device run with NCCL-gathered statistics
// (SURVEY 8(e), CS4): every shard is launched on its own device, its error statistics
// (KB5) and kernel time are reduced into a 64-byte record on that device, and the records
// are all-gathered over NCCL (ncclCommInitAll over the shards' devices, one stream per
// device, inside ncclGroupStart/End).  No array data crosses devices: the collective moves
// 64 B per rank, once per run, outside any timed region of the hot kernel.
//
// The communicator and the small per-device buffers (workspace, record, gathered records,
// timing events) are created once per device list and kept for the process: a second call on
// the same devices reuses them.  Every CUDA and NCCL return is checked; a failing NCCL call
// returns SINCOS_ERR_NCCL with its code in sincos_last_nccl_error(), a failing CUDA call
// SINCOS_ERR_CUDA with its code in sincos_last_cuda_error(); work already queued is drained
// before any error return.
//
// NCCL is bound at run time with dlopen("libnccl.so.2") -- inside a torch process this is
// torch's own NCCL, standalone the system one -- so the library has no link-time NCCL
// dependency and the hot path never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <memory>
#include <mutex>
#include <vector>

#include "../../include/sincos_pairs.h"
#include "sincos_launch.h"

extern "C" sincos_status_t sincos_last_error_set(int e);   // sincos_abi.cu

namespace {

// The few NCCL entry points used (ABI of nccl.h 2.x).
typedef struct ncclComm *ncclComm_t;
typedef int ncclResult_t;                 // ncclSuccess == 0
constexpr int kNcclUint8 = 1;             // ncclDataType_t ncclUint8
using CommInitAll_t = ncclResult_t (*)(ncclComm_t *, int, const int *);
using AllGather_t = ncclResult_t (*)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t);
using Group_t = ncclResult_t (*)();
using CommDestroy_t = ncclResult_t (*)(ncclComm_t);

struct Nccl {
    bool ok = false;
    CommInitAll_t init_all = nullptr;
    AllGather_t all_gather = nullptr;
    Group_t group_start = nullptr, group_end = nullptr;
    CommDestroy_t destroy = nullptr;
};

std::mutex g_nccl_mu;
Nccl g_nccl;
bool g_nccl_tried = false;
thread_local int g_last_nccl_error = 0;

const Nccl &nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl_tried) {
        g_nccl_tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            g_nccl.init_all = reinterpret_cast<CommInitAll_t>(dlsym(h, "ncclCommInitAll"));
            g_nccl.all_gather = reinterpret_cast<AllGather_t>(dlsym(h, "ncclAllGather"));
            g_nccl.group_start = reinterpret_cast<Group_t>(dlsym(h, "ncclGroupStart"));
            g_nccl.group_end = reinterpret_cast<Group_t>(dlsym(h, "ncclGroupEnd"));
            g_nccl.destroy = reinterpret_cast<CommDestroy_t>(dlsym(h, "ncclCommDestroy"));
            g_nccl.ok = g_nccl.init_all && g_nccl.all_gather && g_nccl.group_start && g_nccl.group_end &&
                        g_nccl.destroy;
        }
    }
    return g_nccl;
}

// Everything one device list needs, created once and kept (the communicator is the costly
// part: ncclCommInitAll takes ~0.1-1 s).
struct Ctx {
    std::vector<int> devs;
    std::vector<ncclComm_t> comms;
    std::vector<void *> ws, mine, all;
    std::vector<cudaEvent_t> e0, e1;
    std::mutex busy;                 // one call at a time per device list
};

std::mutex g_ctx_mu;
std::vector<Ctx *> *g_ctxs = new std::vector<Ctx *>();   // never freed (process lifetime)

sincos_status_t nccl_fail(ncclResult_t r) {
    g_last_nccl_error = r;
    return SINCOS_ERR_NCCL;
}

// Release what a partly built context holds (its own devices only).
void release(Ctx *c) {
    const Nccl &N = nccl();
    for (size_t g = 0; g < c->devs.size(); ++g) {
        if (cudaSetDevice(c->devs[g]) != cudaSuccess) continue;
        if (g < c->comms.size() && c->comms[g]) N.destroy(c->comms[g]);
        if (c->ws[g]) cudaFree(c->ws[g]);
        if (c->mine[g]) cudaFree(c->mine[g]);
        if (c->all[g]) cudaFree(c->all[g]);
        if (c->e0[g]) cudaEventDestroy(c->e0[g]);
        if (c->e1[g]) cudaEventDestroy(c->e1[g]);
    }
    delete c;
}

// The cached context of this device list, or a new one (nullptr + status on failure).
Ctx *context(const std::vector<int> &devs, sincos_status_t *st) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (Ctx *c : *g_ctxs)
        if (c->devs == devs) return c;
    const Nccl &N = nccl();
    const size_t G = devs.size(), rec = sizeof(sincos_stats_t);
    Ctx *c = new Ctx();
    c->devs = devs;
    c->ws.assign(G, nullptr);
    c->mine.assign(G, nullptr);
    c->all.assign(G, nullptr);
    c->e0.assign(G, nullptr);
    c->e1.assign(G, nullptr);
    cudaError_t e = cudaSuccess;
    for (size_t g = 0; g < G && e == cudaSuccess; ++g) {
        if ((e = cudaSetDevice(devs[g])) != cudaSuccess) break;
        if ((e = cudaMalloc(&c->ws[g], sincos_b200::stats_ws_bytes())) != cudaSuccess) break;
        if ((e = cudaMalloc(&c->mine[g], rec)) != cudaSuccess) break;
        if ((e = cudaMalloc(&c->all[g], rec * G)) != cudaSuccess) break;
        if ((e = cudaEventCreate(&c->e0[g])) != cudaSuccess) break;
        e = cudaEventCreate(&c->e1[g]);
    }
    if (e != cudaSuccess) {
        *st = sincos_last_error_set(static_cast<int>(e));
        release(c);
        return nullptr;
    }
    c->comms.assign(G, nullptr);
    const ncclResult_t r = N.init_all(c->comms.data(), static_cast<int>(G), devs.data());
    if (r != 0) {
        c->comms.assign(G, nullptr);       // a failed init leaves no communicator to destroy
        *st = nccl_fail(r);
        release(c);
        return nullptr;
    }
    g_ctxs->push_back(c);
    return c;
}

}  // namespace

extern "C" {

int sincos_nccl_available(void) { return nccl().ok ? 1 : 0; }

int sincos_last_nccl_error(void) { return g_last_nccl_error; }

sincos_status_t sincos_pairs_sharded_stats(const sincos_shard_t *shards, int nshards, sincos_variant_t variant,
                                           sincos_stats_t *gathered) {
    if (nshards < 1 || shards == nullptr || gathered == nullptr) return SINCOS_ERR_INVALID_ARGUMENT;
    if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED) return SINCOS_ERR_INVALID_ARGUMENT;
    for (int g = 0; g < nshards; ++g)
        for (int h = 0; h < g; ++h)
            if (shards[g].device == shards[h].device) return SINCOS_ERR_INVALID_ARGUMENT;  // one shard per device
    const Nccl &N = nccl();
    if (!N.ok) return SINCOS_ERR_INVALID_ARGUMENT;
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess) return sincos_last_error_set(static_cast<int>(ce));
    for (int g = 0; g < nshards; ++g)
        if (shards[g].device < 0 || shards[g].device >= ndev) return SINCOS_ERR_INVALID_ARGUMENT;
    int prev = 0;
    if ((ce = cudaGetDevice(&prev)) != cudaSuccess) return sincos_last_error_set(static_cast<int>(ce));

    std::vector<int> devs(nshards);
    for (int g = 0; g < nshards; ++g) devs[g] = shards[g].device;
    sincos_status_t st = SINCOS_OK;
    Ctx *c = context(devs, &st);
    if (c == nullptr) {
        cudaSetDevice(prev);
        return st;
    }
    std::lock_guard<std::mutex> call_lock(c->busy);
    const size_t rec = sizeof(sincos_stats_t);
    auto stream = [&](int g) { return static_cast<cudaStream_t>(shards[g].stream); };
    auto cuda = [&](cudaError_t e) {
        if (e != cudaSuccess && st == SINCOS_OK) st = sincos_last_error_set(static_cast<int>(e));
        return e == cudaSuccess;
    };
    int touched = 0;                 // shards whose streams may hold work of this call

    for (int g = 0; g < nshards && st == SINCOS_OK; ++g) {
        const sincos_shard_t &sh = shards[g];
        if (!cuda(cudaSetDevice(sh.device))) break;
        touched = g + 1;
        if (!cuda(cudaEventRecord(c->e0[g], stream(g)))) break;
        st = sincos_pairs(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n, variant, sh.stream);
        if (st != SINCOS_OK) break;
        if (!cuda(cudaEventRecord(c->e1[g], stream(g)))) break;
        st = sincos_error_stats(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n,
                                static_cast<sincos_stats_t *>(c->mine[g]), c->ws[g], sh.stream);
    }
    // per-shard kernel time and device into the record (the host waits for each shard's stream)
    std::vector<double> ms(nshards, 0.0);
    std::vector<uint32_t> dv(nshards, 0);
    for (int g = 0; g < nshards && st == SINCOS_OK; ++g) {
        if (!cuda(cudaSetDevice(devs[g])) || !cuda(cudaStreamSynchronize(stream(g)))) break;
        float f = 0.0f;
        if (!cuda(cudaEventElapsedTime(&f, c->e0[g], c->e1[g]))) break;
        ms[g] = f;
        dv[g] = static_cast<uint32_t>(devs[g]);
        char *r = static_cast<char *>(c->mine[g]);
        if (!cuda(cudaMemcpyAsync(r + offsetof(sincos_stats_t, kernel_ms), &ms[g], sizeof(double),
                                  cudaMemcpyHostToDevice, stream(g))) ||
            !cuda(cudaMemcpyAsync(r + offsetof(sincos_stats_t, device), &dv[g], sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, stream(g))))
            break;
    }
    // the one collective: 64 B per rank
    if (st == SINCOS_OK) {
        ncclResult_t r = N.group_start();
        if (r != 0) st = nccl_fail(r);
        for (int g = 0; g < nshards && st == SINCOS_OK; ++g) {
            if (!cuda(cudaSetDevice(devs[g]))) break;
            if ((r = N.all_gather(c->mine[g], c->all[g], rec, kNcclUint8, c->comms[g], stream(g))) != 0)
                st = nccl_fail(r);
        }
        // the group is always closed once opened (even after a failed enqueue)
        const ncclResult_t r2 = N.group_end();
        if (r2 != 0 && st == SINCOS_OK) st = nccl_fail(r2);
    }
    if (st == SINCOS_OK && cuda(cudaSetDevice(devs[0])) && cuda(cudaStreamSynchronize(stream(0))))
        cuda(cudaMemcpy(gathered, c->all[0], rec * nshards, cudaMemcpyDeviceToHost));
    // drain every stream this call used before returning (success or not): the records and
    // the staging values above must not be read after the call, nor the caller's buffers
    for (int g = 0; g < (st == SINCOS_OK ? nshards : touched); ++g) {
        if (cudaSetDevice(devs[g]) != cudaSuccess) continue;
        const cudaError_t e = cudaStreamSynchronize(stream(g));
        if (e != cudaSuccess && st == SINCOS_OK) st = sincos_last_error_set(static_cast<int>(e));
    }
    if (st == SINCOS_ERR_NCCL) {
        // a failed collective may leave the communicator unusable: the next call on these devices
        // builds a new context (this one is dropped from the cache -- not destroyed, which could
        // block on a broken communicator -- and its small buffers are leaked)
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        for (size_t i = 0; i < g_ctxs->size(); ++i)
            if ((*g_ctxs)[i] == c) {
                g_ctxs->erase(g_ctxs->begin() + static_cast<long>(i));
                break;
            }
    }
    cudaSetDevice(prev);
    return st;
}

}  // extern "C"
