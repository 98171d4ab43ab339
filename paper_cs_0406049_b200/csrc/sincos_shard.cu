// sincos_shard.cu -- the single-process multi-device run with NCCL-gathered statistics
// (SURVEY 8(e), CS4): every shard is launched on its own device, its error statistics
// (KB5) and kernel time are reduced into a 64-byte record on that device, and the records
// are all-gathered over NCCL (ncclCommInitAll over the shards' devices, one stream per
// device, inside ncclGroupStart/End).  No array data crosses devices: the collective moves
// 64 B per rank, once per run, outside any timed region of the hot kernel.
//
// NCCL is bound at run time with dlopen("libnccl.so.2") -- inside a torch process this is
// torch's own NCCL, standalone the system one -- so the library has no link-time NCCL
// dependency and the hot path never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "../../include/sincos_pairs.h"
#include "sincos_launch.h"

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

}  // namespace

extern "C" sincos_status_t sincos_last_error_set(int e);   // sincos_abi.cu

extern "C" {

int sincos_nccl_available(void) { return nccl().ok ? 1 : 0; }

sincos_status_t sincos_pairs_sharded_stats(const sincos_shard_t *shards, int nshards, sincos_variant_t variant,
                                           sincos_stats_t *gathered) {
    if (nshards < 1 || shards == nullptr || gathered == nullptr) return SINCOS_ERR_INVALID_ARGUMENT;
    for (int g = 0; g < nshards; ++g)
        for (int h = 0; h < g; ++h)
            if (shards[g].device == shards[h].device) return SINCOS_ERR_INVALID_ARGUMENT;  // one shard per device
    const Nccl &N = nccl();
    if (!N.ok) return SINCOS_ERR_INVALID_ARGUMENT;
    int prev = 0;
    cudaGetDevice(&prev);
    const size_t rec = sizeof(sincos_stats_t);
    std::vector<int> devs(nshards);
    std::vector<void *> ws(nshards, nullptr), mine(nshards, nullptr), all(nshards, nullptr);
    std::vector<cudaEvent_t> e0(nshards, nullptr), e1(nshards, nullptr);
    std::vector<ncclComm_t> comms(nshards, nullptr);
    sincos_status_t st = SINCOS_OK;
    cudaError_t ce = cudaSuccess;
    auto fail = [&](cudaError_t e) { ce = e; st = sincos_last_error_set(static_cast<int>(e)); };

    for (int g = 0; g < nshards && st == SINCOS_OK; ++g) {
        const sincos_shard_t &sh = shards[g];
        devs[g] = sh.device;
        cudaStream_t s = static_cast<cudaStream_t>(sh.stream);
        if ((ce = cudaSetDevice(sh.device)) != cudaSuccess) { fail(ce); break; }
        if ((ce = cudaMalloc(&ws[g], sincos_b200::stats_ws_bytes())) != cudaSuccess) { fail(ce); break; }
        if ((ce = cudaMalloc(&mine[g], rec)) != cudaSuccess) { fail(ce); break; }
        if ((ce = cudaMalloc(&all[g], rec * nshards)) != cudaSuccess) { fail(ce); break; }
        if ((ce = cudaEventCreate(&e0[g])) != cudaSuccess || (ce = cudaEventCreate(&e1[g])) != cudaSuccess) {
            fail(ce);
            break;
        }
        cudaEventRecord(e0[g], s);
        st = sincos_pairs(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n, variant, sh.stream);
        if (st != SINCOS_OK) break;
        cudaEventRecord(e1[g], s);
        st = sincos_error_stats(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n,
                                static_cast<sincos_stats_t *>(mine[g]), ws[g], sh.stream);
    }
    // per-shard kernel time into the record (the host waits for each shard's stream)
    for (int g = 0; g < nshards && st == SINCOS_OK; ++g) {
        cudaSetDevice(devs[g]);
        if ((ce = cudaStreamSynchronize(static_cast<cudaStream_t>(shards[g].stream))) != cudaSuccess) {
            fail(ce);
            break;
        }
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        double dms = ms;
        uint32_t dev = static_cast<uint32_t>(devs[g]);
        cudaMemcpy(static_cast<char *>(mine[g]) + offsetof(sincos_stats_t, kernel_ms), &dms, sizeof(dms),
                   cudaMemcpyHostToDevice);
        cudaMemcpy(static_cast<char *>(mine[g]) + offsetof(sincos_stats_t, device), &dev, sizeof(dev),
                   cudaMemcpyHostToDevice);
    }
    // the one collective: 64 B per rank
    if (st == SINCOS_OK) {
        if (N.init_all(comms.data(), nshards, devs.data()) != 0) st = SINCOS_ERR_CUDA;
    }
    if (st == SINCOS_OK) {
        N.group_start();
        for (int g = 0; g < nshards; ++g) {
            cudaSetDevice(devs[g]);
            N.all_gather(mine[g], all[g], rec, kNcclUint8, comms[g], static_cast<cudaStream_t>(shards[g].stream));
        }
        if (N.group_end() != 0) st = SINCOS_ERR_CUDA;
    }
    if (st == SINCOS_OK) {
        cudaSetDevice(devs[0]);
        if ((ce = cudaStreamSynchronize(static_cast<cudaStream_t>(shards[0].stream))) != cudaSuccess ||
            (ce = cudaMemcpy(gathered, all[0], rec * nshards, cudaMemcpyDeviceToHost)) != cudaSuccess)
            fail(ce);
    }
    for (int g = 0; g < nshards; ++g) {
        cudaSetDevice(devs[g]);
        cudaStreamSynchronize(static_cast<cudaStream_t>(shards[g].stream));
        if (comms[g]) N.destroy(comms[g]);
        if (ws[g]) cudaFree(ws[g]);
        if (mine[g]) cudaFree(mine[g]);
        if (all[g]) cudaFree(all[g]);
        if (e0[g]) cudaEventDestroy(e0[g]);
        if (e1[g]) cudaEventDestroy(e1[g]);
    }
    cudaSetDevice(prev);
    return st;
}

}  // extern "C"
