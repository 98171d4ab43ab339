// sincos_abi.cu -- the extern "C" boundary of libsincos_pairs.so (include/sincos_pairs.h).
//
// Validation (no CUDA call on any error path), path selection (256-bit / 128-bit
// vector body with a scalar head and tail; register re-alignment for pointers
// that do not share an alignment), grid sizing, the pipelined host-buffer path,
// and the single-process multi-device sharder (one host thread per device).
// The kernel configuration is fixed (sincos_launch.h Tuning); the A/B build
// (-DSINCOS_AB) adds the settable alternatives and sincos_pairs_batched.
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <stdint.h>
#include <stdlib.h>

#ifndef SINCOS_PHASE_STAGED
#define SINCOS_PHASE_STAGED 1      // 0: rows of 2-7 pairs through the short-row kernel (A/B)
#endif
#ifndef SINCOS_PHASE_STAGED_SPLIT_MIN
#define SINCOS_PHASE_STAGED_SPLIT_MIN 4   // split rows of 2-3 pairs: the tiny-row kernel (A/B: 2)
#endif
#include <string.h>

#include "../../include/sincos_pairs.h"
#include "sincos_launch.h"
#ifdef SINCOS_AB
#include "sincos_ab.h"
#endif
#include "sincos_method.cuh"
#include "sincos_realign.cuh"

using namespace sincos_b200;

namespace {

thread_local int g_last_cuda_error = 0;
std::atomic<uint64_t> g_launches{0};

constexpr int kMaxDev = 64;
std::atomic<int> g_sm_count[kMaxDev];

sincos_status_t cuda_fail(cudaError_t e) {
    g_last_cuda_error = static_cast<int>(e);
    return SINCOS_ERR_CUDA;
}

int sm_count(int dev) {
    if (dev < 0 || dev >= kMaxDev) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 1;
    }
    int v = g_sm_count[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 1;
        g_sm_count[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    return a0 < b0 + bbytes && b0 < a0 + abytes;
}

bool aligned(const void *p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// Shared argument validation of sincos_pairs / sincos_pairs_host / null kernel.
sincos_status_t validate(const float *theta, const float *so, const float *co, const float *io, size_t n,
                         int variant, bool allow_null_variant) {
    if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED && !(allow_null_variant && variant == 2))
        return SINCOS_ERR_INVALID_ARGUMENT;
    if (n == 0) return SINCOS_OK;
    const bool split = so != nullptr && co != nullptr && io == nullptr;
    const bool inter = so == nullptr && co == nullptr && io != nullptr;
    if (theta == nullptr || !(split || inter)) return SINCOS_ERR_INVALID_ARGUMENT;
    if (!aligned(theta, 4) || (so && !aligned(so, 4)) || (co && !aligned(co, 4)) || (io && !aligned(io, 4)))
        return SINCOS_ERR_INVALID_ARGUMENT;
    if (n > (SIZE_MAX / 8)) return SINCOS_ERR_INVALID_ARGUMENT;
    const size_t b4 = 4 * n, b8 = 8 * n;
    if (split) {
        if (overlaps(so, b4, co, b4)) return SINCOS_ERR_OVERLAP;
        if (theta != so && overlaps(theta, b4, so, b4)) return SINCOS_ERR_OVERLAP;
        if (theta != co && overlaps(theta, b4, co, b4)) return SINCOS_ERR_OVERLAP;
    } else if (overlaps(theta, b4, io, b8)) {
        return SINCOS_ERR_OVERLAP;
    }
    return SINCOS_OK;
}

// Blocks for `units` work items of `per_block` per block: the full grid (one trip each), capped at
// SMs x blocks_per_sm when that is configured (grid-stride), and at grid.x's limit.
unsigned grid_for(size_t units, size_t per_block, int sms, int cfg_bps) {
    size_t need = (units + per_block - 1) / per_block;
    if (need < 1) need = 1;
    if (cfg_bps > 0 && need > static_cast<size_t>(sms) * cfg_bps) need = static_cast<size_t>(sms) * cfg_bps;
    if (need > 0x7FFFFFFFu) need = 0x7FFFFFFFu;   // the kernels grid-stride past it
    return static_cast<unsigned>(need);
}

// Launch on already-validated arguments, n > 0.
// Path, first that applies (identical numerics on every path):
//   KB1/KB2 vector kernel (theta and outputs share a 32-B / 16-B alignment after a head) ->
//   KB3b  theta re-aligned (split sin/cos share an offset mod 16 B; interleaved 8-B aligned) ->
//   KB3c  outputs re-aligned (everything else).
// (A/B build, realign = 0: KB3, one element per thread, instead of KB3b/KB3c.)
sincos_status_t launch(const float *theta, float *so, float *co, float *io, size_t n, int variant,
                       cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    const Tuning T = tuning();
    const int sms = sm_count(dev);
    const bool inter = io != nullptr;
    const bool nc = !(theta == so || theta == co);
    const int threads = T.threads;
    const int cfg_bps = T.blocks_per_sm;
    const bool realign = T.realign != 0;

    // Widest vector whose alignment theta and the outputs share after a scalar head.
    int w = 0;
    size_t head = 0;
    for (int cand = T.vec; cand >= 4; cand /= 2) {
        const uintptr_t A = 4u * cand;  // bytes of theta per access
        const uintptr_t t = reinterpret_cast<uintptr_t>(theta);
        const size_t h = ((A - (t & (A - 1))) & (A - 1)) / 4;
        const uintptr_t off = 4 * h;
        bool ok = true;
        if (inter)
            ok = aligned(reinterpret_cast<const char *>(io) + 2 * off, A);
        else
            ok = aligned(reinterpret_cast<const char *>(so) + off, A) &&
                 aligned(reinterpret_cast<const char *>(co) + off, A);
        if (ok) {
            w = cand;
            head = h;
            break;
        }
    }

    // KB3b: theta re-aligned onto the outputs' 256-bit frame -- split outputs whose sin and cos
    // share one offset mod 32 B (theta elsewhere); interleaved outputs without the 256-bit path
    // but 8-B aligned (its 256-bit store per four pairs beats the 128-bit path's half-sector
    // stores).
    size_t hs = SIZE_MAX;
    const uintptr_t sc = reinterpret_cast<uintptr_t>(so) ^ reinterpret_cast<uintptr_t>(co);
    if (realign) {
        if (inter) {
            // (w == 4 with the default vec 8 only: an A/B vec 4 keeps its 128-bit kernel)
            if ((w == 0 || (w == 4 && T.vec == 8)) && aligned(io, 8))
                hs = ((32 - (reinterpret_cast<uintptr_t>(io) & 31)) & 31) / 8;
        } else if (T.realign == 2) {
            // (A/B: the 128-bit form wherever sin and cos share 16 B)
            if (w == 0 && (sc & 15) == 0) hs = ((16 - (reinterpret_cast<uintptr_t>(so) & 15)) & 15) / 4;
        } else if ((w == 0 || (w == 4 && T.vec == 8)) && (sc & 31) == 0) {
            // sin and cos at one offset mod 32 B: theta re-aligned onto their 256-bit frame (also
            // when theta shares only 16 B with them: the 128-bit vector kernel ran 6.2 TB/s there,
            // the 256-bit re-alignment 6.8).  Sharing only 16 B: KB3c below (the 128-bit
            // re-alignment ran 5.6-6.2 TB/s; profiles/r02/ab_layouts_all*.jsonl)
            hs = ((32 - (reinterpret_cast<uintptr_t>(so) & 31)) & 31) / 4;
        }
    }
    // 256-bit form when the outputs take 256-bit stores at a common element (split: sin and cos
    // share their offset mod 32 B; interleaved: always, being 8-B aligned here)
    const bool shift8 = T.realign == 1 || T.realign == 3;
    if (hs != SIZE_MAX && shift8 &&
        (inter || ((reinterpret_cast<uintptr_t>(so) ^ reinterpret_cast<uintptr_t>(co)) & 31) == 0)) {
        const size_t h0 = inter ? ((32 - (reinterpret_cast<uintptr_t>(io) & 31)) & 31) / 8
                                : ((32 - (reinterpret_cast<uintptr_t>(so) & 31)) & 31) / 4;
        const int k = static_cast<int>(((reinterpret_cast<uintptr_t>(theta) + 4 * h0) & 31) / 4);   // 0..7
        if (k != 0) {
            if (!nc) return SINCOS_ERR_OVERLAP;  // unreachable: in place shares theta's alignment
            size_t hb = h0 >= static_cast<size_t>(k) ? h0 : h0 + 8;
            if (hb > n) hb = n;
            // the second aligned vector of every thread inside theta: (hb - k) + 8 nvec + 7 <= n - 1
            const size_t nvec = n + k >= hb + 8 ? (n + k - hb - 8) / 8 : 0;
            e = launch_shift8(variant, inter, k, grid_for(nvec, threads, sms, cfg_bps), threads, theta, so, co, io,
                              hb, nvec, n, stream);
            if (e != cudaSuccess) return cuda_fail(e);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            return SINCOS_OK;
        }
    }
    if (hs != SIZE_MAX) {
#ifdef SINCOS_AB
        const int k = static_cast<int>(((reinterpret_cast<uintptr_t>(theta) + 4 * hs) & 15) / 4);   // 0..3
        size_t hb = hs >= static_cast<size_t>(k) ? hs : hs + 4;    // aligned theta base >= theta
        if (hb > n) hb = n;
        // k > 0: every thread's second aligned vector must lie inside theta:
        // (hb - k) + 4 nvec + 3 <= n - 1
        size_t nvec = (n - hb) / 4;
        if (k > 0) nvec = n + k >= hb + 4 ? (n + k - hb - 4) / 4 : 0;
        if (!nc) return SINCOS_ERR_OVERLAP;      // unreachable: in place shares theta's alignment
        e = launch_shift(variant, inter, k, grid_for(nvec, threads, sms, cfg_bps), threads, theta, so, co, io, hb,
                         nvec, n, stream);
#else
        return SINCOS_ERR_INVALID_ARGUMENT;      // unreachable: the product takes the 256-bit forms
#endif
    } else if ((w == 0 || (w == 4 && !inter && T.vec == 8 && T.realign != 2)) && realign) {
        // KB3c: theta's frame, outputs re-aligned (sin and cos apart mod 16 B; pairs only 4-B aligned)
        const uintptr_t ta = reinterpret_cast<uintptr_t>(theta);
        size_t hb = ((32 - (ta & 31)) & 31) / 4;
        if (hb > n) hb = n;
        const size_t nvec = (n - hb) / 8;
        int ks, kc = 0;
        if (inter) {
            ks = static_cast<int>(((reinterpret_cast<uintptr_t>(io) + 8 * hb) & 31) / 4);
        } else {
            ks = static_cast<int>(((reinterpret_cast<uintptr_t>(so) + 4 * hb) & 31) / 4);
            kc = static_cast<int>(((reinterpret_cast<uintptr_t>(co) + 4 * hb) & 31) / 4);
        }
        // Exact in place (theta == sin or theta == cos) reaches KB3c only with the aliased stream
        // at theta's own alignment (k = 0): each thread then writes exactly the elements of theta
        // it read itself, after reading them -- which is what makes the read-only (.nc) theta
        // loads safe here.  Any other aliasing was refused by validate(); keep the invariant
        // explicit rather than implied.
        if ((theta == so && ks != 0) || (theta == co && kc != 0)) return SINCOS_ERR_OVERLAP;
        e = launch_outshift(variant, inter, ks, kc, grid_for(nvec, threads, sms, cfg_bps), threads, theta, so, co,
                            io, hb, nvec, n, stream);
    } else if (w == 0) {
#ifdef SINCOS_AB
        const unsigned grid = static_cast<unsigned>(
            (n + threads - 1) / threads < static_cast<size_t>(sms) * 8 ? (n + threads - 1) / threads : sms * 8);
        e = launch_scalar(variant, inter, grid, threads, theta, so, co, io, n, stream);
#else
        return SINCOS_ERR_INVALID_ARGUMENT;          // unreachable: the product always re-aligns
#endif
    } else {
        if (head > n) head = n;
        const size_t nvec = (n - head) / w;
        // Default (blocks_per_sm == 0): the full grid, one trip of `unroll` vectors per thread --
        // measured fastest on B200.  blocks_per_sm > 0 (A/B): a grid-stride
        // grid of SMs x blocks_per_sm blocks.
        const unsigned grid = grid_for(nvec, static_cast<size_t>(threads) * T.unroll, sms, cfg_bps);
        e = launch_vec(variant, inter, w, T.unroll, nc, T.prefetch == 1, T.pdl != 0, grid, threads, theta, so, co,
                       io, head, nvec, n, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

// ---- host-buffer pipeline ----------------------------------------------------------
// Three slots, chunks ramping up from 2^16 elements.  Measured against 2 and 4 slots, a tail
// ramping down again, and 256 MiB - 2 GiB of workspace (tools/ab_host.py,
// profiles/r02/ab_host*.jsonl): all within 1% of each other, ~0.97 of the PCIe roofline.
#ifndef SINCOS_HOST_SLOTS
#define SINCOS_HOST_SLOTS 3
#endif
#ifndef SINCOS_HOST_MIN_CHUNK_LOG2
#define SINCOS_HOST_MIN_CHUNK_LOG2 16
#endif
constexpr int kSlots = SINCOS_HOST_SLOTS;
constexpr size_t kMinChunk = size_t(1) << SINCOS_HOST_MIN_CHUNK_LOG2;

struct DevStreams {
    bool init = false;
    cudaStream_t s[kSlots];
    cudaEvent_t done[kSlots];
    cudaEvent_t start;
    // one host-path call at a time per device: the slot streams and events are shared, and an
    // interleaved cudaEventRecord(start) from another thread would re-target this call's waits
    std::mutex busy;
};
std::mutex g_dev_mu;
DevStreams g_dev[kMaxDev];

cudaError_t dev_streams(int dev, DevStreams **out) {
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevStreams &d = g_dev[dev];
    if (!d.init) {
        for (int k = 0; k < kSlots; ++k) {
            cudaError_t e = cudaStreamCreateWithFlags(&d.s[k], cudaStreamNonBlocking);
            if (e != cudaSuccess) return e;
            e = cudaEventCreateWithFlags(&d.done[k], cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaEventCreateWithFlags(&d.start, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        d.init = true;
    }
    *out = &d;
    return cudaSuccess;
}

// ---- one host thread per device (sincos_pairs_sharded) ---------------------------------
// Workers are created on first use and live for the process (heap objects never destroyed,
// so no static destructor races a worker at exit); each runs the jobs posted to it in order.
struct Latch {
    explicit Latch(int n) : left(n) {}
    void count_down() {
        std::lock_guard<std::mutex> lk(mu);
        if (--left == 0) cv.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return left == 0; });
    }
    std::mutex mu;
    std::condition_variable cv;
    int left;
};

class DeviceWorker {
  public:
    explicit DeviceWorker(int dev) : dev_(dev), th_([this] { run(); }) { th_.detach(); }
    void post(std::function<void()> job) {
        std::lock_guard<std::mutex> lk(mu_);
        q_.push_back(std::move(job));
        cv_.notify_one();
    }

  private:
    void run() {
        cudaSetDevice(dev_);
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return !q_.empty(); });
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }
    int dev_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    std::thread th_;
};

std::mutex g_worker_mu;
DeviceWorker *g_workers[kMaxDev] = {};

DeviceWorker *device_worker(int dev) {
    std::lock_guard<std::mutex> lk(g_worker_mu);
    if (g_workers[dev] == nullptr) g_workers[dev] = new DeviceWorker(dev);
    return g_workers[dev];
}

}  // namespace

#ifdef SINCOS_AB
extern "C" int sincos_ab_get(int knob);
namespace sincos_b200 {
Tuning tuning() {
    Tuning t;
    t.threads = sincos_ab_get(SINCOS_AB_THREADS);
    t.blocks_per_sm = sincos_ab_get(SINCOS_AB_BLOCKS_PER_SM);
    t.vec = sincos_ab_get(SINCOS_AB_VEC);
    t.unroll = sincos_ab_get(SINCOS_AB_UNROLL);
    t.prefetch = sincos_ab_get(SINCOS_AB_PREFETCH);
    t.realign = sincos_ab_get(SINCOS_AB_REALIGN);
    t.pdl = sincos_ab_get(SINCOS_AB_PDL);
    t.nudft_packed = sincos_ab_get(SINCOS_AB_NUDFT_PACKED);
    return t;
}
}  // namespace sincos_b200
#endif

extern "C" {

sincos_status_t sincos_pairs(const float *theta_dev, float *sin_dev, float *cos_dev, float *inter_dev, size_t n,
                             sincos_variant_t variant, void *stream) {
    sincos_status_t st = validate(theta_dev, sin_dev, cos_dev, inter_dev, n, variant, false);
    if (st != SINCOS_OK || n == 0) return st;
    return launch(theta_dev, sin_dev, cos_dev, inter_dev, n, variant, static_cast<cudaStream_t>(stream));
}

sincos_status_t sincos_compare_cuda(const float *theta_dev, float *sin_dev, float *cos_dev, float *inter_dev,
                                    size_t n, int which, void *stream) {
    if (which != 3 && which != 4) return SINCOS_ERR_INVALID_ARGUMENT;
    sincos_status_t st = validate(theta_dev, sin_dev, cos_dev, inter_dev, n, SINCOS_NORMALIZED, false);
    if (st != SINCOS_OK || n == 0) return st;
    const bool inter = inter_dev != nullptr;
    if (!aligned(theta_dev, 32) || (inter ? !aligned(inter_dev, 32) : !aligned(sin_dev, 32) || !aligned(cos_dev, 32)))
        return SINCOS_ERR_INVALID_ARGUMENT;
    if (theta_dev == sin_dev || theta_dev == cos_dev) return SINCOS_ERR_OVERLAP;
    const size_t nvec = n / 8;
    size_t grid = (nvec + 127) / 128;
    if (grid < 1) grid = 1;
    if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;
    cudaError_t e = launch_compare(which, inter, static_cast<unsigned>(grid), 128, theta_dev, sin_dev, cos_dev,
                                   inter_dev, nvec, n, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

sincos_status_t sincos_null_4in8out(const float *theta_dev, float *sin_dev, float *cos_dev, float *inter_dev,
                                    size_t n, void *stream) {
    sincos_status_t st = validate(theta_dev, sin_dev, cos_dev, inter_dev, n, 2, true);
    if (st != SINCOS_OK || n == 0) return st;
    return launch(theta_dev, sin_dev, cos_dev, inter_dev, n, 2, static_cast<cudaStream_t>(stream));
}

sincos_status_t sincos_phase_grid(const float *f_dev, size_t nf, const float *t_dev, size_t nt, float *sin_dev,
                                  float *cos_dev, float *inter_dev, sincos_units_t units, sincos_variant_t variant,
                                  void *stream) {
    if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED) return SINCOS_ERR_INVALID_ARGUMENT;
    if (units != SINCOS_RADIANS && units != SINCOS_TURNS) return SINCOS_ERR_INVALID_ARGUMENT;
    if (nf == 0 || nt == 0) return SINCOS_OK;
    if (nt > SIZE_MAX / 8 / nf) return SINCOS_ERR_INVALID_ARGUMENT;
    const size_t n = nf * nt;
    const bool split = sin_dev != nullptr && cos_dev != nullptr && inter_dev == nullptr;
    const bool inter = sin_dev == nullptr && cos_dev == nullptr && inter_dev != nullptr;
    if (f_dev == nullptr || t_dev == nullptr || !(split || inter)) return SINCOS_ERR_INVALID_ARGUMENT;
    if (!aligned(f_dev, 4) || !aligned(t_dev, 4) || (sin_dev && !aligned(sin_dev, 4)) ||
        (cos_dev && !aligned(cos_dev, 4)) || (inter_dev && !aligned(inter_dev, 4)))
        return SINCOS_ERR_INVALID_ARGUMENT;
    const void *outs[2] = {split ? static_cast<const void *>(sin_dev) : inter_dev, split ? cos_dev : nullptr};
    const size_t ob = split ? 4 * n : 8 * n;
    if (split && overlaps(sin_dev, ob, cos_dev, ob)) return SINCOS_ERR_OVERLAP;
    for (const void *o : outs) {
        if (o == nullptr) continue;
        if (overlaps(o, ob, f_dev, 4 * nf) || overlaps(o, ob, t_dev, 4 * nt)) return SINCOS_ERR_OVERLAP;
    }
    // whole-vector rows: the vector kernel from kPhaseVecMinNt on (shorter rows leave its
    // threads idle: nt = 16 ran at 0.7 TB/s; the short-row kernel takes them)
    const bool vec = nt % 8 == 0 && nt >= kPhaseVecMinNt && aligned(t_dev, 32) &&
                     (split ? aligned(sin_dev, 32) && aligned(cos_dev, 32) : aligned(inter_dev, 32));
    cudaError_t e;
    // any other shape: when the outputs can take 256-bit stores from some pair on (split: sin
    // and cos share their alignment mod 32 B; interleaved: 8-B aligned), the row path for
    // nt >= kPhaseRowsMinNt, else the flat path (its fp64 quotient estimate of a pair index needs
    // n < 2^52); else one per thread
    const uintptr_t so_a = reinterpret_cast<uintptr_t>(sin_dev), co_a = reinterpret_cast<uintptr_t>(cos_dev),
                    io_a = reinterpret_cast<uintptr_t>(inter_dev);
    const Tuning T = tuning();
    const bool flat = !vec && T.realign != 0 && n < (size_t(1) << 52) &&
                      (split ? ((so_a ^ co_a) & 31) == 0 : aligned(inter_dev, 8));
    // rows of one pair (split or interleaved) or of 2-3 pairs (split), outputs 32-B aligned at
    // pair 0: the tiny-row kernel (its per-lane store stride, 8 nt pairs, spreads a warp's store
    // over more lines as nt grows: for nt >= 4, and interleaved nt = 2-3, the short-row kernel
    // was faster -- profiles/r02/ab_phase_tiny.jsonl -- and the staged kernel below is now)
    const bool tiny = flat && T.realign != 3 && (nt == 1 || (split && nt < SINCOS_PHASE_STAGED_SPLIT_MIN)) &&
                      (split ? aligned(sin_dev, 32) && aligned(cos_dev, 32) : aligned(inter_dev, 32));
    // rows of 4-14 pairs (split) or 2-15 (interleaved), outputs 16-B aligned at pair 0: the staged
    // short-row kernel (a warp's 128 rows staged in shared memory, written back as contiguous
    // 512-B store instructions)
    const bool staged = SINCOS_PHASE_STAGED && flat && !tiny && T.realign != 3 && phase_staged_ok(inter, nt) &&
                        (split ? nt >= SINCOS_PHASE_STAGED_SPLIT_MIN && aligned(sin_dev, 16) && aligned(cos_dev, 16)
                               : aligned(inter_dev, 16));
    if (tiny) {
        e = launch_phase_tiny(variant, inter, units == SINCOS_TURNS, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                              inter_dev, static_cast<cudaStream_t>(stream));
    } else if (staged) {
        size_t max_grid = 0;                   // the full grid (A/B: blocks_per_sm > 0 grid-strides)
        if (T.blocks_per_sm > 0) {
            int dev = 0;
            if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e);
            max_grid = static_cast<size_t>(sm_count(dev)) * T.blocks_per_sm;
        }
        e = launch_phase_staged(variant, inter, units == SINCOS_TURNS, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                                inter_dev, max_grid, static_cast<cudaStream_t>(stream));
    } else if (flat && nt >= kPhaseRowsMinNt && T.realign != 3) {
        const unsigned h0 = static_cast<unsigned>(split ? ((32 - (so_a & 31)) & 31) / 4 : ((32 - (io_a & 31)) & 31) / 8);
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e);
        e = launch_phase_rows(variant, inter, units == SINCOS_TURNS, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                              inter_dev, h0, sm_count(dev), static_cast<cudaStream_t>(stream));
    } else if (flat) {
        size_t head = split ? ((32 - (so_a & 31)) & 31) / 4 : ((32 - (io_a & 31)) & 31) / 8;
        if (head > n) head = n;
        const size_t nvec = (n - head) / 8;
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e);
        size_t grid = (nvec + 127) / 128;
        if (grid < 1) grid = 1;
        if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;
        const bool short_rows = T.realign != 3 && nt < kPhaseRowsMinNt;
        // the short-row kernel stages t in shared memory once per block: a grid of a few
        // blocks per SM, grid-striding, amortises that
        const size_t cap = static_cast<size_t>(sm_count(dev)) * phase_short_blocks_per_sm(nt);
        if (short_rows && grid > cap) grid = cap;
        e = launch_phase_flat(variant, inter, units == SINCOS_TURNS, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                              inter_dev, head, nvec, static_cast<unsigned>(grid), short_rows,
                              static_cast<cudaStream_t>(stream));
    } else if (!vec && T.realign != 0 && n < (size_t(1) << 52)) {
        // unshared output alignment: sin[]'s frame (interleaved: any), the other stream re-aligned
        size_t head = split ? ((32 - (so_a & 31)) & 31) / 4 : 0;
        if (head > n) head = n;
        const size_t nvec = (n - head) / 8;
        const int kc = split ? static_cast<int>(((co_a + 4 * head) & 31) / 4)
                             : static_cast<int>(((io_a + 8 * head) & 31) / 4);
        size_t grid = (nvec + 127) / 128;
        if (grid < 1) grid = 1;
        if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;
        e = launch_phase_flat_sh(variant, inter, units == SINCOS_TURNS, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                                 inter_dev, head, nvec, static_cast<unsigned>(grid), kc,
                                 static_cast<cudaStream_t>(stream));
    } else {
        e = launch_phase_grid(variant, inter, units == SINCOS_TURNS, vec, f_dev, nf, t_dev, nt, sin_dev, cos_dev,
                              inter_dev, static_cast<cudaStream_t>(stream));
    }
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

sincos_status_t sincos_pairs_dtype(const float *theta_dev, void *sin_dev, void *cos_dev, void *inter_dev, size_t n,
                                   sincos_variant_t variant, sincos_dtype_t out_dtype, void *stream) {
    if (out_dtype == SINCOS_F32)
        return sincos_pairs(theta_dev, static_cast<float *>(sin_dev), static_cast<float *>(cos_dev),
                            static_cast<float *>(inter_dev), n, variant, stream);
    if (out_dtype != SINCOS_F16 && out_dtype != SINCOS_BF16) return SINCOS_ERR_INVALID_ARGUMENT;
    if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED) return SINCOS_ERR_INVALID_ARGUMENT;
    if (n == 0) return SINCOS_OK;
    const bool split = sin_dev != nullptr && cos_dev != nullptr && inter_dev == nullptr;
    const bool inter = sin_dev == nullptr && cos_dev == nullptr && inter_dev != nullptr;
    if (theta_dev == nullptr || !(split || inter) || n > SIZE_MAX / 8) return SINCOS_ERR_INVALID_ARGUMENT;
    if (!aligned(theta_dev, 4) || (sin_dev && !aligned(sin_dev, 2)) || (cos_dev && !aligned(cos_dev, 2)) ||
        (inter_dev && !aligned(inter_dev, 4)))
        return SINCOS_ERR_INVALID_ARGUMENT;
    if (split) {
        if (overlaps(sin_dev, 2 * n, cos_dev, 2 * n) || overlaps(theta_dev, 4 * n, sin_dev, 2 * n) ||
            overlaps(theta_dev, 4 * n, cos_dev, 2 * n))
            return SINCOS_ERR_OVERLAP;
    } else if (overlaps(theta_dev, 4 * n, inter_dev, 4 * n)) {
        return SINCOS_ERR_OVERLAP;
    }
    // vector body: the outputs' alignment fixes the first vector element (split: sin[]'s 128-bit
    // stores, cos[] at the same offset mod 16 B or else in the widest pieces its own alignment
    // allows; interleaved: one 256-bit store per 8 pairs), theta is re-aligned in registers when
    // it sits off that alignment (sincos_realign.cuh)
    const uintptr_t so_a = reinterpret_cast<uintptr_t>(sin_dev), co_a = reinterpret_cast<uintptr_t>(cos_dev),
                    io_a = reinterpret_cast<uintptr_t>(inter_dev);
    bool vec = inter || ((so_a ^ co_a) & 15) == 0 || tuning().realign != 0;
    const size_t h0 = inter ? ((32 - (io_a & 31)) & 31) / 4 : ((16 - (so_a & 15)) & 15) / 2;
    int k = 0;
    size_t head = 0, nvec = 0;
    if (vec) {
        realign_plan(theta_dev, n, h0, &k, &head, &nvec);
        if (k != 0 && tuning().realign == 0) vec = false;
    }
    if (!vec) head = nvec = 0, k = 0;
    int cw = 16;                                   // cos[]'s alignment at the vector elements
    if (!inter) {
        const uintptr_t ca = (co_a + 2 * head) & 15;
        cw = ca == 0 ? 16 : (ca & 7) == 0 ? 8 : (ca & 3) == 0 ? 4 : 2;
    }
    // without the vector path every element is a "tail" element: one per thread
    const size_t work = vec ? (nvec > 8 ? nvec : 8) : n;
    size_t grid = (work + 127) / 128;
    if (grid > 0x7FFFFFFFu) return SINCOS_ERR_INVALID_ARGUMENT;
    cudaError_t e = launch_pairs16(variant, out_dtype, inter, static_cast<unsigned>(grid), theta_dev, sin_dev,
                                   cos_dev, inter_dev, head, nvec, n, k, cw, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

static sincos_status_t interleave_impl(bool to_inter, const float *s, const float *c, float *io, size_t n,
                                       void *stream) {
    if (n == 0) return SINCOS_OK;
    if (s == nullptr || c == nullptr || io == nullptr || n > SIZE_MAX / 8) return SINCOS_ERR_INVALID_ARGUMENT;
    if (!aligned(s, 4) || !aligned(c, 4) || !aligned(io, 8)) return SINCOS_ERR_INVALID_ARGUMENT;
    if (overlaps(s, 4 * n, c, 4 * n) || overlaps(s, 4 * n, io, 8 * n) || overlaps(c, 4 * n, io, 8 * n))
        return SINCOS_ERR_OVERLAP;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    size_t grid = (n / 4 + 255) / 256;                // a vector of 4 per thread, one trip
    if (grid < 1) grid = 1;
    if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;
    e = launch_interleave(to_inter, static_cast<unsigned>(grid), s, c, io, n, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

sincos_status_t sincos_interleave(const float *sin_dev, const float *cos_dev, float *inter_dev, size_t n,
                                  void *stream) {
    return interleave_impl(true, sin_dev, cos_dev, inter_dev, n, stream);
}

sincos_status_t sincos_deinterleave(const float *inter_dev, float *sin_dev, float *cos_dev, size_t n, void *stream) {
    return interleave_impl(false, sin_dev, cos_dev, const_cast<float *>(inter_dev), n, stream);
}

sincos_status_t sincos_pairs_method(const float *theta_dev, float *sin_dev, float *cos_dev, float *inter_dev,
                                    size_t n, const sincos_method_t *m, void *stream) {
    if (m == nullptr || m->n_ss < 1 || m->n_ss > 8 || m->n_cc < 0 || m->n_cc > 8 || m->doublings < 0 ||
        m->doublings > 8 || !(m->fix == 0 || m->fix == 1 || m->fix == 3) || (m->fix != 3 && m->doublings < 1))
        return SINCOS_ERR_INVALID_ARGUMENT;
    sincos_status_t st = validate(theta_dev, sin_dev, cos_dev, inter_dev, n, SINCOS_NORMALIZED, false);
    if (st != SINCOS_OK || n == 0) return st;
    if (theta_dev == sin_dev || theta_dev == cos_dev) return SINCOS_ERR_OVERLAP;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    const bool inter = inter_dev != nullptr;
    // 256-bit vector body where the outputs take 256-bit stores (split: sin and cos at one
    // offset mod 32 B; interleaved: 8-B aligned), theta re-aligned in registers when it sits
    // off that alignment (sincos_realign.cuh)
    const uintptr_t so_a = reinterpret_cast<uintptr_t>(sin_dev), co_a = reinterpret_cast<uintptr_t>(cos_dev),
                    io_a = reinterpret_cast<uintptr_t>(inter_dev);
    // (split with cos[] off sin[]'s 32-B offset: cos re-aligned by shuffles in the kernel;
    // interleaved pairs only 4-B aligned: theta's own 32-B frame, the pairs re-aligned)
    const bool inter4 = inter && !aligned(inter_dev, 8);
    bool vec = inter ? (!inter4 || tuning().realign != 0)
                     : (((so_a ^ co_a) & 31) == 0 || tuning().realign != 0);
    const size_t h0 = inter4  ? ((32 - (reinterpret_cast<uintptr_t>(theta_dev) & 31)) & 31) / 4
                      : inter ? ((32 - (io_a & 31)) & 31) / 8
                              : ((32 - (so_a & 31)) & 31) / 4;
    int k = 0;
    size_t head = 0, nvec = 0;
    if (vec) {
        realign_plan(theta_dev, n, h0, &k, &head, &nvec);
        if (k != 0 && tuning().realign == 0) vec = false;
    }
    if (!vec) head = nvec = 0, k = 0;
    size_t work = vec ? (nvec > 0 ? nvec : 1) : n;
    size_t grid = (work + 127) / 128;
    if (!vec && grid > static_cast<size_t>(sm_count(dev)) * 16) grid = static_cast<size_t>(sm_count(dev)) * 16;
    if (grid > 0x7FFFFFFFu) grid = 0x7FFFFFFFu;
    e = launch_method(m->ss, m->n_ss, m->cc, m->n_cc, m->doublings, m->fix, inter, vec, static_cast<unsigned>(grid),
                      theta_dev, sin_dev, cos_dev, inter_dev, head, nvec, n, k, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

size_t sincos_nudft_chunk(size_t nt) { return nudft_chunk(nt); }

size_t sincos_nudft_workspace_bytes(size_t nf, size_t nt) { return nudft_ws_bytes(nf, nt); }

namespace {
bool method_ok(const sincos_method_t *m) {
    return m != nullptr && m->n_ss >= 1 && m->n_ss <= 8 && m->n_cc >= 0 && m->n_cc <= 8 && m->doublings >= 0 &&
           m->doublings <= 8 && (m->fix == 0 || m->fix == 1 || m->fix == 3) && (m->fix == 3 || m->doublings >= 1);
}

// a compile-time kernel shape for common methods (-1: the generic padded kernel)
int method_spec(const sincos_method_t *m) {
    if (m->n_ss == 4 && m->n_cc == 3 && m->doublings == 2) return 0;
    if (m->n_ss == 3 && m->n_cc == 2 && m->doublings == 1) return 1;
    return -1;
}

// variant 0..4, or 5 with a general method m
sincos_status_t nudft_impl(const float *f_dev, size_t nf, const float *t_dev, const float *a_dev, size_t nt,
                           float *out_dev, sincos_units_t units, int variant, const sincos_method_t *m,
                           void *ws_dev, size_t ws_bytes, void *stream) {
    if (variant < 0 || variant > 5 || (variant == 5 && !method_ok(m))) return SINCOS_ERR_INVALID_ARGUMENT;
    if (units != SINCOS_RADIANS && units != SINCOS_TURNS) return SINCOS_ERR_INVALID_ARGUMENT;
    if (nf == 0) return SINCOS_OK;
    if (f_dev == nullptr || out_dev == nullptr || !aligned(f_dev, 4) || !aligned(out_dev, 8))
        return SINCOS_ERR_INVALID_ARGUMENT;
    if (nf > SIZE_MAX / 16 || nt > SIZE_MAX / 16) return SINCOS_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (overlaps(out_dev, 8 * nf, f_dev, 4 * nf)) return SINCOS_ERR_OVERLAP;
    if (nt == 0) {
        cudaError_t e = cudaMemsetAsync(out_dev, 0, 8 * nf, s);
        return e == cudaSuccess ? SINCOS_OK : cuda_fail(e);
    }
    if (t_dev == nullptr || a_dev == nullptr || ws_dev == nullptr || !aligned(t_dev, 4) || !aligned(a_dev, 8) ||
        !aligned(ws_dev, 16))                            // fp64 {re, im} partials: 16-B accesses
        return SINCOS_ERR_INVALID_ARGUMENT;
    const size_t need = nudft_ws_bytes(nf, nt);
    if (ws_bytes < need) return SINCOS_ERR_INVALID_ARGUMENT;
    if (overlaps(out_dev, 8 * nf, t_dev, 4 * nt) || overlaps(out_dev, 8 * nf, a_dev, 8 * nt) ||
        overlaps(ws_dev, need, out_dev, 8 * nf) || overlaps(ws_dev, need, f_dev, 4 * nf) ||
        overlaps(ws_dev, need, t_dev, 4 * nt) || overlaps(ws_dev, need, a_dev, 8 * nt))
        return SINCOS_ERR_OVERLAP;
    MethodParams mp{};
    if (variant == 5) mp = make_params(m->ss, m->n_ss, m->cc, m->n_cc, m->doublings);
    cudaError_t e = launch_nudft(variant, units == SINCOS_TURNS, f_dev, nf, t_dev, a_dev, nt, out_dev, ws_dev, s,
                                 variant == 5 ? &mp : nullptr, variant == 5 && (m->n_ss > 4 || m->n_cc > 4) ? 8 : 4,
                                 variant == 5 ? m->fix : 0, variant == 5 ? method_spec(m) : -1,
                                 tuning().nudft_packed != 0);
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return SINCOS_OK;
}

}  // namespace

sincos_status_t sincos_nudft(const float *f_dev, size_t nf, const float *t_dev, const float *a_dev, size_t nt,
                             float *out_dev, sincos_units_t units, int variant, void *ws_dev, size_t ws_bytes,
                             void *stream) {
    if (variant > 4) return SINCOS_ERR_INVALID_ARGUMENT;
    return nudft_impl(f_dev, nf, t_dev, a_dev, nt, out_dev, units, variant, nullptr, ws_dev, ws_bytes, stream);
}

sincos_status_t sincos_nudft_method(const float *f_dev, size_t nf, const float *t_dev, const float *a_dev,
                                    size_t nt, float *out_dev, sincos_units_t units, const sincos_method_t *method,
                                    void *ws_dev, size_t ws_bytes, void *stream) {
    if (!method_ok(method)) return SINCOS_ERR_INVALID_ARGUMENT;
    return nudft_impl(f_dev, nf, t_dev, a_dev, nt, out_dev, units, 5, method, ws_dev, ws_bytes, stream);
}

size_t sincos_host_workspace_min_bytes(void) { return kSlots * kMinChunk * 12; }

sincos_status_t sincos_pairs_host(const float *theta_host, float *sin_host, float *cos_host, float *inter_host,
                                  size_t n, sincos_variant_t variant, void *dev_ws, size_t ws_bytes, void *stream) {
    sincos_status_t st = validate(theta_host, sin_host, cos_host, inter_host, n, variant, false);
    if (st != SINCOS_OK || n == 0) return st;
    if (dev_ws == nullptr || ws_bytes < sincos_host_workspace_min_bytes() || !aligned(dev_ws, 256))
        return SINCOS_ERR_INVALID_ARGUMENT;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    DevStreams *ds = nullptr;
    if ((e = dev_streams(dev, &ds)) != cudaSuccess) return cuda_fail(e);

    std::lock_guard<std::mutex> call_lock(ds->busy);   // reentrancy (header: thread-safe)

    // slot capacity in elements, a multiple of 64 so every slot buffer stays 256-B aligned
    const size_t cap = (ws_bytes / (kSlots * 12)) & ~size_t(63);
    const bool inter = inter_host != nullptr;
    char *ws = static_cast<char *>(dev_ws);
    cudaStream_t caller = static_cast<cudaStream_t>(stream);

    if ((e = cudaEventRecord(ds->start, caller)) != cudaSuccess) return cuda_fail(e);
    for (int k = 0; k < kSlots; ++k)
        if ((e = cudaStreamWaitEvent(ds->s[k], ds->start, 0)) != cudaSuccess) return cuda_fail(e);

    // From here on work may be queued on the slot streams: every exit drains them first, so no
    // copy or kernel of this call is still using the caller's buffers when it returns.
    auto drain = [&](sincos_status_t s) {
        for (int k = 0; k < kSlots; ++k) cudaStreamSynchronize(ds->s[k]);
        return s;
    };
    // Chunk sizes ramp up from kMinChunk, doubling to the slot capacity: the first device->host
    // copy starts after a short first chunk, not after a whole slot's copy and kernel (the fill
    // of the pipeline; its drain is the last chunk's device->host copy either way).
    size_t chunk = kMinChunk < cap ? kMinChunk : cap;
    size_t j = 0;
    for (size_t off = 0, m = 0; off < n; off += m, ++j) {
        if (j > 0 && chunk < cap) chunk = 2 * chunk < cap ? 2 * chunk : cap;
        m = n - off < chunk ? n - off : chunk;
        const int k = static_cast<int>(j % kSlots);
        cudaStream_t s = ds->s[k];
        float *th = reinterpret_cast<float *>(ws + k * cap * 12);
        float *o1 = th + cap;        // sin, or interleaved pairs
        float *o2 = o1 + cap;        // cos
        if ((e = cudaMemcpyAsync(th, theta_host + off, 4 * m, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return drain(cuda_fail(e));
        st = inter ? launch(th, nullptr, nullptr, o1, m, variant, s) : launch(th, o1, o2, nullptr, m, variant, s);
        if (st != SINCOS_OK) return drain(st);
        if (inter) {
            if ((e = cudaMemcpyAsync(inter_host + 2 * off, o1, 8 * m, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
                return drain(cuda_fail(e));
        } else {
            if ((e = cudaMemcpyAsync(sin_host + off, o1, 4 * m, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
                return drain(cuda_fail(e));
            if ((e = cudaMemcpyAsync(cos_host + off, o2, 4 * m, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
                return drain(cuda_fail(e));
        }
    }
    for (int k = 0; k < kSlots; ++k) {
        if ((e = cudaEventRecord(ds->done[k], ds->s[k])) != cudaSuccess) return drain(cuda_fail(e));
        if ((e = cudaStreamWaitEvent(caller, ds->done[k], 0)) != cudaSuccess) return drain(cuda_fail(e));
    }
    sincos_status_t result = SINCOS_OK;
    for (int k = 0; k < kSlots; ++k)
        if ((e = cudaStreamSynchronize(ds->s[k])) != cudaSuccess && result == SINCOS_OK) result = cuda_fail(e);
    return result;
}

int sincos_shard_range(size_t n, int nshards, int g, size_t *lo, size_t *hi) {
    if (nshards < 1 || g < 0 || g >= nshards || lo == nullptr || hi == nullptr) return -1;
    auto cut = [&](int k) -> size_t {
        if (k >= nshards) return n;
        const unsigned __int128 p = static_cast<unsigned __int128>(n) * static_cast<unsigned>(k) /
                                    static_cast<unsigned>(nshards);
        return static_cast<size_t>(p) & ~size_t(7);
    };
    *lo = cut(g);
    *hi = cut(g + 1);
    if (*hi < *lo) *hi = *lo;
    return 0;
}

sincos_status_t sincos_pairs_sharded(const sincos_shard_t *shards, int nshards, sincos_variant_t variant) {
    if (nshards < 0 || (nshards > 0 && shards == nullptr)) return SINCOS_ERR_INVALID_ARGUMENT;
    for (int g = 0; g < nshards; ++g) {
        const sincos_shard_t &sh = shards[g];
        sincos_status_t st = validate(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n, variant, false);
        if (st != SINCOS_OK) return st;
    }
    if (nshards == 0) return SINCOS_OK;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e);
    for (int g = 0; g < nshards; ++g)
        if (shards[g].device < 0 || shards[g].device >= ndev || shards[g].device >= kMaxDev)
            return SINCOS_ERR_INVALID_ARGUMENT;                        // before anything is launched
    // the shards of each device, in shard order
    std::vector<int> devs;
    std::vector<std::vector<int>> of;
    for (int g = 0; g < nshards; ++g) {
        if (shards[g].n == 0) continue;
        size_t i = 0;
        while (i < devs.size() && devs[i] != shards[g].device) ++i;
        if (i == devs.size()) {
            devs.push_back(shards[g].device);
            of.emplace_back();
        }
        of[i].push_back(g);
    }
    std::vector<sincos_status_t> st(nshards, SINCOS_OK);
    std::vector<int> err(nshards, 0);
    auto run_device = [&](size_t i) {          // on the device's worker thread (or inline)
        cudaError_t ce = cudaSetDevice(devs[i]);
        for (int g : of[i]) {
            const sincos_shard_t &sh = shards[g];
            if (ce != cudaSuccess) {
                st[g] = SINCOS_ERR_CUDA;
                err[g] = static_cast<int>(ce);
                continue;
            }
            st[g] = launch(sh.theta_dev, sh.sin_dev, sh.cos_dev, sh.inter_dev, sh.n, variant,
                           static_cast<cudaStream_t>(sh.stream));
            err[g] = st[g] == SINCOS_ERR_CUDA ? g_last_cuda_error : 0;
        }
    };
    // SINCOS_SHARDED_WORKERS=1 (test hook, read once): the worker threads even for one device,
    // so a one-GPU box exercises the multi-device launch machinery too
    static const bool force_workers = [] {
        const char *v = getenv("SINCOS_SHARDED_WORKERS");
        return v != nullptr && v[0] == '1';
    }();
    if (devs.size() <= 1 && !(force_workers && !devs.empty())) {
        // one device: launch from the calling thread, keeping its current device
        int prev = 0;
        if ((e = cudaGetDevice(&prev)) != cudaSuccess) return cuda_fail(e);
        if (!devs.empty()) run_device(0);
        cudaSetDevice(prev);
    } else {
        // several devices: one host thread per device launches its shards, so the devices
        // start together instead of one launch latency apart each (launch skew)
        Latch latch(static_cast<int>(devs.size()));
        for (size_t i = 0; i < devs.size(); ++i)
            device_worker(devs[i])->post([&, i] {
                run_device(i);
                latch.count_down();
            });
        latch.wait();
    }
    for (int g = 0; g < nshards; ++g)          // the first failing shard's status (and CUDA error)
        if (st[g] != SINCOS_OK) {
            if (st[g] == SINCOS_ERR_CUDA) g_last_cuda_error = err[g];
            return st[g];
        }
    return SINCOS_OK;
}

size_t sincos_stats_workspace_bytes(void) { return stats_ws_bytes(); }

sincos_status_t sincos_error_stats(const float *theta_dev, const float *sin_dev, const float *cos_dev,
                                   const float *inter_dev, size_t n, sincos_stats_t *stats_dev, void *ws_dev,
                                   void *stream) {
    const bool split = sin_dev != nullptr && cos_dev != nullptr && inter_dev == nullptr;
    const bool inter = sin_dev == nullptr && cos_dev == nullptr && inter_dev != nullptr;
    if (stats_dev == nullptr || ws_dev == nullptr || (n > 0 && (theta_dev == nullptr || !(split || inter))))
        return SINCOS_ERR_INVALID_ARGUMENT;
    // fp64 / 64-bit fields in the record and the workspace; fp32 arrays
    if (!aligned(stats_dev, 8) || !aligned(ws_dev, 8) ||
        (n > 0 && (!aligned(theta_dev, 4) || (split && (!aligned(sin_dev, 4) || !aligned(cos_dev, 4))) ||
                   (inter && !aligned(inter_dev, 4)))))
        return SINCOS_ERR_INVALID_ARGUMENT;
    cudaError_t e = launch_stats(theta_dev, sin_dev, cos_dev, inter_dev, n, stats_dev, ws_dev,
                                 static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

#ifdef SINCOS_AB
// ---- A/B build only (csrc/sincos_ab.h) -------------------------------------------------
sincos_status_t sincos_pairs_batched(const sincos_item_t *items, int count, sincos_variant_t variant,
                                     void *stream) {
    if (count < 0 || (count > 0 && items == nullptr)) return SINCOS_ERR_INVALID_ARGUMENT;
    if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED) return SINCOS_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < count; ++i) {           // every item valid before anything is launched
        const sincos_item_t &it = items[i];
        sincos_status_t st = validate(it.theta_dev, it.sin_dev, it.cos_dev, it.inter_dev, it.n, variant, false);
        if (st != SINCOS_OK) return st;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static thread_local BatchParams p;          // ~29 KB: not on the stack
    for (int first = 0; first < count; first += kBatchMax) {
        const int m = count - first < kBatchMax ? count - first : kBatchMax;
        p.count = m;
        p.pad = 0;
        p.prefix[0] = 0;
        for (int i = 0; i < m; ++i) {
            const sincos_item_t &it = items[first + i];
            BatchItem &b = p.items[i];
            b.theta = it.theta_dev;
            b.so = it.sin_dev;
            b.co = it.cos_dev;
            b.io = it.inter_dev;
            b.n = it.n;
            // 256-bit body when theta and the outputs share a 32-B alignment after the same head
            // (exact in-place items take the plain-load one-per-thread form)
            const uintptr_t t = reinterpret_cast<uintptr_t>(it.theta_dev);
            const uint64_t h = ((32 - (t & 31)) & 31) / 4;
            bool vec = it.n > 0 && it.theta_dev != it.sin_dev && it.theta_dev != it.cos_dev;
            if (vec) {
                if (it.inter_dev)
                    vec = aligned(reinterpret_cast<const char *>(it.inter_dev) + 8 * h, 32);
                else
                    vec = aligned(reinterpret_cast<const char *>(it.sin_dev) + 4 * h, 32) &&
                          aligned(reinterpret_cast<const char *>(it.cos_dev) + 4 * h, 32);
            }
            b.head = vec ? (h < it.n ? h : it.n) : 0;
            b.vec = vec ? 1u : 0u;
            b.pad = 0;
            p.prefix[i + 1] = p.prefix[i] + batched_chunks(it.n, b.head, vec);
        }
        if (p.prefix[m] > 0x7FFFFFFFull) return SINCOS_ERR_INVALID_ARGUMENT;
        if (p.prefix[m] == 0) continue;
        cudaError_t e = launch_batched(variant, p, s);   // parameters are copied at launch
        if (e != cudaSuccess) return cuda_fail(e);
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return SINCOS_OK;
}

namespace {
std::atomic<int> g_ab[SINCOS_AB_KNOBS] = {{128}, {0}, {8}, {1}, {0}, {1}, {1}, {1}};
bool ab_ok(int knob, int v) {
    switch (knob) {
    case SINCOS_AB_THREADS: return v == 128 || v == 256 || v == 512;
    case SINCOS_AB_BLOCKS_PER_SM: return v >= 0 && v <= 4096;
    case SINCOS_AB_VEC: return v == 4 || v == 8;
    case SINCOS_AB_UNROLL: return v == 1 || v == 2 || v == 4;
    case SINCOS_AB_PREFETCH: return v == 0 || v == 1;
    case SINCOS_AB_REALIGN: return v >= 0 && v <= 3;
    case SINCOS_AB_PDL: return v == 0 || v == 1;
    case SINCOS_AB_NUDFT_PACKED: return v == 0 || v == 1;
    default: return false;
    }
}
}  // namespace

int sincos_ab_set(int knob, int value) {
    if (!ab_ok(knob, value)) return -1;
    return g_ab[knob].exchange(value);
}

int sincos_ab_get(int knob) { return knob >= 0 && knob < SINCOS_AB_KNOBS ? g_ab[knob].load() : -1; }
#endif  // SINCOS_AB

sincos_status_t sincos_debug_packed_check(int variant, const sincos_method_t *method,
                                          unsigned long long *mismatch_dev, void *stream) {
    if (mismatch_dev == nullptr || !aligned(mismatch_dev, 8)) return SINCOS_ERR_INVALID_ARGUMENT;
    int shape = -1, fix = 0;
    MethodParams mp{};
    if (method != nullptr) {
        if (!method_ok(method)) return SINCOS_ERR_INVALID_ARGUMENT;
        shape = method_spec(method);
        fix = method->fix;
        if (shape < 0 || (fix != 0 && fix != 1)) return SINCOS_ERR_INVALID_ARGUMENT;
        mp = make_params(method->ss, method->n_ss, method->cc, method->n_cc, method->doublings);
    } else if (variant == -1) {
        shape = -2;                      // negative control
    } else if (variant != SINCOS_NORMALIZED && variant != SINCOS_RENORMALIZED) {
        return SINCOS_ERR_INVALID_ARGUMENT;
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((e = cudaMemsetAsync(mismatch_dev, 0, sizeof(unsigned long long), s)) != cudaSuccess) return cuda_fail(e);
    e = launch_packcheck(variant, shape, fix, method ? &mp : nullptr, static_cast<unsigned>(sm_count(dev)) * 16,
                         mismatch_dev, s);
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

sincos_status_t sincos_debug_reciprocal(const float *d_dev, float *out_dev, size_t n, void *stream) {
    if (n == 0) return SINCOS_OK;
    if (d_dev == nullptr || out_dev == nullptr || !aligned(d_dev, 4) || !aligned(out_dev, 4))
        return SINCOS_ERR_INVALID_ARGUMENT;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    const size_t want = (n + 255) / 256;
    const size_t cap = static_cast<size_t>(sm_count(dev)) * 8;
    e = launch_rcp(static_cast<unsigned>(want < cap ? want : cap), 256, d_dev, out_dev, n,
                   static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SINCOS_OK;
}

const char *sincos_status_string(sincos_status_t s) {
    switch (s) {
    case SINCOS_OK: return "ok";
    case SINCOS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SINCOS_ERR_OVERLAP: return "output buffers overlap each other or the input";
    case SINCOS_ERR_CUDA: return "CUDA error (see sincos_last_cuda_error)";
    case SINCOS_ERR_NCCL: return "NCCL error (see sincos_last_nccl_error)";
    default: return "unknown status";
    }
}

int sincos_last_cuda_error(void) { return g_last_cuda_error; }

// internal (hidden): lets sincos_shard.cu record a CUDA error the same way
sincos_status_t sincos_last_error_set(int e) { return cuda_fail(static_cast<cudaError_t>(e)); }

const char *sincos_version(void) { return "sincos_pairs 0.1 (sm_100a; arXiv cs/0406049)"; }

uint64_t sincos_launch_count(void) { return g_launches.load(); }

}  // extern "C"
