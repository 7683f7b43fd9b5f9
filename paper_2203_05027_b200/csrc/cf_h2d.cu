// Host -> device upload of pageable host arrays through pinned staging buffers.
//
// solve() receives numpy arrays (pageable memory); a plain cudaMemcpyAsync from
// pageable memory runs at ~11 GB/s on the B200 boxes (one driver thread copies
// into its own bounce buffer). Here T worker threads each own two pinned
// staging buffers and a stream: a worker memcpy's its next chunk into the free
// buffer while the DMA engine drains the other one, so the CPU copies run in
// parallel and overlap the PCIe transfer. The staging buffers are cached for the
// process (allocated on first use), like torch's pinned-memory cache.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "cf_common.h"

namespace cf {
namespace {

constexpr size_t kChunk = 8u << 20;   // bytes per staged chunk

struct Worker {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaStream_t stream = nullptr;
};

struct Pool {
    std::mutex mu;
    std::vector<Worker> w;
    int device = -1;
    bool failed = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

int n_threads() {
    const char* e = getenv("CF_H2D_THREADS");
    int t = e ? atoi(e) : 0;
    if (t <= 0) {
        const unsigned hw = std::thread::hardware_concurrency();
        t = (int)std::min<unsigned>(16u, hw ? hw : 4u);
    }
    return std::max(1, std::min(t, 32));
}

bool ensure_pool(Pool& P, int threads) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    if (P.failed) return false;
    if (P.device == dev && (int)P.w.size() >= threads) return true;
    if (P.device != dev) P.w.clear();   // (buffers of another device are leaked; one device per process in practice)
    P.device = dev;
    while ((int)P.w.size() < threads) {
        Worker w;
        bool ok = cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking) == cudaSuccess;
        for (int b = 0; b < 2 && ok; ++b) {
            ok = cudaMallocHost(&w.buf[b], kChunk) == cudaSuccess &&
                 cudaEventCreateWithFlags(&w.done[b], cudaEventDisableTiming) == cudaSuccess;
        }
        if (!ok) {
            cudaGetLastError();
            P.failed = true;
            return false;
        }
        P.w.push_back(w);
    }
    return true;
}

}  // namespace

// Copy `jobs` (device dst, host src, bytes) and make `stream` wait for them.
// Falls back to plain cudaMemcpyAsync when pinned staging is unavailable.
int h2d_staged(const std::vector<H2DJob>& jobs, cudaStream_t stream) {
    size_t total = 0;
    for (const auto& j : jobs) total += j.bytes;
    Pool& P = pool();
    std::lock_guard<std::mutex> lock(P.mu);
    const int threads = n_threads();
    if (total < (size_t)4 * kChunk || !ensure_pool(P, threads)) {
        for (const auto& j : jobs)
            if (j.bytes) CF_CUDA(cudaMemcpyAsync(j.dst, j.src, j.bytes, cudaMemcpyHostToDevice, stream));
        return CF_OK;
    }
    // chunk list (job, offset, length), dealt to workers round-robin
    struct Piece {
        const H2DJob* job;
        size_t off, len;
    };
    std::vector<Piece> pieces;
    for (const auto& j : jobs)
        for (size_t off = 0; off < j.bytes; off += kChunk) pieces.push_back({&j, off, std::min(kChunk, j.bytes - off)});
    // the staging streams must not start before earlier work on `stream` (the destinations may be in use)
    cudaEvent_t start;
    CF_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CF_CUDA(cudaEventRecord(start, stream));
    std::atomic<int> err{0};
    std::vector<std::thread> th;
    th.reserve(threads);
    for (int t = 0; t < threads; ++t) {
        th.emplace_back([&, t]() {
            Worker& w = P.w[t];
            if (cudaSetDevice(P.device) != cudaSuccess) err = 1;   // a new thread starts on device 0
            // the buffers may still feed the previous call's copies
            if (cudaStreamSynchronize(w.stream) != cudaSuccess || cudaStreamWaitEvent(w.stream, start, 0) != cudaSuccess)
                err = 1;
            int k = 0;
            for (size_t i = t; i < pieces.size() && !err; i += threads, ++k) {
                const int b = k & 1;
                if (k >= 2 && cudaEventSynchronize(w.done[b]) != cudaSuccess) {
                    err = 1;
                    break;
                }
                const Piece& pc = pieces[i];
                std::memcpy(w.buf[b], static_cast<const char*>(pc.job->src) + pc.off, pc.len);
                if (cudaMemcpyAsync(static_cast<char*>(pc.job->dst) + pc.off, w.buf[b], pc.len,
                                    cudaMemcpyHostToDevice, w.stream) != cudaSuccess ||
                    cudaEventRecord(w.done[b], w.stream) != cudaSuccess) {
                    err = 1;
                    break;
                }
            }
        });
    }
    for (auto& x : th) x.join();
    cudaEventDestroy(start);
    if (err) {
        set_error("h2d_staged: CUDA error during the staged upload");
        return CF_ECUDA;
    }
    // `stream` waits for every worker's last copy; the buffers are reusable once
    // those complete (the next call synchronises on the same events)
    for (int t = 0; t < threads; ++t) {
        cudaEvent_t ev;
        CF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CF_CUDA(cudaEventRecord(ev, P.w[t].stream));
        CF_CUDA(cudaStreamWaitEvent(stream, ev, 0));
        CF_CUDA(cudaEventDestroy(ev));
    }
    return CF_OK;
}

namespace {
std::mutex g_scratch_mu;
void* g_scratch = nullptr;
size_t g_scratch_bytes = 0;
}  // namespace

PinnedScratch::PinnedScratch() { g_scratch_mu.lock(); }
PinnedScratch::~PinnedScratch() { g_scratch_mu.unlock(); }
void* PinnedScratch::get(size_t bytes) {
    if (bytes <= g_scratch_bytes) return g_scratch;
    if (g_scratch) cudaFreeHost(g_scratch);
    g_scratch = nullptr;
    g_scratch_bytes = 0;
    const size_t want = bytes + bytes / 4;   // some headroom for the next, larger plan
    if (cudaMallocHost(&g_scratch, want) != cudaSuccess) {
        cudaGetLastError();
        g_scratch = nullptr;
        return nullptr;
    }
    g_scratch_bytes = want;
    return g_scratch;
}

}  // namespace cf
