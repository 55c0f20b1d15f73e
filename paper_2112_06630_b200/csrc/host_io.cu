// Host <-> device transfers of the host-pointer entry points (knng_cuda_run,
// knng_cuda_nndescent_l2, knng_cuda_bruteforce ...): the rows in, the graph out.
//
// A caller of the reference's API hands over pageable memory (std::vector
// rows, KnnGraph vectors: descent.hpp:193, graph.hpp:20-31).  A pageable
// cudaMemcpyAsync goes through the driver's own small bounce buffer, one
// thread, ~10 GB/s into freshly mapped pages — on C5's 180 MB graph that was
// 33 ms of a 620 ms end-to-end build.  Here pageable buffers go through a
// ring of pinned slots instead: the copy engine fills (or drains) slot i
// while up to 8 host threads memcpy the slots before it, so the transfer runs
// at the PCIe rate.  Pinned (page-locked or registered) buffers are copied
// directly.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace knng_cuda {
namespace {

constexpr size_t kRingBytes = size_t(64) << 20;  // pinned, allocated once
constexpr uint32_t kMaxSlots = 64;
// 1 MiB slots by default (KNNG_STAGE_KB overrides; A/B only): small enough
// that a 12 MB graph spreads over all workers
size_t slot_bytes() {
    static const size_t b = [] {
        const char* v = getenv("KNNG_STAGE_KB");
        size_t kb = v ? size_t(atol(v)) : 1024;
        if (kb < 64) kb = 64;
        if (kb * 1024 * kMaxSlots < kRingBytes) kb = kRingBytes / kMaxSlots / 1024;
        if (kb * 1024 > kRingBytes) kb = kRingBytes / 1024;
        return kb * 1024;
    }();
    return b;
}
constexpr uint32_t kMaxWorkers = 8;
constexpr size_t kDirectBelow = size_t(2) << 20;  // small pageable copies: plain async copy

struct Ring {
    std::mutex mu;  // one staged transfer at a time per process
    unsigned char* host = nullptr;
    cudaEvent_t ev[kMaxDevices][kMaxSlots] = {};
};

Ring& ring() {
    static Ring r;
    return r;
}

struct Chunk {
    unsigned char* host;
    unsigned char* dev;
    size_t bytes;
};

std::vector<Chunk> split(const std::vector<HostSeg>& segs) {
    const size_t slot_b = slot_bytes();
    std::vector<Chunk> out;
    for (const HostSeg& g : segs)
        for (size_t off = 0; off < g.bytes; off += slot_b)
            out.push_back({static_cast<unsigned char*>(g.host) + off,
                           static_cast<unsigned char*>(g.dev) + off,
                           g.bytes - off < slot_b ? g.bytes - off : slot_b});
    return out;
}

uint32_t worker_count(size_t chunks) {
    uint32_t hw = std::thread::hardware_concurrency();
    hw = hw > 1 ? hw / 2 : 1;
    uint32_t t = hw < kMaxWorkers ? hw : kMaxWorkers;
    return chunks < t ? uint32_t(chunks) : t;
}

void spin_until(const std::atomic<int>& a, int at_least, const std::atomic<bool>& failed) {
    while (a.load(std::memory_order_acquire) < at_least && !failed.load(std::memory_order_relaxed))
        std::this_thread::yield();
}

// The pinned ring and this device's slot events (created on first use).
Ring& acquire(std::unique_lock<std::mutex>& lk) {
    Ring& r = ring();
    lk = std::unique_lock<std::mutex>(r.mu);
    if (!r.host) {
        void* p = nullptr;
        check_launch(cudaHostAlloc(&p, kRingBytes, cudaHostAllocPortable),
                     "pinned staging ring");
        r.host = static_cast<unsigned char*>(p);
    }
    const int d = current_device();
    if (!r.ev[d][0])
        for (uint32_t i = 0; i < kMaxSlots; ++i)
            check_launch(cudaEventCreateWithFlags(&r.ev[d][i], cudaEventDisableTiming));
    return r;
}

// Runs `issue(i)` on this thread for every chunk in order and `host(j)` on the
// workers; the state machine is described at each call site.
template <typename Issue, typename Host>
void pipeline(size_t nchunks, Issue&& issue, Host&& host) {
    std::atomic<size_t> next{0};
    std::atomic<bool> failed{false};
    std::string err;
    std::mutex err_mu;
    const int dev = current_device();
    auto work = [&] {
        try {
            check_launch(cudaSetDevice(dev));
            for (size_t j = next.fetch_add(1); j < nchunks && !failed; j = next.fetch_add(1))
                host(j, failed);
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> g(err_mu);
            if (err.empty()) err = e.what();
            failed = true;
        }
    };
    std::vector<std::thread> pool;
    const uint32_t nw = worker_count(nchunks);
    for (uint32_t w = 0; w < nw; ++w) pool.emplace_back(work);
    try {
        for (size_t i = 0; i < nchunks && !failed; ++i) issue(i, failed);
    } catch (const std::exception& e) {
        std::lock_guard<std::mutex> g(err_mu);
        if (err.empty()) err = e.what();
        failed = true;
    }
    for (auto& t : pool) t.join();
    if (failed) throw std::runtime_error(err);
}

bool all_pinned(const std::vector<HostSeg>& segs, size_t& pageable_bytes) {
    pageable_bytes = 0;
    bool pinned = true;
    for (const HostSeg& g : segs)
        if (g.bytes && !host_is_pinned(g.host)) {
            pinned = false;
            pageable_bytes += g.bytes;
        }
    return pinned;
}

}  // namespace

bool host_is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void copy_from_host(const std::vector<HostSeg>& segs, cudaStream_t s) {
    size_t pageable = 0;
    if (all_pinned(segs, pageable) || pageable < kDirectBelow) {
        for (const HostSeg& g : segs)
            if (g.bytes)
                check_launch(cudaMemcpyAsync(g.dev, g.host, g.bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    std::unique_lock<std::mutex> lk;
    Ring& r = acquire(lk);
    cudaEvent_t* ev = r.ev[current_device()];
    const size_t slot_b = slot_bytes();
    const uint32_t nslots = uint32_t(kRingBytes / slot_b);
    const std::vector<Chunk> ch = split(segs);
    // state[j]: 0 empty, 1 staged in slot j % nslots by a worker, 2 copy issued
    // (slot event recorded).  A worker reuses slot j % nslots only after the
    // copy of chunk j - nslots out of it completed.
    std::vector<std::atomic<int>> state(ch.size());
    for (auto& a : state) a.store(0);
    pipeline(
        ch.size(),
        [&](size_t i, std::atomic<bool>& failed) {
            spin_until(state[i], 1, failed);
            if (failed) return;
            const uint32_t slot = uint32_t(i % nslots);
            check_launch(cudaMemcpyAsync(ch[i].dev, r.host + slot * slot_b, ch[i].bytes,
                                         cudaMemcpyHostToDevice, s));
            check_launch(cudaEventRecord(ev[slot], s));
            state[i].store(2, std::memory_order_release);
        },
        [&](size_t j, std::atomic<bool>& failed) {
            const uint32_t slot = uint32_t(j % nslots);
            if (j >= nslots) {
                spin_until(state[j - nslots], 2, failed);
                if (failed) return;
                check_launch(cudaEventSynchronize(ev[slot]));
            }
            std::memcpy(r.host + slot * slot_b, ch[j].host, ch[j].bytes);
            state[j].store(1, std::memory_order_release);
        });
    // the ring is reused by the next transfer: its last copies must be done
    for (uint32_t i = 0; i < nslots && i < ch.size(); ++i)
        check_launch(cudaEventSynchronize(ev[i]));
}

void copy_to_host(const std::vector<HostSeg>& segs, cudaStream_t s) {
    size_t pageable = 0;
    if (all_pinned(segs, pageable) || pageable < kDirectBelow) {
        for (const HostSeg& g : segs)
            if (g.bytes)
                check_launch(cudaMemcpyAsync(g.host, g.dev, g.bytes, cudaMemcpyDeviceToHost, s));
        check_launch(cudaStreamSynchronize(s));
        return;
    }
    std::unique_lock<std::mutex> lk;
    Ring& r = acquire(lk);
    cudaEvent_t* ev = r.ev[current_device()];
    const size_t slot_b = slot_bytes();
    const uint32_t nslots = uint32_t(kRingBytes / slot_b);
    const std::vector<Chunk> ch = split(segs);
    // state[j]: 0 not issued, 1 copy into slot j % nslots issued (event
    // recorded), 2 drained to the caller's buffer.  Chunk i reuses its slot
    // only after chunk i - nslots was drained.
    std::vector<std::atomic<int>> state(ch.size());
    for (auto& a : state) a.store(0);
    pipeline(
        ch.size(),
        [&](size_t i, std::atomic<bool>& failed) {
            if (i >= nslots) {
                spin_until(state[i - nslots], 2, failed);
                if (failed) return;
            }
            const uint32_t slot = uint32_t(i % nslots);
            check_launch(cudaMemcpyAsync(r.host + slot * slot_b, ch[i].dev, ch[i].bytes,
                                         cudaMemcpyDeviceToHost, s));
            check_launch(cudaEventRecord(ev[slot], s));
            state[i].store(1, std::memory_order_release);
        },
        [&](size_t j, std::atomic<bool>& failed) {
            spin_until(state[j], 1, failed);
            if (failed) return;
            const uint32_t slot = uint32_t(j % nslots);
            check_launch(cudaEventSynchronize(ev[slot]));
            std::memcpy(ch[j].host, r.host + slot * slot_b, ch[j].bytes);
            state[j].store(2, std::memory_order_release);
        });
}

}  // namespace knng_cuda
