// Host orchestrator and C-ABI of libknng_cuda.so (declared in include/knng_cuda.h).
//
// knng::run (reference descent.hpp:193-255) re-designed for one B200:
//   init_random -> [ indegree -> sample -> finalize -> join -> (reorder once) ]*
// with every stage a device kernel on one stream, and one 32-byte
// device->host read of the iteration counters per iteration for the
// termination test `changes < delta * n * k` (descent.hpp:215-216, 242).
// Seeds follow the reference exactly: a std::mt19937_64 master seeded with
// params.seed hands out the init seed, then one seed per iteration
// (descent.hpp:201-221); the device kernels key Philox streams with them.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "../../include/knng_cuda.h"
#include "kernels.cuh"

using namespace knng_cuda;

#include <csignal>
#include <execinfo.h>
#include <unistd.h>

namespace {

// KNNG_SEGV_TRACE=1: print a native backtrace on SIGSEGV (diagnostics; map
// the addresses with addr2line -e libknng_cuda.so)
void segv_trace(int sig) {
    void* frames[64];
    const int nf = backtrace(frames, 64);
    const char msg[] = "knng_cuda: fatal signal, native backtrace:\n";
    (void)!write(2, msg, sizeof(msg) - 1);
    backtrace_symbols_fd(frames, nf, 2);
    signal(sig, SIG_DFL);
    raise(sig);
}
struct SegvTraceInstaller {
    SegvTraceInstaller() {
        const char* v = getenv("KNNG_SEGV_TRACE");
        if (v && v[0] == '1') signal(SIGSEGV, segv_trace);
    }
} g_segv_trace_installer;

thread_local std::string g_err;

struct Status {
    int code;
    std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg) { throw Status{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    const int code =
        e == cudaErrorMemoryAllocation ? KNNG_CUDA_OUT_OF_MEMORY : KNNG_CUDA_CUDA_ERROR;
    cudaGetLastError();  // clear sticky-free errors
    raise(code, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) check_cuda((x), #x)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return KNNG_CUDA_OK;
    } catch (const Status& s) {
        g_err = s.msg;
        return s.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KNNG_CUDA_CUDA_ERROR;
    }
}

// Stream-ordered allocations from a per-device pool that keeps freed memory
// (release threshold = max) so repeated builds do not pay cudaMalloc again.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t pool_for(int device) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    if (device < 0 || device >= 64) raise(KNNG_CUDA_INVALID_ARGUMENT, "device ordinal out of range");
    if (!g_pools[device]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        CK(cudaMemPoolCreate(&g_pools[device], &props));
        uint64_t threshold = ~0ull;
        CK(cudaMemPoolSetAttribute(g_pools[device], cudaMemPoolAttrReleaseThreshold, &threshold));
    }
    return g_pools[device];
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void alloc(size_t count, cudaMemPool_t pool, cudaStream_t stream) {
        s = stream;
        CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T),
                                   pool, stream));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int device) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            raise(KNNG_CUDA_CUDA_ERROR, "no CUDA device available (this library has no CPU path)");
        }
        if (device < 0 || device >= count) raise(KNNG_CUDA_INVALID_ARGUMENT, "device ordinal out of range");
        CK(cudaGetDevice(&prev));
        CK(cudaSetDevice(device));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// The caller's stream, or this host thread's cached library stream for the
// current device.  Reusing one stream per (thread, device) keeps the pool's
// freed blocks immediately reusable by the next call (stream-ordered reuse)
// instead of growing the pool for every new stream.
struct StreamHolder {
    cudaStream_t s = nullptr;
    explicit StreamHolder(void* user) {
        if (user) {
            s = static_cast<cudaStream_t>(user);
            return;
        }
        thread_local cudaStream_t cached[64] = {};
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (dev < 0 || dev >= 64) raise(KNNG_CUDA_INVALID_ARGUMENT, "device ordinal out of range");
        if (!cached[dev]) CK(cudaStreamCreateWithFlags(&cached[dev], cudaStreamNonBlocking));
        s = cached[dev];
    }
    ~StreamHolder() { cudaStreamSynchronize(s); }
};

// Per-kernel CUDA-event timing on the library stream (params.profile).
struct KernelTimer {
    bool on;
    cudaStream_t s;
    std::vector<cudaEvent_t> pool;       // reused across flushes
    struct Open {
        int kernel;
        size_t first;  // first event index
        uint32_t tag;  // iteration
    };
    std::vector<Open> open;
    size_t used = 0;
    uint32_t tag = 0;  // iteration of the launches being recorded
    knng_cuda_metrics* m;
    KernelTimer(bool enabled, cudaStream_t stream, knng_cuda_metrics* metrics)
        : on(enabled && metrics), s(stream), m(metrics) {}
    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    int begin(int kernel) {
        if (!on) return -1;
        const size_t i = used;
        CK(cudaEventRecord(next(), s));
        next();
        open.push_back({kernel, i, tag});
        return int(open.size()) - 1;
    }
    void end(int h) {
        if (h < 0) return;
        CK(cudaEventRecord(pool[open[size_t(h)].first + 1], s));
    }
    double last_join_ms = 0.0;         // distance-kernel time of the flushed launches
    std::vector<double> join_ms_by_tag;  // ... per iteration
    void flush() {  // after a stream sync
        last_join_ms = 0.0;
        for (auto& e : open) {
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, pool[e.first], pool[e.first + 1]));
            m->kernel_ms[e.kernel] += ms;
            m->kernel_launches[e.kernel] += 1;
            if (e.kernel == KNNG_CUDA_KERNEL_JOIN) {
                last_join_ms += ms;
                if (join_ms_by_tag.size() <= e.tag) join_ms_by_tag.resize(e.tag + 1, 0.0);
                join_ms_by_tag[e.tag] += ms;
            }
        }
        open.clear();
        used = 0;
    }
    double join_ms_of(uint32_t t) const { return t < join_ms_by_tag.size() ? join_ms_by_tag[t] : 0.0; }
    ~KernelTimer() {
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

void validate_shape(uint32_t n, uint32_t d, uint32_t k) {
    if (n < 2) raise(KNNG_CUDA_INVALID_ARGUMENT, "Dataset: need at least 2 points");
    if (d < 1) raise(KNNG_CUDA_INVALID_ARGUMENT, "Dataset: need at least 1 dimension");
    if (n >= (1u << 31)) raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports n < 2^31");
    if (k < 2) raise(KNNG_CUDA_INVALID_ARGUMENT, "k must be at least 2");
    if (k > KNNG_CUDA_MAX_K) raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports k <= 32");
    if (k >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "k must be smaller than n");
}

void validate_params(uint32_t n, uint32_t d, const knng_cuda_params& p) {
    // RunParams::validate (descent.hpp:29-35) and run's n > k (descent.hpp:197)
    if (p.k < 2) raise(KNNG_CUDA_INVALID_ARGUMENT, "RunParams: k must be at least 2");
    if (p.max_candidates < p.k)
        raise(KNNG_CUDA_INVALID_ARGUMENT, "RunParams: max_candidates must be at least k");
    if (!(p.termination_delta > 0.0 && p.termination_delta < 1.0))
        raise(KNNG_CUDA_INVALID_ARGUMENT, "RunParams: termination_delta must be in (0,1)");
    if (n <= p.k) raise(KNNG_CUDA_INVALID_ARGUMENT, "run: need n > k");
    if (p.max_candidates > KNNG_CUDA_MAX_CANDIDATES)
        raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports max_candidates <= 64");
    validate_shape(n, d, p.k);
}

inline uint32_t padded_stride(uint32_t d) { return (d + 7u) / 8u * 8u; }

// All device state of one build on one GPU.
struct Engine {
    uint32_t n, d, stride, k, cap;
    cudaStream_t s;
    cudaMemPool_t pool;
    DevBuf<float> data, maxd;
    DevBuf<uint64_t> keys;
    DevBuf<uint32_t> flags, indeg, cand, raw_new, raw_old, nc, oc, active;
    DevBuf<uint64_t> dsz, doff;
    DevBuf<float> cmax;
    DevBuf<uint4> arec;
    DevBuf<uint32_t> hubs;
    DevBuf<uint32_t> revcnt, roff, rcur;
    DevBuf<unsigned char> scan_tmp;
    size_t scan_bytes = 0;
    // grow-only per-iteration buffers: reverse index and distance blocks
    DevBuf<uint64_t> rev;
    DevBuf<uint64_t> dblocks;
    int filter = 1;  // join proposals prefiltered by the row maxima (0: keep all)
    bool det = false;            // deterministic mode (CandView::det)
    bool indeg_inc = false;      // merges maintain indeg (CandView::indeg_inc)
    DevBuf<unsigned long long> rawlist;  // its raw sampled lists (keys), n x 4 cap
    size_t rev_cap = 0, d_cap = 0;
    DevBuf<IterCounters> ctr;    // slot 0, or one slot per iteration (ensure_slots)
    IterCounters* cur = nullptr;  // the slot the kernels of the current iteration use
    uint32_t slots = 1;
    IterCounters* h_ctr = nullptr;  // pinned: h_ctr[i] mirrors slot i
    // tensor-core screened join (join_tc.cu): per-row norms for its bound,
    // computed on first use and after the data is permuted
    DevBuf<float> nrm2, nrmu;
    DevBuf<uint4> ovf;           // its overflow list (nodes too large for its arena)
    DevBuf<IterCounters> octr;   // and that list's counters
    bool norms_valid = false;
    // byte-valued data (join_u8.cu): lane-major byte copy and lane norms,
    // decided on first use and after the data is permuted
    DevBuf<uint8_t> packed;
    DevBuf<int32_t> lnorm;
    DevBuf<uint32_t> u8_flag;
    int u8_state = -1;  // -1 unknown, 0 not eligible, 1 packed
    // long rows (join_gl.cu): lane-major copy of the data, made on first use
    // and after the data is permuted
    DevBuf<float> dl;
    bool dl_valid = false;
    uint32_t iteration = 0;  // the running iteration (1-based; 0 = fixed-state entry)
    uint64_t h2d = 0, d2h = 0;

    uint32_t lo = 0, hi = 0;  // owned rows (multi-GPU); [0, n) otherwise
    uint32_t rows_alloc = 0;  // graph rows allocated (>= n: equal shards for allgather)

    Engine(int device, uint32_t n_, uint32_t d_, uint32_t k_, uint32_t cap_, cudaStream_t stream,
           uint32_t rows = 0)
        : n(n_), d(d_), stride(padded_stride(d_)), k(k_), cap(cap_), s(stream) {
        pool = pool_for(device);
        lo = 0;
        hi = n;
        rows_alloc = rows > n ? rows : n;
        data.alloc(size_t(n) * stride, pool, s);
        keys.alloc(size_t(rows_alloc) * k, pool, s);
        flags.alloc(rows_alloc, pool, s);
        maxd.alloc(rows_alloc, pool, s);
        indeg.alloc(n, pool, s);
        ctr.alloc(1, pool, s);
        if (cap) {
            cand.alloc(size_t(n) * 2 * cap, pool, s);
            raw_new.alloc(n, pool, s);
            raw_old.alloc(n, pool, s);
            nc.alloc(n, pool, s);
            oc.alloc(n, pool, s);
            active.alloc(n, pool, s);
            dsz.alloc(n, pool, s);
            doff.alloc(n, pool, s);
            // pool memory is recycled: rows outside a shard's range are never
            // written, so start from zero
            CK(cudaMemsetAsync(dsz.p, 0, sizeof(uint64_t) * n, s));
            cmax.alloc(size_t(n) * 2 * cap, pool, s);
            arec.alloc(n, pool, s);
            hubs.alloc(n, pool, s);
            revcnt.alloc(n, pool, s);
            roff.alloc(n, pool, s);
            rcur.alloc(n, pool, s);
            scan_bytes = join_scan_scratch(n);
            scan_tmp.alloc(scan_bytes, pool, s);
            // every active list names at most 2 cap candidates
            // (KNNG_TEST_DWORDS: a small initial proposal buffer, so tests
            // exercise the overflow -> grow -> rerun path)
            const char* tv = getenv("KNNG_TEST_DWORDS");
            reserve_join(uint64_t(n) * 2 * cap,
                         tv ? uint64_t(atoll(tv)) : uint64_t(n) * 4 * k * k);
        }
        cur = ctr.p;
        h_ctr = pinned_slots(1);
        CK(cudaMemsetAsync(ctr.p, 0, sizeof(IterCounters), s));
    }
    // pinned counter slots: each Engine holds its own buffer, recycled
    // through a per-thread free list (cudaMallocHost is slow); a buffer is
    // never freed while an Engine still points at it
    struct Pinned {
        IterCounters* p = nullptr;
        size_t n = 0;
    };
    static std::vector<Pinned>& pinned_free() {
        thread_local std::vector<Pinned> list;
        return list;
    }
    Pinned pin;
    IterCounters* pinned_slots(size_t count) {
        count = std::max<size_t>(count, 64);
        if (pin.n >= count) return pin.p;
        release_pinned();
        auto& fl = pinned_free();
        for (size_t i = 0; i < fl.size(); ++i)
            if (fl[i].n >= count) {
                pin = fl[i];
                fl.erase(fl.begin() + long(i));
                return pin.p;
            }
        CK(cudaMallocHost(reinterpret_cast<void**>(&pin.p), sizeof(IterCounters) * count));
        pin.n = count;
        return pin.p;
    }
    void release_pinned() {
        if (pin.p) pinned_free().push_back(pin);
        pin = Pinned{};
    }
    // one zeroed counter slot per iteration (slot i = iteration i), so that
    // iterations can be enqueued ahead of the host's termination test
    void ensure_slots(uint32_t count) {
        if (count > slots) {
            ctr.~DevBuf();
            new (&ctr) DevBuf<IterCounters>();
            ctr.alloc(count, pool, s);
            slots = count;
        }
        CK(cudaMemsetAsync(ctr.p, 0, sizeof(IterCounters) * count, s));
        cur = ctr.p;
        h_ctr = pinned_slots(count);
    }
    ~Engine() {
        h_ctr = nullptr;
        release_pinned();  // back to this thread's free list for the next Engine
    }

    GraphView gv() const {
        return GraphView{data.p, n, k, stride, keys.p, flags.p, maxd.p, lo, hi};
    }
    CandView cv() const {
        return CandView{cap,   cand.p,   raw_new.p, raw_old.p, nc.p, oc.p, dsz.p,
                        doff.p, revcnt.p, roff.p,   rcur.p,    rev.p, dblocks.p, filter,
                        cmax.p, arec.p, hubs.p, rawlist.p, det ? 1 : 0,
                        indeg_inc ? indeg.p : nullptr};
    }

    void reserve_join(uint64_t rev_entries, uint64_t dwords) {
        if (rev_entries > rev_cap) {
            rev.~DevBuf();
            new (&rev) DevBuf<uint64_t>();
            rev_cap = rev_entries + rev_entries / 4 + 1024;
            rev.alloc(rev_cap, pool, s);
        }
        if (dwords > d_cap) {
            dblocks.~DevBuf();
            new (&dblocks) DevBuf<uint64_t>();
            d_cap = dwords + dwords / 4 + 4096;
            dblocks.alloc(d_cap, pool, s);
        }
    }

    // Rows padded to ceil8(d) with zeros (dataset.hpp:72-77).
    // Host rows cross PCIe as one contiguous copy (a pitched host-to-device
    // copy of 3136-byte rows ran at 34 GB/s against 57 for a flat one, C2) and
    // are padded on the device.
    void upload(const float* src, bool src_on_device) {
        const size_t bytes = sizeof(float) * size_t(n) * d;
        if (stride != d) CK(cudaMemsetAsync(data.p, 0, sizeof(float) * size_t(n) * stride, s));
        if (src_on_device) {
            CK(cudaMemcpy2DAsync(data.p, sizeof(float) * stride, src, sizeof(float) * d,
                                 sizeof(float) * d, n, cudaMemcpyDeviceToDevice, s));
            return;
        }
        h2d += bytes;
        if (stride == d) {
            copy_from_host({{const_cast<float*>(src), data.p, bytes}}, s);
            return;
        }
        DevBuf<float> flat;
        flat.alloc(size_t(n) * d, pool, s);
        copy_from_host({{const_cast<float*>(src), flat.p, bytes}}, s);
        CK(cudaMemcpy2DAsync(data.p, sizeof(float) * stride, flat.p, sizeof(float) * d,
                             sizeof(float) * d, n, cudaMemcpyDeviceToDevice, s));
    }

    // the current slot's counters -> h_ctr[0]
    void read_counters() {
        CK(cudaMemcpyAsync(h_ctr, cur, sizeof(IterCounters), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        d2h += sizeof(IterCounters);
    }

    // selection: in-degree, turbo sampling, finalize (dedup, flag_consumed, active list)
    void select(uint64_t seed, KernelTimer& timer) {
        const GraphView g = gv();
        const CandView c = cv();
        int h = timer.begin(KNNG_CUDA_KERNEL_DEGREE);
        if (indeg_inc)
            launch_indegree_gated(g, indeg.p, cur, s);  // recount only when cur->recount
        else
            launch_indegree(g, indeg.p, s, cur);
        launch_reset_raw(c, n, s, cur);
        timer.end(h);
        h = timer.begin(KNNG_CUDA_KERNEL_SAMPLE);
        launch_sample(g, c, indeg.p, seed, s, cur, seed);
        timer.end(h);
        h = timer.begin(KNNG_CUDA_KERNEL_FINALIZE);
        launch_finalize(g, c, active.p, cur, s, seed);
        timer.end(h);
        CK(cudaGetLastError());
    }

    // The local join after finalize/bookkeeping, with no host round trip:
    // block offsets, a device-side capacity check, the reverse index, then
    // the distance and merge stages.  Ends with the iteration's one counter
    // read; when the distance blocks outgrew their buffer (the stages skipped
    // themselves) the buffer grows and the stages run again.
    void join(KernelTimer& timer, bool distances_only = false) {
        join_enqueue(timer, distances_only);
        read_counters();
        if (h_ctr->screened && getenv("KNNG_TC_STATS"))
            fprintf(stderr, "[knng] iteration %u screened join: %llu pairs, %llu exact (%.4f)\n",
                    iteration, h_ctr->screened, h_ctr->survivors,
                    double(h_ctr->survivors) / double(h_ctr->screened));
        if (h_ctr->overflow) {
            reserve_join(h_ctr->rev, h_ctr->dwords);
            CK(cudaMemsetAsync(&cur->overflow, 0, sizeof(uint32_t), s));
            join_stages(timer, distances_only);
            read_counters();
        }
    }

    // the join's launches, no host round trip
    void join_enqueue(KernelTimer& timer, bool distances_only = false) {
        int h = timer.begin(KNNG_CUDA_KERNEL_INDEX);
        launch_join_offsets(cv(), n, lo, hi, scan_tmp.p, scan_bytes, s);
        timer.end(h);
        join_stages(timer, distances_only);
    }

    void join_stages(KernelTimer& timer, bool distances_only) {
        launch_check_capacity(cur, d_cap, s);
        int h = timer.begin(KNNG_CUDA_KERNEL_INDEX);
        launch_scatter_rev(cv(), active.p, cur, n, n, s);
        timer.end(h);
        h = timer.begin(KNNG_CUDA_KERNEL_JOIN);
        if (use_u8_join()) {
            if (use_u8_tc())
                launch_join_u8_tc(u8_map, cv(), cur, n, lnorm.p, s);
            else
                launch_join_u8(gv(), cv(), cur, n, packed.p, lnorm.p, s);
        } else if (use_gl_join()) {
            if (!dl_valid) {
                if (!dl.p) dl.alloc(size_t(n + 1) * gl_row_floats(stride), pool, s);
                launch_gl_pack(data.p, n, stride, dl.p, s);
                dl_valid = true;
            }
            launch_join_gl(cv(), dl.p, n, stride, cur, n, s);
        } else if (use_screened_join(distances_only)) {
            if (!norms_valid) {
                if (!nrm2.p) {
                    nrm2.alloc(n, pool, s);
                    nrmu.alloc(n, pool, s);
                    ovf.alloc(n, pool, s);
                    octr.alloc(1, pool, s);
                }
                launch_row_norms(data.p, n, stride, nrm2.p, nrmu.p, s);
                norms_valid = true;
            }
            launch_join_tc(gv(), cv(), cur, n, nrm2.p, nrmu.p, ovf.p, octr.p, s);
        } else if (use_t5_join()) {
            launch_join5(gv(), cv(), cur, n, s);
        } else {
            launch_join_distances(gv(), cv(), active.p, cur, n, s);
        }
        timer.end(h);
        CK(cudaGetLastError());
        if (distances_only) return;
        h = timer.begin(KNNG_CUDA_KERNEL_MERGE);
        launch_join_merge(gv(), cv(), cur, s);
        timer.end(h);
        CK(cudaGetLastError());
    }

    // Byte-valued data takes the integer tensor-core join (join_u8.cu,
    // bit-identical); KNNG_JOIN_U8=0 forces the FP32 kernel (A/B).
    bool use_u8_join() {
        const char* v = getenv("KNNG_JOIN_U8");
        if (v && v[0] == '0') return false;
        if (u8_state < 0) {
            if (!u8_flag.p) u8_flag.alloc(1, pool, s);
            u8_state = u8_eligible(data.p, n, stride, u8_flag.p, s) ? 1 : 0;
            if (u8_state == 1) {
                if (!packed.p) {
                    packed.alloc(size_t(n) * 8 * u8_lane_bytes(stride), pool, s);
                    lnorm.alloc(size_t(n) * 8, pool, s);
                }
                launch_u8_pack(data.p, n, stride, packed.p, lnorm.p, s);
            }
        }
        return u8_state == 1;
    }

    // Byte-valued data on tcgen05 (join_u8_tc.cu) when its shapes are
    // supported: KNNG_U8_TC=1 / 0 forces it on / off.  The tensor map of the
    // byte copy is made once per packing.
    alignas(64) unsigned char u8_map[128] = {};
    const unsigned char* u8_map_for = nullptr;
    bool use_u8_tc() {
        const char* v = getenv("KNNG_U8_TC");
        const bool want = v ? v[0] == '1' : false;
        if (!want || !u8_tc_supported(stride, cap)) return false;
        if (u8_map_for != packed.p) {
            if (!u8_tc_make_map(packed.p, n, stride, u8_map))
                raise(KNNG_CUDA_CUDA_ERROR, "cuTensorMapEncodeTiled failed for the byte copy");
            u8_map_for = packed.p;
        }
        return true;
    }

    // The 5-aligned tile kernel (join5.cu) is the FP32 distance stage;
    // KNNG_JOIN_T5=0 falls back to join.cu's 8 x 8 tile kernel (kept for A/B).
    bool use_t5_join() const {
        const char* v = getenv("KNNG_JOIN_T5");
        return !(v && v[0] == '0');
    }

    // The register-staged join (join_gl.cu) is opt-in: KNNG_JOIN_GL=1.
    // Measured 3x slower than the shared-memory tile kernel on C5 (DESIGN.md
    // §3.5): loads straight into registers leave the L2 latency exposed.
    bool use_gl_join() const {
        const char* v = getenv("KNNG_JOIN_GL");
        return v && v[0] == '1';
    }

    // The tensor-core screened join (join_tc.cu) is opt-in: KNNG_JOIN_TC=1
    // runs it for every prefiltered join, =auto from iteration 2 on rows of
    // >= 256 floats.  It needs the prefilter (it drops pairs that cannot beat
    // an endpoint's row maximum).  Measured slower than the FP32 tile kernel
    // on B200, so the default is off.
    bool use_screened_join(bool distances_only) const {
        if (distances_only || !filter) return false;
        const char* v = getenv("KNNG_JOIN_TC");
        if (!v || v[0] == '0') return false;
        if (v[0] == '1') return true;
        return iteration >= 2 && stride >= 256;  // "auto"
    }

    // ---- locality reorder (reorder.hpp:22-50, dataset.hpp:237-245,
    //      graph.hpp:150-166)
    DevBuf<uint32_t> sigma, sigma_inv;

    // KnnGraph::remap: row u -> row perm[u], ids renamed, rows re-sorted
    void remap_graph(const uint32_t* perm) {
        DevBuf<uint64_t> keys2;
        DevBuf<uint32_t> flags2;
        DevBuf<float> maxd2;
        // rows_alloc rows (>= n): multi-GPU shards all-gather equal slices
        keys2.alloc(size_t(rows_alloc) * k, pool, s);
        flags2.alloc(rows_alloc, pool, s);
        maxd2.alloc(rows_alloc, pool, s);
        GraphView out = gv();
        out.keys = keys2.p;
        out.flags = flags2.p;
        out.maxd = maxd2.p;
        launch_remap_graph(gv(), out, perm, s);
        CK(cudaGetLastError());
        std::swap(keys.p, keys2.p);
        std::swap(flags.p, flags2.p);
        std::swap(maxd.p, maxd2.p);
    }

    // sigma from the current graph, rows gathered, graph relabelled
    void reorder() {
        compute_sigma();
        apply_sigma();
    }
    void compute_sigma() {
        if (!sigma.p) {
            sigma.alloc(n, pool, s);
            sigma_inv.alloc(n, pool, s);
        }
        const size_t scratch_bytes = locality_permutation_scratch(n);
        DevBuf<unsigned char> scratch;
        scratch.alloc(scratch_bytes, pool, s);
        GraphView g = gv();
        g.lo = 0;
        g.hi = n;
        launch_locality_permutation(g, sigma.p, sigma_inv.p, scratch.p, scratch_bytes, s);
        CK(cudaGetLastError());
    }
    // the data rows and every graph row (ids renamed) into the order sigma
    // (sigma / sigma_inv already in place)
    void apply_sigma() {
        DevBuf<float> data2;
        data2.alloc(size_t(n) * stride, pool, s);
        launch_permute_rows(data.p, data2.p, sigma.p, n, stride, s);
        std::swap(data.p, data2.p);
        norms_valid = false;
        dl_valid = false;
        if (u8_state == 1) u8_state = -1;  // repack in the new row order
        remap_graph(sigma.p);
    }
    // remap_graph over every row, whatever the owned range (multi-GPU)
    void remap_all(const uint32_t* perm) {
        const uint32_t lo0 = lo, hi0 = hi;
        lo = 0;
        hi = n;
        remap_graph(perm);
        lo = lo0;
        hi = hi0;
    }

    void export_rows(uint32_t* ids, float* dists, uint8_t* fl) {
        launch_export_rows(gv(), ids, dists, fl, s);
        CK(cudaGetLastError());
    }

    // the owned rows [lo, hi) only (multi-GPU)
    void export_owned(uint32_t* ids, float* dists, uint8_t* fl) {
        GraphView g = gv();
        g.keys += size_t(lo) * k;
        g.flags += lo;
        g.maxd += lo;
        g.n = hi - lo;
        launch_export_rows(g, ids, dists, fl, s);
        CK(cudaGetLastError());
    }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

void metrics_reset(knng_cuda_metrics* m) {
    if (!m) return;
    m->n_rows = 0;
    m->total_wall_time_s = 0;
    m->total_dist_evals = 0;
    m->total_changes = 0;
    for (int i = 0; i < KNNG_CUDA_KERNEL_COUNT; ++i) {
        m->kernel_ms[i] = 0;
        m->kernel_launches[i] = 0;
    }
    m->join_candidates = 0;
    m->join_evals = 0;
    m->h2d_bytes = 0;
    m->d2h_bytes = 0;
}

void metrics_push(knng_cuda_metrics* m, uint32_t iteration, double wall, uint64_t evals,
                  uint64_t changes, uint64_t cands = 0, double join_ms = 0.0) {
    if (!m) return;
    if (m->iterations && m->n_rows < m->capacity)
        m->iterations[m->n_rows] =
            knng_cuda_iteration{iteration, wall, evals, changes, cands, join_ms};
    ++m->n_rows;
    m->total_wall_time_s += wall;
    m->total_dist_evals += evals;
    m->total_changes += changes;
}

// Counter slot j's recount flag <- 1 (stream-ordered; pageable source is
// copied before the call returns).
void set_recount(Engine& e, uint32_t j) {
    const uint32_t one = 1;
    CK(cudaMemcpyAsync(&e.ctr.p[j].recount, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, e.s));
}

// knng::run (descent.hpp:193-255) on one GPU; data already on the device or
// on the host per data_on_device; outputs device pointers.
void run_engine(Engine& e, const float* data, bool data_on_device, const knng_cuda_params& p,
                uint32_t* d_ids, float* d_dists, uint8_t* d_flags, knng_cuda_metrics* m,
                uint32_t* d_sigma = nullptr) {
    KernelTimer timer(p.profile != 0, e.s, m);
    bool reordered = false;
    if (p.deterministic && !e.det) {
        e.det = true;
        e.rawlist.alloc(size_t(e.n) * 4 * e.cap, e.pool, e.s);
    }
    std::mt19937_64 master(p.seed);
    double t0 = now_s();
    e.upload(data, data_on_device);
    const uint64_t init_seed = master();
    int h = timer.begin(KNNG_CUDA_KERNEL_INIT);
    // per-build data preparation (byte-valued data check + packing); init then
    // reads the byte copy
    const bool u8 = e.use_u8_join();
    launch_init_random(e.gv(), init_seed, e.s, u8 ? e.packed.p : nullptr, u8 ? e.lnorm.p : nullptr);
    timer.end(h);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e.s));
    timer.flush();
    double t1 = now_s();
    metrics_push(m, 0, t1 - t0, uint64_t(e.n) * e.k, 0);

    const double threshold = p.termination_delta * double(e.n) * double(e.k);
    // Iterations are enqueued in batches without a host round trip: each ends
    // with iter_end_kernel, which applies the termination test
    // (descent.hpp:242) on the device and sets the next slot's halt flag, so
    // iterations enqueued past termination do nothing and leave the graph as
    // the reference's loop leaves it.  The host reads the batch's counters
    // once; per-iteration wall time is device time between iteration events.
    // A batch ends at the reorder iteration (host work follows it).  When an
    // iteration's proposal blocks outgrew their buffer (its later iterations
    // halted too), the buffer grows, that iteration's join reruns, and
    // enqueueing resumes after it.  KNNG_ITER_BATCH=1 restores one round trip
    // per iteration.
    // The merges keep indeg current while iterations change few rows; an
    // iteration after one that changed more than 5% of the n·k entries
    // recounts instead (KNNG_INDEG_INC=0: recount every iteration)
    const char* iv = getenv("KNNG_INDEG_INC");
    const char* fv = getenv("KNNG_INDEG_RECOUNT_FRAC");
    const double frac = fv ? atof(fv) : 0.05;
    const double recount_above = (iv && iv[0] == '0') ? -1.0 : frac * double(e.n) * double(e.k);
    const char* bv = getenv("KNNG_ITER_BATCH");
    // an observer sees every iteration's graph: one iteration per round trip
    const uint32_t batch = p.observer ? 1u : bv && atoi(bv) > 0 ? uint32_t(atoi(bv)) : 4u;
    DevBuf<uint32_t> obs_ids;
    DevBuf<float> obs_dists;
    DevBuf<uint8_t> obs_flags;
    std::vector<uint32_t> h_obs_ids;
    std::vector<float> h_obs_dists;
    std::vector<uint8_t> h_obs_flags;
    auto observe = [&](uint32_t j) {
        if (!p.observer) return;
        const size_t nk = size_t(e.n) * e.k;
        if (!obs_ids.p) {
            obs_ids.alloc(nk, e.pool, e.s);
            obs_dists.alloc(nk, e.pool, e.s);
            obs_flags.alloc(nk, e.pool, e.s);
            h_obs_ids.resize(nk);
            h_obs_dists.resize(nk);
            h_obs_flags.resize(nk);
        }
        e.export_rows(obs_ids.p, obs_dists.p, obs_flags.p);
        CK(cudaMemcpyAsync(h_obs_ids.data(), obs_ids.p, sizeof(uint32_t) * nk,
                           cudaMemcpyDeviceToHost, e.s));
        CK(cudaMemcpyAsync(h_obs_dists.data(), obs_dists.p, sizeof(float) * nk,
                           cudaMemcpyDeviceToHost, e.s));
        CK(cudaMemcpyAsync(h_obs_flags.data(), obs_flags.p, nk, cudaMemcpyDeviceToHost, e.s));
        CK(cudaStreamSynchronize(e.s));
        e.d2h += 9 * nk;
        p.observer(j, e.n, e.k, h_obs_ids.data(), h_obs_dists.data(), h_obs_flags.data(),
                   p.observer_user);
    };
    const uint32_t T = p.max_iterations;
    e.ensure_slots(T + 3);
    e.indeg_inc = true;
    // iterations 1 and 2 recount (nothing counted yet / no change count to go by)
    {
        const uint32_t one = 1;
        for (uint32_t j = 1; j <= 2; ++j)
            CK(cudaMemcpyAsync(&e.ctr.p[j].recount, &one, sizeof(uint32_t),
                               cudaMemcpyHostToDevice, e.s));
        CK(cudaStreamSynchronize(e.s));
    }
    std::vector<uint64_t> seeds(T + 1);
    for (uint32_t i = 1; i <= T; ++i) seeds[i] = master();  // the reference's order
    thread_local std::vector<cudaEvent_t> iev;
    while (iev.size() < T + 2) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        iev.push_back(ev);
    }
    uint32_t it = 1;
    bool done = false;
    while (!done && it <= T) {
        uint32_t last = std::min(T, it + batch - 1);
        if (p.reorder && !reordered && p.reorder_after_iteration >= it &&
            p.reorder_after_iteration <= last)
            last = p.reorder_after_iteration;
        for (uint32_t j = it; j <= last; ++j) {
            e.cur = e.ctr.p + j;
            e.iteration = j;
            timer.tag = j;
            CK(cudaEventRecord(iev[j], e.s));
            e.select(seeds[j], timer);
            e.join_enqueue(timer);
            launch_iter_end(e.cur, e.cur + 1, threshold, recount_above, e.s);
        }
        CK(cudaEventRecord(iev[last + 1], e.s));
        CK(cudaMemcpyAsync(e.h_ctr + it, e.ctr.p + it, sizeof(IterCounters) * (last - it + 1),
                           cudaMemcpyDeviceToHost, e.s));
        e.d2h += sizeof(IterCounters) * (last - it + 1);
        CK(cudaStreamSynchronize(e.s));
        uint32_t next = last + 1;
        for (uint32_t j = it; j <= last; ++j) {
            IterCounters c = e.h_ctr[j];
            if (c.halt) {  // defensive: the previous iteration's test already stopped the run
                done = true;
                break;
            }
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, iev[j], iev[j + 1]));
            double wall = 1e-3 * ms;
            if (c.overflow) {
                const double r0 = now_s();
                e.cur = e.ctr.p + j;
                e.iteration = j;
                timer.tag = j;
                e.reserve_join(c.rev, c.dwords);
                CK(cudaMemsetAsync(&e.cur->overflow, 0, sizeof(uint32_t), e.s));
                e.join_stages(timer, false);
                e.read_counters();
                c = e.h_ctr[0];
                // the later slots of this batch ran halted: reset them; the
                // next iteration recounts the in-degree (always safe)
                CK(cudaMemsetAsync(e.ctr.p + j + 1, 0, sizeof(IterCounters) * (T + 2 - j), e.s));
                set_recount(e, j + 1);
                launch_iter_end(e.cur, e.cur + 1, threshold, recount_above, e.s);
                wall += now_s() - r0;
                next = j + 1;
            }
            timer.flush();
            metrics_push(m, j, wall, c.evals, c.changes, c.cands, timer.join_ms_of(j));
            if (m) {
                m->join_candidates += c.cands;
                m->join_evals += c.evals;
            }
            // the locality reorder runs once, after iteration reorder_after_iteration
            // (descent.hpp:230-235); the rest of the run works in permuted ids
            if (p.reorder && !reordered && j == p.reorder_after_iteration) {
                const double r0 = now_s();
                const int h = timer.begin(KNNG_CUDA_KERNEL_REORDER);
                e.reorder();
                timer.end(h);
                reordered = true;
                set_recount(e, j + 1);  // ids renamed: recount
                CK(cudaStreamSynchronize(e.s));
                timer.flush();
                if (m && m->iterations && m->n_rows > 0 && m->n_rows <= m->capacity)
                    m->iterations[m->n_rows - 1].wall_time_s += now_s() - r0;
                if (m) m->total_wall_time_s += now_s() - r0;
            }
            observe(j);  // descent.hpp:241, after the reorder of this iteration
            if (double(c.changes) < threshold) {
                done = true;
                break;
            }
            if (next == j + 1) break;  // resume enqueueing after the rerun iteration
        }
        it = next;
    }
    if (reordered) {
        // back to the caller's ids (descent.hpp:245)
        e.remap_graph(e.sigma_inv.p);
        if (d_sigma)
            CK(cudaMemcpyAsync(d_sigma, e.sigma.p, sizeof(uint32_t) * e.n,
                               cudaMemcpyDeviceToDevice, e.s));
    }
    e.export_rows(d_ids, d_dists, d_flags);
    CK(cudaStreamSynchronize(e.s));
}

template <typename T>
void to_device(DevBuf<T>& buf, const T* host, size_t count, Engine& e) {
    buf.alloc(count, e.pool, e.s);
    CK(cudaMemcpyAsync(buf.p, host, sizeof(T) * count, cudaMemcpyHostToDevice, e.s));
    e.h2d += sizeof(T) * count;
}

// Returns with the data on the host (host_io.cu stages pageable buffers).
template <typename T>
void to_host(T* host, const T* dev, size_t count, Engine& e) {
    if (!host) return;
    copy_to_host({{host, const_cast<T*>(dev), sizeof(T) * count}}, e.s);
    e.d2h += sizeof(T) * count;
}

// Several results in one staged transfer (null host buffers skipped).
void results_to_host(std::vector<HostSeg> segs, Engine& e) {
    std::vector<HostSeg> out;
    for (const HostSeg& g : segs)
        if (g.host && g.bytes) {
            out.push_back(g);
            e.d2h += g.bytes;
        }
    copy_to_host(out, e.s);
}

// from_rows validation (graph.hpp:70-93)
void validate_rows(uint32_t n, uint32_t k, const uint32_t* ids) {
    std::vector<uint32_t> seen;
    for (uint32_t u = 0; u < n; ++u) {
        const uint32_t* r = ids + size_t(u) * k;
        for (uint32_t i = 0; i < k; ++i) {
            if (r[i] == u) raise(KNNG_CUDA_INVALID_ARGUMENT, "from_rows: self loop");
            if (r[i] >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "from_rows: id out of range");
            for (uint32_t j = 0; j < i; ++j)
                if (r[j] == r[i]) raise(KNNG_CUDA_INVALID_ARGUMENT, "from_rows: duplicate id");
        }
    }
}

void validate_cands(uint32_t n, uint32_t cap, const uint32_t* cand_ids, const uint32_t* nc,
                    const uint32_t* oc) {
    for (uint32_t u = 0; u < n; ++u) {
        if (nc[u] > cap || oc[u] > cap)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "candidate count exceeds cap");
        const uint32_t* b = cand_ids + size_t(u) * 2 * cap;
        for (uint32_t i = 0; i < nc[u]; ++i)
            if (b[i] >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "candidate id out of range");
        for (uint32_t i = 0; i < oc[u]; ++i)
            if (b[cap + i] >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "candidate id out of range");
    }
}

}  // namespace

extern "C" {

void knng_cuda_params_default(knng_cuda_params* p) {
    if (!p) return;
    p->k = 20;
    p->max_candidates = 50;
    p->termination_delta = 0.001;
    p->max_iterations = 30;
    p->reorder = 0;
    p->reorder_after_iteration = 1;
    p->seed = 0;
    p->device = 0;
    p->profile = 0;
    p->deterministic = 0;
    p->observer = nullptr;
    p->observer_user = nullptr;
}

const char* knng_cuda_last_error(void) { return g_err.c_str(); }

int knng_cuda_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

int knng_cuda_run_device(const float* d_data, uint32_t n, uint32_t d, const knng_cuda_params* params,
                         uint32_t* d_out_ids, float* d_out_dists, knng_cuda_metrics* out_metrics,
                         void* stream) {
    return guarded([&] {
        if (!params || !d_data || !d_out_ids || !d_out_dists)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        const knng_cuda_params p = *params;
        validate_params(n, d, p);
        DeviceGuard dg(p.device);
        StreamHolder sh(stream);
        metrics_reset(out_metrics);
        Engine e(p.device, n, d, p.k, p.max_candidates, sh.s);
        run_engine(e, d_data, true, p, d_out_ids, d_out_dists, nullptr, out_metrics);
        if (out_metrics) {
            out_metrics->h2d_bytes = e.h2d;
            out_metrics->d2h_bytes = e.d2h;
        }
    });
}

int knng_cuda_run(const float* data, uint32_t n, uint32_t d, const knng_cuda_params* params,
                  uint32_t* out_ids, float* out_dists, uint8_t* out_flags, uint32_t* out_sigma,
                  knng_cuda_metrics* out_metrics) {
    return guarded([&] {
        if (!params || !data || !out_ids || !out_dists)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        const knng_cuda_params p = *params;
        validate_params(n, d, p);
        DeviceGuard dg(p.device);
        StreamHolder sh(nullptr);
        metrics_reset(out_metrics);
        Engine e(p.device, n, d, p.k, p.max_candidates, sh.s);
        DevBuf<uint32_t> ids, sig;
        DevBuf<float> dists;
        DevBuf<uint8_t> fl;
        const size_t nk = size_t(n) * p.k;
        ids.alloc(nk, e.pool, e.s);
        dists.alloc(nk, e.pool, e.s);
        if (out_flags) fl.alloc(nk, e.pool, e.s);
        const bool want_sigma = out_sigma && p.reorder;
        if (want_sigma) sig.alloc(n, e.pool, e.s);
        run_engine(e, data, false, p, ids.p, dists.p, out_flags ? fl.p : nullptr, out_metrics,
                   want_sigma ? sig.p : nullptr);
        results_to_host({{out_ids, ids.p, sizeof(uint32_t) * nk},
                         {out_dists, dists.p, sizeof(float) * nk},
                         {out_flags, fl.p, nk},
                         {want_sigma ? out_sigma : nullptr, sig.p, sizeof(uint32_t) * n}},
                        e);
        if (out_metrics) {
            out_metrics->h2d_bytes = e.h2d;
            out_metrics->d2h_bytes = e.d2h;
        }
    });
}

int knng_cuda_nndescent_l2(const float* data, uint32_t n, uint32_t d, uint32_t k,
                           double sample_rate, double delta, uint64_t seed,
                           uint32_t max_iterations, int num_gpus, uint32_t* out_ids,
                           float* out_dists, knng_cuda_metrics* out_metrics) {
    int rc = guarded([&] {
        if (!(sample_rate > 0.0) || !std::isfinite(sample_rate))
            raise(KNNG_CUDA_INVALID_ARGUMENT, "sample_rate must be positive");
        if (num_gpus < 1) raise(KNNG_CUDA_INVALID_ARGUMENT, "num_gpus must be at least 1");
    });
    if (rc) return rc;
    knng_cuda_params p;
    knng_cuda_params_default(&p);
    p.k = k;
    const double cap = std::llround(sample_rate * double(k));
    p.max_candidates = cap > 4294967295.0 ? 0xffffffffu : uint32_t(cap);
    p.termination_delta = delta;
    p.seed = seed;
    p.max_iterations = max_iterations;
    if (num_gpus > 1)  // shard r on device r % device count, in this process
        return knng_cuda_run_multi(data, n, d, &p, num_gpus, nullptr, out_ids, out_dists,
                                   out_metrics);
    return knng_cuda_run(data, n, d, &p, out_ids, out_dists, nullptr, nullptr, out_metrics);
}

int knng_cuda_local_join(const float* data, uint32_t n, uint32_t d, uint32_t k, uint32_t cap,
                         const uint32_t* in_ids, const float* in_dists, const uint8_t* in_flags,
                         const uint32_t* cand_ids, const uint32_t* new_counts,
                         const uint32_t* old_counts, uint32_t* out_ids, float* out_dists,
                         uint8_t* out_flags, uint32_t* out_rev_deg, uint64_t* changes,
                         uint64_t* evals, int device) {
    return guarded([&] {
        if (!data || !in_ids || !in_dists || !in_flags || !cand_ids || !new_counts || !old_counts)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        validate_shape(n, d, k);
        if (cap == 0) raise(KNNG_CUDA_INVALID_ARGUMENT, "CandidateSet: cap must be positive");
        if (cap > KNNG_CUDA_MAX_CANDIDATES)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports max_candidates <= 64");
        validate_rows(n, k, in_ids);
        validate_cands(n, cap, cand_ids, new_counts, old_counts);
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, d, k, cap, sh.s);
        e.upload(data, false);
        DevBuf<uint32_t> ids;
        DevBuf<float> dists;
        DevBuf<uint8_t> fl;
        const size_t nk = size_t(n) * k;
        to_device(ids, in_ids, nk, e);
        to_device(dists, in_dists, nk, e);
        to_device(fl, in_flags, nk, e);
        launch_load_rows(e.gv(), ids.p, dists.p, fl.p, e.s);
        CK(cudaMemcpyAsync(e.cand.p, cand_ids, sizeof(uint32_t) * size_t(n) * 2 * cap,
                           cudaMemcpyHostToDevice, e.s));
        CK(cudaMemcpyAsync(e.nc.p, new_counts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e.s));
        CK(cudaMemcpyAsync(e.oc.p, old_counts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e.s));
        // finalize's bookkeeping on the injected lists, then the join stages
        launch_bookkeeping(e.gv(), e.cv(), e.active.p, e.ctr.p, e.s);
        KernelTimer timer(false, e.s, nullptr);
        e.join(timer);
        e.read_counters();
        const uint64_t ev = e.h_ctr->evals;
        e.export_rows(ids.p, dists.p, fl.p);
        to_host(out_ids, ids.p, nk, e);
        to_host(out_dists, dists.p, nk, e);
        to_host(out_flags, fl.p, nk, e);
        if (out_rev_deg) {
            launch_indegree(e.gv(), e.indeg.p, e.s);
            std::vector<uint32_t> indeg(n);
            CK(cudaMemcpyAsync(indeg.data(), e.indeg.p, sizeof(uint32_t) * n,
                               cudaMemcpyDeviceToHost, e.s));
            CK(cudaStreamSynchronize(e.s));
            for (uint32_t u = 0; u < n; ++u) out_rev_deg[u] = k + indeg[u];
        }
        CK(cudaStreamSynchronize(e.s));
        if (changes) *changes = e.h_ctr->changes;
        if (evals) *evals = ev;
    });
}

int knng_cuda_candidate_distances(const float* data, uint32_t n, uint32_t d, uint32_t cap,
                                  const uint32_t* cand_ids, const uint32_t* new_counts,
                                  const uint32_t* old_counts, const uint64_t* offsets,
                                  float* out_dists, uint64_t total, int device) {
    return guarded([&] {
        if (!data || !cand_ids || !new_counts || !old_counts || !offsets || !out_dists)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        if (n < 2 || d < 1) raise(KNNG_CUDA_INVALID_ARGUMENT, "Dataset: degenerate shape");
        if (cap == 0 || cap > KNNG_CUDA_MAX_CANDIDATES)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "cap must be in [1, 64]");
        validate_cands(n, cap, cand_ids, new_counts, old_counts);
        for (uint32_t u = 0; u < n; ++u)
            if (new_counts[u] > 0 &&
                offsets[u] + uint64_t(new_counts[u]) * (new_counts[u] + old_counts[u]) > total)
                raise(KNNG_CUDA_INVALID_ARGUMENT, "offsets exceed the output size");
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, d, 2, cap, sh.s);
        e.upload(data, false);
        CK(cudaMemcpyAsync(e.cand.p, cand_ids, sizeof(uint32_t) * size_t(n) * 2 * cap,
                           cudaMemcpyHostToDevice, e.s));
        CK(cudaMemcpyAsync(e.nc.p, new_counts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e.s));
        CK(cudaMemcpyAsync(e.oc.p, old_counts, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, e.s));
        e.filter = 0;
        launch_bookkeeping(e.gv(), e.cv(), e.active.p, e.ctr.p, e.s);
        KernelTimer timer(false, e.s, nullptr);
        e.join(timer, /*distances_only=*/true);
        // unfiltered proposal blocks: row i (new candidate i) holds every
        // partner as (distance, id); place each by its partner's position
        const uint64_t dtotal = e.h_ctr->dwords;
        std::vector<uint64_t> blocks(dtotal);
        std::vector<uint64_t> doff(n);
        if (dtotal) to_host(blocks.data(), e.dblocks.p, dtotal, e);
        to_host(doff.data(), e.doff.p, n, e);
        CK(cudaStreamSynchronize(e.s));
        for (uint32_t u = 0; u < n; ++u) {
            const uint64_t nn = new_counts[u], m = nn + old_counts[u];
            if (!nn) continue;
            const uint32_t* list = cand_ids + size_t(u) * 2 * cap;
            for (uint64_t i = 0; i < nn; ++i) {
                const uint64_t* row = blocks.data() + doff[u] + i * m;
                for (uint64_t q = 0; q < row[0]; ++q) {
                    const uint32_t id = uint32_t(row[1 + q]);
                    const uint32_t bits = uint32_t(row[1 + q] >> 32);
                    float dist;
                    std::memcpy(&dist, &bits, 4);
                    for (uint64_t j = 0; j < m; ++j)
                        if (j != i && (j < nn ? list[j] : list[cap + j - nn]) == id)
                            out_dists[offsets[u] + i * m + j] = dist;
                }
            }
        }
    });
}

int knng_cuda_init_random(const float* data, uint32_t n, uint32_t d, uint32_t k, uint64_t seed,
                          uint32_t* out_ids, float* out_dists, uint8_t* out_flags,
                          uint32_t* out_rev_deg, uint64_t* evals, int device) {
    return guarded([&] {
        if (!data) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        validate_shape(n, d, k);
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, d, k, 0, sh.s);
        e.upload(data, false);
        const bool u8 = e.use_u8_join();
        launch_init_random(e.gv(), seed, e.s, u8 ? e.packed.p : nullptr, u8 ? e.lnorm.p : nullptr);
        const size_t nk = size_t(n) * k;
        DevBuf<uint32_t> ids;
        DevBuf<float> dists;
        DevBuf<uint8_t> fl;
        ids.alloc(nk, e.pool, e.s);
        dists.alloc(nk, e.pool, e.s);
        fl.alloc(nk, e.pool, e.s);
        e.export_rows(ids.p, dists.p, fl.p);
        to_host(out_ids, ids.p, nk, e);
        to_host(out_dists, dists.p, nk, e);
        to_host(out_flags, fl.p, nk, e);
        if (out_rev_deg) {
            launch_indegree(e.gv(), e.indeg.p, e.s);
            std::vector<uint32_t> indeg(n);
            CK(cudaMemcpyAsync(indeg.data(), e.indeg.p, sizeof(uint32_t) * n,
                               cudaMemcpyDeviceToHost, e.s));
            CK(cudaStreamSynchronize(e.s));
            for (uint32_t u = 0; u < n; ++u) out_rev_deg[u] = k + indeg[u];
        }
        CK(cudaStreamSynchronize(e.s));
        if (evals) *evals = nk;
    });
}

int knng_cuda_select(uint32_t n, uint32_t k, uint32_t cap, const uint32_t* in_ids,
                     const float* in_dists, const uint8_t* in_flags, uint64_t seed,
                     uint32_t* cand_ids, uint32_t* new_counts, uint32_t* old_counts,
                     uint8_t* out_flags_after, int device) {
    return guarded([&] {
        if (!in_ids || !in_dists || !in_flags || !cand_ids || !new_counts || !old_counts)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        validate_shape(n, 1, k);
        if (cap == 0) raise(KNNG_CUDA_INVALID_ARGUMENT, "CandidateSet: cap must be positive");
        if (cap > KNNG_CUDA_MAX_CANDIDATES)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports max_candidates <= 64");
        validate_rows(n, k, in_ids);
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, 1, k, cap, sh.s);
        const size_t nk = size_t(n) * k;
        DevBuf<uint32_t> ids;
        DevBuf<float> dists;
        DevBuf<uint8_t> fl;
        to_device(ids, in_ids, nk, e);
        to_device(dists, in_dists, nk, e);
        to_device(fl, in_flags, nk, e);
        launch_load_rows(e.gv(), ids.p, dists.p, fl.p, e.s);
        KernelTimer timer(false, e.s, nullptr);
        e.select(seed, timer);
        to_host(cand_ids, e.cand.p, size_t(n) * 2 * cap, e);
        to_host(new_counts, e.nc.p, n, e);
        to_host(old_counts, e.oc.p, n, e);
        std::vector<uint32_t> sorted_ids(nk);
        std::vector<uint8_t> sorted_flags(nk);
        e.export_rows(ids.p, nullptr, fl.p);
        to_host(sorted_ids.data(), ids.p, nk, e);
        to_host(sorted_flags.data(), fl.p, nk, e);
        CK(cudaStreamSynchronize(e.s));
        if (out_flags_after) {
            // report flags in the caller's entry order
            for (uint32_t u = 0; u < n; ++u)
                for (uint32_t i = 0; i < k; ++i) {
                    const uint32_t id = in_ids[size_t(u) * k + i];
                    for (uint32_t j = 0; j < k; ++j)
                        if (sorted_ids[size_t(u) * k + j] == id)
                            out_flags_after[size_t(u) * k + i] = sorted_flags[size_t(u) * k + j];
                }
        }
    });
}

int knng_cuda_bruteforce_queries(const float* data, uint32_t n, uint32_t d, uint32_t k,
                                 const uint32_t* queries, uint32_t nq, uint32_t* out_ids,
                                 double* out_dists, int device) {
    return guarded([&] {
        if (!data || !out_ids) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        if (k == 0 || k >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "brute_force_knng: need 0 < k < n");
        if (k > KNNG_CUDA_MAX_K) raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports k <= 32");
        if (d < 1) raise(KNNG_CUDA_INVALID_ARGUMENT, "Dataset: need at least 1 dimension");
        if (n >= (1u << 31)) raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports n < 2^31");
        if (queries)
            for (uint32_t i = 0; i < nq; ++i)
                if (queries[i] >= n) raise(KNNG_CUDA_INVALID_ARGUMENT, "query id out of range");
        const uint32_t count = queries ? nq : n;
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, d, k, 0, sh.s);
        e.upload(data, false);
        DevBuf<uint32_t> q;
        if (queries) {
            to_device(q, queries, count, e);
        } else {
            q.alloc(count, e.pool, e.s);
            launch_iota(q.p, count, e.s);
        }
        const size_t nk = size_t(count) * k;
        DevBuf<uint32_t> ids;
        DevBuf<double> dists;
        DevBuf<uint64_t> top;
        ids.alloc(nk, e.pool, e.s);
        dists.alloc(nk, e.pool, e.s);
        top.alloc(bruteforce_scratch_keys(count), e.pool, e.s);
        launch_bruteforce_queries(e.data.p, n, d, e.stride, k, q.p, count, top.p, ids.p, dists.p,
                                  e.s);
        CK(cudaGetLastError());
        to_host(out_ids, ids.p, nk, e);
        if (out_dists) to_host(out_dists, dists.p, nk, e);
        CK(cudaStreamSynchronize(e.s));
    });
}

int knng_cuda_bruteforce_knng(const float* data, uint32_t n, uint32_t d, uint32_t k,
                              uint32_t* out_ids, double* out_dists, int device) {
    return knng_cuda_bruteforce_queries(data, n, d, k, nullptr, n, out_ids, out_dists, device);
}

int knng_cuda_locality_permutation(uint32_t n, uint32_t k, const uint32_t* ids,
                                   const float* dists, uint32_t* sigma, uint32_t* sigma_inv,
                                   int device) {
    return guarded([&] {
        if (!ids || !dists || !sigma || !sigma_inv)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        validate_shape(n, 1, k);
        validate_rows(n, k, ids);
        DeviceGuard dg(device);
        StreamHolder sh(nullptr);
        Engine e(device, n, 1, k, 0, sh.s);
        const size_t nk = size_t(n) * k;
        DevBuf<uint32_t> d_ids;
        DevBuf<float> d_dists;
        DevBuf<uint8_t> d_fl;
        to_device(d_ids, ids, nk, e);
        to_device(d_dists, dists, nk, e);
        d_fl.alloc(nk, e.pool, e.s);
        CK(cudaMemsetAsync(d_fl.p, 0, nk, e.s));
        launch_load_rows(e.gv(), d_ids.p, d_dists.p, d_fl.p, e.s);
        e.sigma.alloc(n, e.pool, e.s);
        e.sigma_inv.alloc(n, e.pool, e.s);
        const size_t scratch_bytes = locality_permutation_scratch(n);
        DevBuf<unsigned char> scratch;
        scratch.alloc(scratch_bytes, e.pool, e.s);
        launch_locality_permutation(e.gv(), e.sigma.p, e.sigma_inv.p, scratch.p, scratch_bytes,
                                    e.s);
        CK(cudaGetLastError());
        to_host(sigma, e.sigma.p, n, e);
        to_host(sigma_inv, e.sigma_inv.p, n, e);
        CK(cudaStreamSynchronize(e.s));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-GPU shards: vertex-range ownership with the data
// replicated.  Shard r owns rows [r*chunk, min(n, (r+1)*chunk)): their graph
// rows, their candidate lists, their joins and their merges.  Only the row
// maxima (n floats, the join prefilter's bound) are replicated.  Per iteration
// (reference loop descent.hpp:219-243):
//   degree   partial in-degree of the owned rows' edges   -> all-reduce (n u32)
//   sample   owned edges only; reverse offers for rows owned elsewhere,
//            accepted with the global in-degree, grouped by owner -> all-to-all
//   offers   received offers into the owned lists
//   step     finalize, local join, merges into owned rows, pre-reduced
//            proposal records for rows owned elsewhere    -> all-to-all
//   merge    received records into owned rows            -> all-gather maxd,
//                                                           all-reduce changes
// Every phase is split into an enqueue part and a finish part (the host
// reads the counts it needs), so the in-process driver (knng_cuda_run_multi)
// keeps every GPU busy while it waits for one; the C-ABI phase functions run
// both back to back for callers that exchange with NCCL (shard.py).
// ---------------------------------------------------------------------------
struct knng_cuda_shard {
    // the stream a shard created for itself outlives every buffer freed on it
    // (declared first, destroyed last)
    struct OwnedStream {
        cudaStream_t s = nullptr;
        ~OwnedStream() {
            if (s) cudaStreamDestroy(s);
        }
    } owned;
    int device = 0;
    knng_cuda_params p{};
    uint32_t rank = 0, nranks = 1, chunk = 0;
    cudaStream_t s = nullptr;
    Engine* e = nullptr;
    KernelTimer* timer = nullptr;
    knng_cuda_metrics kmetrics{};  // per-kernel times of the shard's stream (params.profile)
    // reverse offers for rows owned elsewhere: nranks segments of seg_cap
    // records {target, cand, is_new, slot draw}; their counts
    DevBuf<uint4> osend;
    DevBuf<uint32_t> ocnt;
    uint64_t seg_cap = 0;
    // proposal records for rows owned elsewhere
    DevBuf<uint32_t> exp_counts, rcnt, roff2, rcur2, send;
    DevBuf<uint64_t> exp_off, bounds, grouped;
    DevBuf<unsigned char> scan_tmp;
    size_t scan_bytes = 0, send_cap = 0, grouped_cap = 0;
    // pinned host mirror: [0, nranks) offer counts, [nranks, 2 nranks + 1) record bounds
    uint64_t* h_pin = nullptr;
    uint32_t* h_ocnt = nullptr;
    IterCounters last{};  // counters of the last finished phase
    IterCounters joined{};  // this iteration's join counters (evaluations, candidates)
    std::vector<knng_cuda_iteration> rows;  // per iteration: this shard's share
    ~knng_cuda_shard() {
        delete timer;
        delete e;
        if (h_pin) cudaFreeHost(h_pin);
        if (h_ocnt) cudaFreeHost(h_ocnt);
    }

    // ---- degree
    void enq_degree() {
        ++e->iteration;
        timer->tag = e->iteration;
        CK(cudaMemsetAsync(e->ctr.p, 0, sizeof(IterCounters), s));
        launch_indegree_owned(e->gv(), e->indeg.p, s);
        CK(cudaGetLastError());
    }
    // ---- sample (the in-degree is global by now)
    void enq_sample(uint64_t seed) {
        const GraphView g = e->gv();
        const CandView c = e->cv();
        const int h = timer->begin(KNNG_CUDA_KERNEL_SAMPLE);
        launch_reset_raw(c, e->n, s, e->ctr.p);
        launch_sample_owned(g, c, e->indeg.p, seed, e->ctr.p, chunk, nranks, ocnt.p, osend.p,
                            seg_cap, s);
        timer->end(h);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_ocnt, ocnt.p, sizeof(uint32_t) * nranks, cudaMemcpyDeviceToHost, s));
    }
    void fin_sample(uint64_t* counts) {
        CK(cudaStreamSynchronize(s));
        for (uint32_t r = 0; r < nranks; ++r) counts[r] = h_ocnt[r];
        e->d2h += sizeof(uint32_t) * nranks;
    }
    // ---- offers
    void enq_offers(const uint4* recs, uint64_t count) {
        launch_apply_offers(e->cv(), recs, count, e->ctr.p, s);
        CK(cudaGetLastError());
    }
    // ---- step: finalize + join + merges of owned targets, then the export count
    void enq_step_join() {
        const int h = timer->begin(KNNG_CUDA_KERNEL_FINALIZE);
        launch_finalize(e->gv(), e->cv(), e->active.p, e->ctr.p, s);
        timer->end(h);
        CK(cudaGetLastError());
        e->cur = e->ctr.p;
        e->join_enqueue(*timer);
        CK(cudaMemcpyAsync(e->h_ctr, e->cur, sizeof(IterCounters), cudaMemcpyDeviceToHost, s));
    }
    void fin_step_join() {
        CK(cudaStreamSynchronize(s));
        e->d2h += sizeof(IterCounters);
        if (e->h_ctr->overflow) {
            e->reserve_join(e->h_ctr->rev, e->h_ctr->dwords);
            CK(cudaMemsetAsync(&e->cur->overflow, 0, sizeof(uint32_t), s));
            e->join_stages(*timer, false);
            e->read_counters();
        }
        last = *e->h_ctr;
        joined = last;
        // records for targets owned elsewhere: count pass, offsets, bounds
        const GraphView g = e->gv();
        const int h = timer->begin(KNNG_CUDA_KERNEL_MERGE);
        launch_export_remote(g, e->cv(), e->ctr.p, exp_counts.p, nullptr, nullptr, false, s);
        size_t bytes = scan_bytes;
        CK(cub::DeviceScan::ExclusiveScan(scan_tmp.p, bytes, exp_counts.p, exp_off.p, cub::Sum(),
                                          uint64_t(0), int(e->n), s));
        shard_bounds(s);
        timer->end(h);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h_pin + nranks, bounds.p, sizeof(uint64_t) * (nranks + 1),
                           cudaMemcpyDeviceToHost, s));
    }
    void fin_step_export(uint64_t* send_counts) {
        CK(cudaStreamSynchronize(s));
        e->d2h += sizeof(uint64_t) * (nranks + 1);
        const uint64_t* b = h_pin + nranks;
        const uint64_t total = b[nranks];
        if (3 * total > send_cap) {
            send.~DevBuf();
            new (&send) DevBuf<uint32_t>();
            send_cap = 3 * (total + total / 4 + 1024);
            send.alloc(send_cap, e->pool, s);
        }
        if (total)
            launch_export_remote(e->gv(), e->cv(), e->ctr.p, exp_counts.p, exp_off.p, send.p, true,
                                 s);
        CK(cudaGetLastError());
        for (uint32_t r = 0; r < nranks; ++r) send_counts[r] = b[r + 1] - b[r];
    }
    // ---- merge of received records
    void enq_merge(const uint32_t* recs, uint64_t count) {
        if (count > grouped_cap) {
            grouped.~DevBuf();
            new (&grouped) DevBuf<uint64_t>();
            grouped_cap = count + count / 4 + 1024;
            grouped.alloc(grouped_cap, e->pool, s);
        }
        const int h = timer->begin(KNNG_CUDA_KERNEL_MERGE);
        launch_merge_received(e->gv(), recs, count, rcnt.p, roff2.p, rcur2.p, grouped.p,
                              scan_tmp.p, scan_bytes, e->ctr.p, s);
        timer->end(h);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(e->h_ctr, e->ctr.p, sizeof(IterCounters), cudaMemcpyDeviceToHost, s));
    }
    void fin_merge() {
        CK(cudaStreamSynchronize(s));
        e->d2h += sizeof(IterCounters);
        last = *e->h_ctr;
        timer->flush();
        rows.push_back(knng_cuda_iteration{e->iteration, 0.0, joined.evals, last.changes,
                                           joined.cands, timer->join_ms_of(e->iteration)});
    }
    void shard_bounds(cudaStream_t st);
};

namespace {

__global__ void shard_bounds_kernel(const uint64_t* off, const uint32_t* counts, uint32_t n,
                                    uint32_t chunk, uint32_t nranks, uint64_t* bounds) {
    const uint64_t total = n ? off[n - 1] + counts[n - 1] : 0;
    for (uint32_t r = threadIdx.x; r <= nranks; r += blockDim.x) {
        const uint64_t start = uint64_t(r) * chunk;
        bounds[r] = start >= n ? total : off[start];
    }
}

constexpr uint32_t kMaxShards = 1023;

knng_cuda_shard* shard_new(const float* data, bool data_on_device, uint32_t n, uint32_t d,
                           const knng_cuda_params& p, uint32_t rank, uint32_t nranks,
                           cudaStream_t stream, bool allow_reorder = false) {
    if (nranks == 0 || rank >= nranks) raise(KNNG_CUDA_INVALID_ARGUMENT, "bad rank / nranks");
    if (nranks > kMaxShards)
        raise(KNNG_CUDA_INVALID_ARGUMENT, "this build supports at most 1023 shards");
    validate_params(n, d, p);
    (void)allow_reorder;  // the phase API reorders through knng_cuda_shard_reorder
    if (p.deterministic)
        raise(KNNG_CUDA_NOT_IMPLEMENTED, "deterministic mode is not supported on the sharded path");
    auto* sh = new knng_cuda_shard();
    try {
        sh->device = p.device;
        sh->p = p;
        sh->rank = rank;
        sh->nranks = nranks;
        sh->chunk = (n + nranks - 1) / nranks;
        if (stream) {
            sh->s = stream;
        } else {
            CK(cudaStreamCreateWithFlags(&sh->owned.s, cudaStreamNonBlocking));
            sh->s = sh->owned.s;
        }
        sh->e = new Engine(p.device, n, d, p.k, p.max_candidates, sh->s, sh->chunk * nranks);
        Engine& e = *sh->e;
        e.lo = std::min(n, rank * sh->chunk);
        e.hi = std::min(n, (rank + 1) * sh->chunk);
        e.upload(data, data_on_device);
        // byte-valued data: check and pack once here (KNNG_SHARD_U8=0 keeps
        // the FP32 join on the shards)
        const char* sv = getenv("KNNG_SHARD_U8");
        if (sv && sv[0] == '0')
            e.u8_state = 0;
        else
            e.use_u8_join();
        const uint64_t owned_edges = uint64_t(e.hi - e.lo) * p.k;
        sh->seg_cap = std::max<uint64_t>(owned_edges, 1);
        sh->osend.alloc(sh->seg_cap * nranks, e.pool, e.s);
        sh->ocnt.alloc(nranks, e.pool, e.s);
        sh->exp_counts.alloc(n, e.pool, e.s);
        sh->exp_off.alloc(n, e.pool, e.s);
        sh->rcnt.alloc(n, e.pool, e.s);
        sh->roff2.alloc(n, e.pool, e.s);
        sh->rcur2.alloc(n, e.pool, e.s);
        sh->bounds.alloc(nranks + 1, e.pool, e.s);
        size_t a = 0, b = 0;
        CK(cub::DeviceScan::ExclusiveScan(nullptr, a, sh->exp_counts.p, sh->exp_off.p, cub::Sum(),
                                          uint64_t(0), int(n)));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, b, sh->rcnt.p, sh->roff2.p, int(n)));
        sh->scan_bytes = std::max(a, b);
        sh->scan_tmp.alloc(sh->scan_bytes, e.pool, e.s);
        CK(cudaMallocHost(reinterpret_cast<void**>(&sh->h_pin), sizeof(uint64_t) * (2 * nranks + 2)));
        CK(cudaMallocHost(reinterpret_cast<void**>(&sh->h_ocnt), sizeof(uint32_t) * nranks));
        sh->timer = new KernelTimer(p.profile != 0, sh->s, &sh->kmetrics);
        metrics_reset(&sh->kmetrics);
        CK(cudaStreamSynchronize(e.s));
    } catch (...) {
        delete sh;
        throw;
    }
    return sh;
}

void shard_fill_info(const knng_cuda_shard* sh, knng_cuda_shard_info* info) {
    const Engine& e = *sh->e;
    info->keys = e.keys.p;
    info->flags = e.flags.p;
    info->maxd = e.maxd.p;
    info->indeg = e.indeg.p;
    info->rows_alloc = e.rows_alloc;
    info->chunk = sh->chunk;
    info->lo = e.lo;
    info->hi = e.hi;
    info->stream = sh->s;
    info->seg_cap = sh->seg_cap;
}

}  // namespace

void knng_cuda_shard::shard_bounds(cudaStream_t st) {
    shard_bounds_kernel<<<1, 256, 0, st>>>(exp_off.p, exp_counts.p, e->n, chunk, nranks, bounds.p);
}

extern "C" {

int knng_cuda_shard_create(const float* d_data, uint32_t n, uint32_t d,
                           const knng_cuda_params* params, uint32_t rank, uint32_t nranks,
                           void* stream, knng_cuda_shard** out, knng_cuda_shard_info* info) {
    return guarded([&] {
        if (!d_data || !params || !out || !info) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(params->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        knng_cuda_shard* sh = shard_new(d_data, true, n, d, *params, rank, nranks, st);
        shard_fill_info(sh, info);
        *out = sh;
    });
}

void knng_cuda_seed_sequence(uint64_t seed, uint32_t count, uint64_t* out) {
    std::mt19937_64 master(seed);  // descent.hpp:201-221
    for (uint32_t i = 0; i < count; ++i) out[i] = master();
}

int knng_cuda_shard_destroy(knng_cuda_shard* sh) {
    return guarded([&] {
        if (!sh) return;
        DeviceGuard dg(sh->device);
        cudaStreamSynchronize(sh->s);
        delete sh;
    });
}

int knng_cuda_shard_init(knng_cuda_shard* sh, uint64_t seed) {
    return guarded([&] {
        if (!sh) raise(KNNG_CUDA_INVALID_ARGUMENT, "null shard");
        DeviceGuard dg(sh->device);
        const bool u8 = sh->e->u8_state == 1;  // byte copy made at creation
        launch_init_random(sh->e->gv(), seed, sh->s, u8 ? sh->e->packed.p : nullptr,
                           u8 ? sh->e->lnorm.p : nullptr);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(sh->s));
    });
}

int knng_cuda_shard_degree(knng_cuda_shard* sh) {
    return guarded([&] {
        if (!sh) raise(KNNG_CUDA_INVALID_ARGUMENT, "null shard");
        DeviceGuard dg(sh->device);
        sh->enq_degree();
    });
}

int knng_cuda_shard_sample(knng_cuda_shard* sh, uint64_t seed, uint64_t* send_counts,
                           const uint32_t** send_records) {
    return guarded([&] {
        if (!sh || !send_counts || !send_records) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        sh->enq_sample(seed);
        sh->fin_sample(send_counts);
        *send_records = reinterpret_cast<const uint32_t*>(sh->osend.p);
    });
}

int knng_cuda_shard_offers(knng_cuda_shard* sh, const uint32_t* d_records, uint64_t count) {
    return guarded([&] {
        if (!sh || (count && !d_records)) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        sh->enq_offers(reinterpret_cast<const uint4*>(d_records), count);
    });
}

int knng_cuda_shard_step(knng_cuda_shard* sh, uint64_t* out_counters, uint64_t* send_counts,
                         const uint32_t** send_records) {
    return guarded([&] {
        if (!sh || !out_counters || !send_counts || !send_records)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        sh->enq_step_join();
        sh->fin_step_join();
        sh->fin_step_export(send_counts);
        *send_records = sh->send.p;
        out_counters[0] = sh->last.evals;
        out_counters[1] = sh->last.cands;
        out_counters[2] = sh->last.changes;
        out_counters[3] = sh->last.active;
    });
}

int knng_cuda_shard_merge(knng_cuda_shard* sh, const uint32_t* d_records, uint64_t count,
                          uint64_t* changes) {
    return guarded([&] {
        if (!sh || !changes || (count && !d_records))
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        sh->enq_merge(d_records, count);
        sh->fin_merge();
        *changes = sh->last.changes;  // local + received merges of this iteration
    });
}

int knng_cuda_shard_reorder(knng_cuda_shard* sh, knng_cuda_shard_info* info,
                            const uint32_t** d_sigma, const uint32_t** d_sigma_inv) {
    return guarded([&] {
        if (!sh || !info || !d_sigma || !d_sigma_inv)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        Engine& e = *sh->e;
        // sigma is a deterministic function of the (gathered) graph, so every
        // shard computes the same one
        e.compute_sigma();
        const uint32_t lo0 = e.lo, hi0 = e.hi;
        e.lo = 0;
        e.hi = e.n;
        e.apply_sigma();
        e.lo = lo0;
        e.hi = hi0;
        CK(cudaStreamSynchronize(sh->s));
        shard_fill_info(sh, info);  // the graph buffers were reallocated
        *d_sigma = e.sigma.p;
        *d_sigma_inv = e.sigma_inv.p;
    });
}

int knng_cuda_shard_metrics(knng_cuda_shard* sh, knng_cuda_metrics* out) {
    return guarded([&] {
        if (!sh || !out) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        CK(cudaStreamSynchronize(sh->s));
        sh->timer->flush();
        metrics_reset(out);
        for (int kk = 0; kk < KNNG_CUDA_KERNEL_COUNT; ++kk) {
            out->kernel_ms[kk] = sh->kmetrics.kernel_ms[kk];
            out->kernel_launches[kk] = sh->kmetrics.kernel_launches[kk];
        }
        for (const knng_cuda_iteration& r : sh->rows) {
            if (out->iterations && out->n_rows < out->capacity) out->iterations[out->n_rows] = r;
            ++out->n_rows;
            out->total_dist_evals += r.dist_evals;
            out->total_changes += r.changes;
            out->join_candidates += r.join_candidates;
            out->join_evals += r.dist_evals;
        }
    });
}

int knng_cuda_shard_export(knng_cuda_shard* sh, uint32_t* d_ids, float* d_dists) {
    return guarded([&] {
        if (!sh || !d_ids || !d_dists) raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(sh->device);
        sh->e->export_owned(d_ids, d_dists, nullptr);
        CK(cudaStreamSynchronize(sh->s));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// In-process multi-GPU driver: knng::run (descent.hpp:193-255) over P shards,
// shard r on device devices[r] (default r % device count), one host thread,
// one stream per shard.  The exchanges are peer copies (cudaMemcpyPeerAsync:
// NVLink between B200s, a device copy when two shards share a GPU) ordered by
// events between the shards' streams; the host reads only the counts an
// exchange needs and the iteration's change counts.
// ---------------------------------------------------------------------------
namespace {

struct MultiRun {
    std::vector<knng_cuda_shard*> sh;
    std::vector<int> dev;
    std::vector<cudaEvent_t> ev;                  // one per shard, reused
    std::unique_ptr<DevBuf<uint32_t>[]> ipart;    // per shard: P x n partial in-degrees
    std::unique_ptr<DevBuf<uint4>[]> orecv;       // received offers
    std::vector<size_t> orecv_cap;
    std::unique_ptr<DevBuf<uint32_t>[]> rrecv;    // received proposal records
    std::vector<size_t> rrecv_cap;
    uint32_t P = 0, n = 0;
    ~MultiRun() {
        for (size_t r = 0; r < sh.size(); ++r) {
            if (!sh[r]) continue;
            cudaSetDevice(dev[r]);
            cudaStreamSynchronize(sh[r]->s);
            ipart[r].~DevBuf();
            new (&ipart[r]) DevBuf<uint32_t>();
            orecv[r].~DevBuf();
            new (&orecv[r]) DevBuf<uint4>();
            rrecv[r].~DevBuf();
            new (&rrecv[r]) DevBuf<uint32_t>();
            cudaStreamSynchronize(sh[r]->s);
            delete sh[r];
            if (ev[r]) cudaEventDestroy(ev[r]);
        }
    }
    // every stream waits for every other stream's work so far (device-side)
    void barrier() {
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(dev[r]));
            CK(cudaEventRecord(ev[r], sh[r]->s));
        }
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(dev[r]));
            for (uint32_t q = 0; q < P; ++q)
                if (q != r) CK(cudaStreamWaitEvent(sh[r]->s, ev[q], 0));
        }
    }
    // the owned graph rows (keys, flags, maxd) of every shard into shard
    // `only` (or every shard when only == ~0)
    void gather_rows(uint32_t only = ~0u) {
        barrier();
        const uint32_t k = sh[0]->e->k;
        for (uint32_t r = 0; r < P; ++r) {
            if (only != ~0u && r != only) continue;
            CK(cudaSetDevice(dev[r]));
            Engine& er = *sh[r]->e;
            for (uint32_t q = 0; q < P; ++q) {
                if (q == r) continue;
                const Engine& eq = *sh[q]->e;
                const uint32_t lo = eq.lo, hi = eq.hi;
                if (hi <= lo) continue;
                CK(cudaMemcpyPeerAsync(er.keys.p + size_t(lo) * k, dev[r], eq.keys.p + size_t(lo) * k,
                                       dev[q], sizeof(uint64_t) * size_t(hi - lo) * k, sh[r]->s));
                CK(cudaMemcpyPeerAsync(er.flags.p + lo, dev[r], eq.flags.p + lo, dev[q],
                                       sizeof(uint32_t) * (hi - lo), sh[r]->s));
                CK(cudaMemcpyPeerAsync(er.maxd.p + lo, dev[r], eq.maxd.p + lo, dev[q],
                                       sizeof(float) * (hi - lo), sh[r]->s));
            }
        }
        barrier();
    }
    // the owned maxd slice of every shard into every other shard
    void allgather_maxd() {
        barrier();
        const uint32_t chunk = sh[0]->chunk;
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(dev[r]));
            for (uint32_t q = 0; q < P; ++q) {
                if (q == r) continue;
                const uint32_t lo = sh[q]->e->lo, hi = sh[q]->e->hi;
                if (hi > lo)
                    CK(cudaMemcpyPeerAsync(sh[r]->e->maxd.p + lo, dev[r], sh[q]->e->maxd.p + lo,
                                           dev[q], sizeof(float) * (hi - lo), sh[r]->s));
            }
        }
        (void)chunk;
        barrier();
    }
};

__global__ void sum_partials_kernel(uint32_t* out, const uint32_t* parts, uint32_t P,
                                    uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s = 0;
    for (uint32_t q = 0; q < P; ++q) s += parts[size_t(q) * n + i];
    out[i] = s;
}

void run_multi(const float* data, uint32_t n, uint32_t d, const knng_cuda_params& p, int num_gpus,
               const int* devices, uint32_t* out_ids, float* out_dists,
               knng_cuda_metrics* m) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        raise(KNNG_CUDA_CUDA_ERROR, "no CUDA device available (this library has no CPU path)");
    }
    if (num_gpus < 1 || uint32_t(num_gpus) > kMaxShards)
        raise(KNNG_CUDA_INVALID_ARGUMENT, "num_gpus must be in [1, 1023]");
    int prev = 0;
    CK(cudaGetDevice(&prev));
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    MultiRun R;
    R.P = uint32_t(num_gpus);
    R.n = n;
    const uint32_t P = R.P;
    R.sh.assign(P, nullptr);
    R.dev.resize(P);
    R.ev.assign(P, nullptr);
    R.ipart.reset(new DevBuf<uint32_t>[P]);
    R.orecv.reset(new DevBuf<uint4>[P]);
    R.orecv_cap.assign(P, 0);
    R.rrecv.reset(new DevBuf<uint32_t>[P]);
    R.rrecv_cap.assign(P, 0);
    for (uint32_t r = 0; r < P; ++r) {
        R.dev[r] = devices ? devices[r] : int(r % uint32_t(ndev));
        if (R.dev[r] < 0 || R.dev[r] >= ndev)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "device ordinal out of range");
    }
    // peer access where the hardware has it (NVLink / NVSwitch)
    for (uint32_t r = 0; r < P; ++r)
        for (uint32_t q = 0; q < P; ++q) {
            if (R.dev[r] == R.dev[q]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, R.dev[r], R.dev[q]);
            if (can) {
                cudaSetDevice(R.dev[r]);
                const cudaError_t e = cudaDeviceEnablePeerAccess(R.dev[q], 0);
                if (e != cudaSuccess) cudaGetLastError();  // already enabled
            }
        }
    metrics_reset(m);
    const double t_start = now_s();
    for (uint32_t r = 0; r < P; ++r) {
        CK(cudaSetDevice(R.dev[r]));
        knng_cuda_params pr = p;
        pr.device = R.dev[r];
        R.sh[r] = shard_new(data, false, n, d, pr, r, P, nullptr, true);
        CK(cudaEventCreateWithFlags(&R.ev[r], cudaEventDisableTiming));
        R.ipart[r].alloc(size_t(P) * n, R.sh[r]->e->pool, R.sh[r]->s);
    }
    std::mt19937_64 master(p.seed);
    const uint64_t init_seed = master();
    for (uint32_t r = 0; r < P; ++r) {
        CK(cudaSetDevice(R.dev[r]));
        Engine& e = *R.sh[r]->e;
        const bool u8 = e.u8_state == 1;
        launch_init_random(e.gv(), init_seed, R.sh[r]->s, u8 ? e.packed.p : nullptr,
                           u8 ? e.lnorm.p : nullptr);
        CK(cudaGetLastError());
    }
    R.allgather_maxd();
    for (uint32_t r = 0; r < P; ++r) {
        CK(cudaSetDevice(R.dev[r]));
        CK(cudaStreamSynchronize(R.sh[r]->s));
    }
    double t1 = now_s();
    metrics_push(m, 0, t1 - t_start, uint64_t(n) * p.k, 0);
    const double threshold = p.termination_delta * double(n) * double(p.k);
    std::vector<uint64_t> counts(size_t(P) * P);
    bool reordered = false;
    std::vector<uint64_t> seeds(p.max_iterations + 1);
    for (uint32_t i = 1; i <= p.max_iterations; ++i) seeds[i] = master();  // reference order
    for (uint32_t it = 1; it <= p.max_iterations; ++it) {
        const double t0 = now_s();
        // degree: partials, then every shard sums all of them
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            R.sh[r]->enq_degree();
        }
        R.barrier();
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            for (uint32_t q = 0; q < P; ++q)
                CK(cudaMemcpyPeerAsync(R.ipart[r].p + size_t(q) * n, R.dev[r], R.sh[q]->e->indeg.p,
                                       R.dev[q], sizeof(uint32_t) * n, R.sh[r]->s));
        }
        R.barrier();  // nobody overwrites its partial before every shard copied it
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            sum_partials_kernel<<<(n + 255) / 256, 256, 0, R.sh[r]->s>>>(R.sh[r]->e->indeg.p,
                                                                         R.ipart[r].p, P, n);
            CK(cudaGetLastError());
            R.sh[r]->enq_sample(seeds[it]);
        }
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            R.sh[r]->fin_sample(counts.data() + size_t(r) * P);
        }
        // offers: shard q's segment for r -> r
        R.barrier();
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            uint64_t total = 0;
            for (uint32_t q = 0; q < P; ++q) total += counts[size_t(q) * P + r];
            if (total > R.orecv_cap[r]) {
                R.orecv[r].~DevBuf();
                new (&R.orecv[r]) DevBuf<uint4>();
                R.orecv_cap[r] = total + total / 4 + 1024;
                R.orecv[r].alloc(R.orecv_cap[r], R.sh[r]->e->pool, R.sh[r]->s);
            }
            uint64_t at = 0;
            for (uint32_t q = 0; q < P; ++q) {
                const uint64_t c = counts[size_t(q) * P + r];
                if (c)
                    CK(cudaMemcpyPeerAsync(R.orecv[r].p + at, R.dev[r],
                                           R.sh[q]->osend.p + size_t(r) * R.sh[q]->seg_cap,
                                           R.dev[q], sizeof(uint4) * c, R.sh[r]->s));
                at += c;
            }
            R.sh[r]->enq_offers(R.orecv[r].p, total);
            R.sh[r]->enq_step_join();
        }
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            R.sh[r]->fin_step_join();
        }
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            R.sh[r]->fin_step_export(counts.data() + size_t(r) * P);
        }
        // proposal records: shard q's records for r -> r (q's records are
        // grouped by target, hence by owner, in rank order)
        R.barrier();
        uint64_t evals = 0, cands = 0;
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            uint64_t total = 0;
            for (uint32_t q = 0; q < P; ++q) total += counts[size_t(q) * P + r];
            if (3 * total > R.rrecv_cap[r]) {
                R.rrecv[r].~DevBuf();
                new (&R.rrecv[r]) DevBuf<uint32_t>();
                R.rrecv_cap[r] = 3 * (total + total / 4 + 1024);
                R.rrecv[r].alloc(R.rrecv_cap[r], R.sh[r]->e->pool, R.sh[r]->s);
            }
            uint64_t at = 0;
            for (uint32_t q = 0; q < P; ++q) {
                const uint64_t c = counts[size_t(q) * P + r];
                uint64_t before = 0;
                for (uint32_t t = 0; t < r; ++t) before += counts[size_t(q) * P + t];
                if (c)
                    CK(cudaMemcpyPeerAsync(R.rrecv[r].p + 3 * at, R.dev[r],
                                           R.sh[q]->send.p + 3 * before, R.dev[q],
                                           sizeof(uint32_t) * 3 * c, R.sh[r]->s));
                at += c;
            }
            R.sh[r]->enq_merge(R.rrecv[r].p, total);
            evals += R.sh[r]->last.evals;
            cands += R.sh[r]->last.cands;
        }
        uint64_t changes = 0;
        for (uint32_t r = 0; r < P; ++r) {
            CK(cudaSetDevice(R.dev[r]));
            R.sh[r]->fin_merge();
            changes += R.sh[r]->last.changes;
        }
        R.allgather_maxd();
        // the locality reorder (descent.hpp:230-235): sigma from the whole
        // graph on shard 0, the data and the graph of every shard permuted;
        // the shards then own contiguous ranges of sigma, so graph
        // neighbours mostly share a shard
        if (p.reorder && !reordered && it == p.reorder_after_iteration) {
            R.gather_rows();
            CK(cudaSetDevice(R.dev[0]));
            R.sh[0]->e->compute_sigma();
            R.barrier();
            for (uint32_t r = 0; r < P; ++r) {
                CK(cudaSetDevice(R.dev[r]));
                Engine& er = *R.sh[r]->e;
                if (r && !er.sigma.p) {
                    er.sigma.alloc(n, er.pool, er.s);
                    er.sigma_inv.alloc(n, er.pool, er.s);
                }
                if (r) {
                    CK(cudaMemcpyPeerAsync(er.sigma.p, R.dev[r], R.sh[0]->e->sigma.p, R.dev[0],
                                           sizeof(uint32_t) * n, R.sh[r]->s));
                    CK(cudaMemcpyPeerAsync(er.sigma_inv.p, R.dev[r], R.sh[0]->e->sigma_inv.p,
                                           R.dev[0], sizeof(uint32_t) * n, R.sh[r]->s));
                }
            }
            R.barrier();
            for (uint32_t r = 0; r < P; ++r) {
                CK(cudaSetDevice(R.dev[r]));
                Engine& er = *R.sh[r]->e;
                const uint32_t lo0 = er.lo, hi0 = er.hi;
                er.lo = 0;
                er.hi = n;
                er.apply_sigma();  // data rows and every graph row
                er.lo = lo0;
                er.hi = hi0;
            }
            R.barrier();
            reordered = true;
        }
        const double wall = now_s() - t0;
        metrics_push(m, it, wall, evals, changes, cands, 0.0);
        if (m) {
            m->join_candidates += cands;
            m->join_evals += evals;
        }
        if (double(changes) < threshold) break;
    }
    if (reordered) {
        // back to the caller's ids (descent.hpp:245): every row on shard 0,
        // relabelled by sigma_inv, exported from there
        R.gather_rows(0);
        CK(cudaSetDevice(R.dev[0]));
        Engine& e0 = *R.sh[0]->e;
        e0.remap_all(e0.sigma_inv.p);
        const size_t cnt = size_t(n) * p.k;
        DevBuf<uint32_t> ids;
        DevBuf<float> dd;
        ids.alloc(cnt, e0.pool, e0.s);
        dd.alloc(cnt, e0.pool, e0.s);
        e0.export_rows(ids.p, dd.p, nullptr);
        copy_to_host({{out_ids, ids.p, sizeof(uint32_t) * cnt}, {out_dists, dd.p, sizeof(float) * cnt}},
                     e0.s);
    }
    // owned rows -> host
    for (uint32_t r = 0; r < P && !reordered; ++r) {
        CK(cudaSetDevice(R.dev[r]));
        knng_cuda_shard* s = R.sh[r];
        const uint32_t lo = s->e->lo, hi = s->e->hi;
        if (hi <= lo) continue;
        const size_t cnt = size_t(hi - lo) * p.k;
        DevBuf<uint32_t> ids;
        DevBuf<float> dd;
        ids.alloc(cnt, s->e->pool, s->s);
        dd.alloc(cnt, s->e->pool, s->s);
        s->e->export_owned(ids.p, dd.p, nullptr);
        copy_to_host({{out_ids + size_t(lo) * p.k, ids.p, sizeof(uint32_t) * cnt},
                      {out_dists + size_t(lo) * p.k, dd.p, sizeof(float) * cnt}},
                     s->s);
    }
    if (m) {
        uint64_t h2d = 0, d2h = 0;
        for (uint32_t r = 0; r < P; ++r) {
            h2d += R.sh[r]->e->h2d;
            d2h += R.sh[r]->e->d2h + sizeof(float) * 2 * size_t(R.sh[r]->e->hi - R.sh[r]->e->lo) * p.k;
            for (int kk = 0; kk < KNNG_CUDA_KERNEL_COUNT; ++kk) {
                m->kernel_ms[kk] += R.sh[r]->kmetrics.kernel_ms[kk];
                m->kernel_launches[kk] += R.sh[r]->kmetrics.kernel_launches[kk];
            }
        }
        m->h2d_bytes = h2d;
        m->d2h_bytes = d2h;
    }
}

}  // namespace

extern "C" int knng_cuda_run_multi(const float* data, uint32_t n, uint32_t d,
                                   const knng_cuda_params* params, int num_gpus,
                                   const int* devices, uint32_t* out_ids, float* out_dists,
                                   knng_cuda_metrics* out_metrics) {
    return guarded([&] {
        if (!params || !data || !out_ids || !out_dists)
            raise(KNNG_CUDA_INVALID_ARGUMENT, "null argument");
        run_multi(data, n, d, *params, num_gpus, devices, out_ids, out_dists, out_metrics);
    });
}
