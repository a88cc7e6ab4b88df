// capi.cu -- host orchestration and the C ABI of libbisim.so (include/bisim.h).
//
// One call = H2D (host entry points only) -> preprocessing kernels -> label
// pre-partition (cooperative kernel) -> refinement loop (one persistent
// cooperative kernel, or one launch per round when an observer is attached)
// -> D2H.  Device buffers live in a per-device context and are reused across
// calls; every call runs on the context's own stream and is timed with CUDA
// events on that stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/bisim.h"
#include "kernels.cuh"
#include "kernels_sparse.cuh"
#include "kernels_label.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace bisim {
namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

#define CK(expr)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw Error(BISIM_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* ensure(size_t bytes) {
        bytes = std::max<size_t>(bytes, 16);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Ctx {
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    int grid_refine_bcrp = 0, grid_refine_rcpp = 0, grid_label = 0, grid_label_common = 0;
    int grid_sparse_bcrp = 0, grid_sparse_rcpp = 0;
    std::mutex mu;
    DevBuf src, act, dst, pi0, lmask, off, rev_ptr, cursor, rev_slot, block, nl, mark, unstable,
        split_list, cmem, splits, ctrl, scan_tmp, rev2, members, bstart, bsize, tblock,
        small_list, big_list, big_base, tmp, scnt, kcur, scur, counter, brange, bar, trace, lhash, lkeys,
        lmins, sarr, big_list4, big_base4, big_info, big_info4, sinfo, nrm, bcur, stage, act8;
    uint8_t* act8_host = nullptr;     // pinned: host actions narrowed to bytes (pipelined input path)
    size_t act8_cap = 0;
    int launches = 0;
    struct Stager* stager = nullptr;  // pinned staging of pageable host arrays (lazy)
    cudaStream_t cstream = nullptr;   // host-to-device copies overlapping preprocessing
    std::vector<cudaEvent_t> pev;     // their events (lazy)
    ~Ctx();
};

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<Ctx>> g_ctx;

int occupancy_grid(const void* fn, int sms, int threads = kThreads, int max_per_sm = 2) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0));
    if (occ < 1) throw Error(BISIM_CUDA, "persistent kernel cannot be resident");
    return sms * std::min(occ, max_per_sm);
}

std::unique_ptr<Ctx> make_ctx(int device);

Ctx* get_ctx(int device) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        throw Error(BISIM_CUDA, "no CUDA device available (libbisim has no CPU fallback)");
    if (device < 0 || device >= count) throw Error(BISIM_CUDA, "invalid CUDA device ordinal");
    if ((int)g_ctx.size() < count) g_ctx.resize(count);
    if (!g_ctx[device]) g_ctx[device] = make_ctx(device);
    return g_ctx[device].get();
}

std::unique_ptr<Ctx> make_ctx(int device) {
    {
        auto c = std::make_unique<Ctx>();
        c->device = device;
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (!prop.cooperativeLaunch) throw Error(BISIM_CUDA, "device lacks cooperative launch");
        c->sms = prop.multiProcessorCount;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        c->grid_refine_bcrp = occupancy_grid((const void*)k_refine<false>, c->sms);
        c->grid_refine_rcpp = occupancy_grid((const void*)k_refine<true>, c->sms);
        c->grid_label = occupancy_grid((const void*)k_label_rounds, c->sms);
        c->grid_label_common = occupancy_grid((const void*)k_label_rounds_common, c->sms);
        c->grid_sparse_bcrp = occupancy_grid((const void*)k_refine_sparse<false, false>, c->sms, kSparseThreads, kSparsePerSm);
        c->grid_sparse_rcpp = occupancy_grid((const void*)k_refine_sparse<true, false>, c->sms, kSparseThreads, kSparsePerSm);
        return c;
    }
}

// ---- host <-> device copies of caller arrays ------------------------------
//
// Pinned (page-locked) host arrays go straight to cudaMemcpyAsync.  Pageable
// arrays -- what a Python caller normally passes -- are staged: the array is
// split over T worker threads, each owning two pinned chunk buffers and a
// stream; a worker memcpy's chunk k into one buffer while the DMA of chunk
// k-1 drains from the other, so T host copies run beside the DMA engine
// instead of the driver's single staging pipeline.
struct Stager {
    static constexpr size_t kChunk = 8u << 20;
    int T = 0;
    std::vector<void*> buf;             // 2 per worker
    std::vector<cudaStream_t> streams;  // 1 per worker
    std::vector<cudaEvent_t> done;      // 2 per worker (buffer free again)
    std::vector<cudaEvent_t> fin;       // 1 per worker
    cudaEvent_t start = nullptr;
};

Stager& stager(Ctx& c) {
    if (c.stager) return *c.stager;
    auto* S = new Stager();
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    S->T = (int)std::max(1u, std::min(8u, hw / 2));
    if (const char* e = getenv("BISIM_DEV") ? getenv("BISIM_STAGE_THREADS") : nullptr) S->T = std::max(1, atoi(e));
    S->buf.resize(2 * S->T);
    S->streams.resize(S->T);
    S->done.resize(2 * S->T);
    S->fin.resize(S->T);
    for (auto& b : S->buf) CK(cudaHostAlloc(&b, Stager::kChunk, cudaHostAllocPortable));
    for (auto& st : S->streams) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : S->done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : S->fin) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S->start, cudaEventDisableTiming));
    c.stager = S;
    return *S;
}

Ctx::~Ctx() {
    // errors are ignored: at process exit the runtime may already be gone
    cudaSetDevice(device);
    if (stager) {
        for (void* b : stager->buf) cudaFreeHost(b);
        for (auto st : stager->streams) cudaStreamDestroy(st);
        for (auto e : stager->done) cudaEventDestroy(e);
        for (auto e : stager->fin) cudaEventDestroy(e);
        if (stager->start) cudaEventDestroy(stager->start);
        delete stager;
    }
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    for (auto e : pev) cudaEventDestroy(e);
    if (act8_host) cudaFreeHost(act8_host);
    if (cstream) cudaStreamDestroy(cstream);
    if (stream) cudaStreamDestroy(stream);
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// Staged copy of `bytes` between host `h` and device `d` (dir = H2D / D2H),
// ordered after the work already queued on `st`; on return the copies are
// queued (H2D) or complete (D2H), and `st` waits for them.
void staged_copy(Ctx& c, void* d, void* h, size_t bytes, cudaMemcpyKind dir, cudaStream_t st) {
    if (bytes < (size_t)4 * Stager::kChunk || host_pinned(h)) {
        CK(cudaMemcpyAsync(dir == cudaMemcpyHostToDevice ? d : h, dir == cudaMemcpyHostToDevice ? h : d, bytes,
                           dir, st));
        if (dir == cudaMemcpyDeviceToHost) CK(cudaStreamSynchronize(st));
        return;
    }
    Stager& S = stager(c);
    CK(cudaEventRecord(S.start, st));
    const size_t per = ((bytes + S.T - 1) / S.T + 4095) & ~(size_t)4095;
    std::vector<cudaError_t> err(S.T, cudaSuccess);
    auto work = [&](int t) {
        cudaError_t e = cudaSetDevice(c.device);
        cudaStream_t ws = S.streams[t];
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ws, S.start, 0);
        const size_t lo = std::min(bytes, (size_t)t * per), hi = std::min(bytes, lo + per);
        size_t prev_off = 0, prev_len = 0;
        int k = 0;
        for (size_t off = lo; off < hi && e == cudaSuccess; off += Stager::kChunk, ++k) {
            const size_t len = std::min(Stager::kChunk, hi - off);
            const int slot = 2 * t + (k & 1);
            char* b = (char*)S.buf[slot];
            if (dir == cudaMemcpyHostToDevice) {
                e = cudaEventSynchronize(S.done[slot]);  // the DMA out of this buffer finished
                if (e != cudaSuccess) break;
                memcpy(b, (const char*)h + off, len);
                e = cudaMemcpyAsync((char*)d + off, b, len, dir, ws);
                if (e == cudaSuccess) e = cudaEventRecord(S.done[slot], ws);
            } else {
                e = cudaMemcpyAsync(b, (const char*)d + off, len, dir, ws);
                if (e == cudaSuccess) e = cudaEventRecord(S.done[slot], ws);
                if (e == cudaSuccess && k > 0) {  // drain the previous chunk while this one flies
                    const int ps = 2 * t + ((k - 1) & 1);
                    e = cudaEventSynchronize(S.done[ps]);
                    if (e == cudaSuccess) memcpy((char*)h + prev_off, S.buf[ps], prev_len);
                }
                prev_off = off;
                prev_len = len;
            }
        }
        if (e == cudaSuccess && dir == cudaMemcpyDeviceToHost && prev_len) {
            const int ps = 2 * t + ((k - 1) & 1);
            e = cudaEventSynchronize(S.done[ps]);
            if (e == cudaSuccess) memcpy((char*)h + prev_off, S.buf[ps], prev_len);
        }
        if (e == cudaSuccess) e = cudaEventRecord(S.fin[t], ws);
        err[t] = e;
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < S.T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < S.T; ++t) {
        if (err[t] != cudaSuccess) CK(err[t]);
        CK(cudaStreamWaitEvent(st, S.fin[t], 0));
    }
}

void h2d(Ctx& c, void* d, const void* h, size_t bytes, cudaStream_t st) {
    if (bytes) staged_copy(c, d, const_cast<void*>(h), bytes, cudaMemcpyHostToDevice, st);
}

// Complete on return.
void d2h(Ctx& c, void* h, const void* d, size_t bytes, cudaStream_t st) {
    if (bytes) staged_copy(c, const_cast<void*>(d), h, bytes, cudaMemcpyDeviceToHost, st);
}

int grid_for(int64_t work, int threads, int sms) {
    const int64_t g = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

void scan_excl(Ctx& c, int32_t* d, int64_t N) {
    // d[0..N) counts -> exclusive prefix, d[N] = total
    const int64_t ntiles = std::max<int64_t>(1, (N + kScanTile - 1) / kScanTile);
    int64_t* tiles = (int64_t*)c.scan_tmp.ensure(ntiles * sizeof(int64_t));
    k_scan_tiles<<<(unsigned)ntiles, kScanThreads, 0, c.stream>>>(d, N, tiles);
    k_scan_sums<<<1, kScanThreads, 0, c.stream>>>(tiles, ntiles);
    k_scan_apply<<<(unsigned)ntiles, kScanThreads, 0, c.stream>>>(d, N, tiles);
    c.launches += 3;
    CK(cudaGetLastError());
}

struct Job {
    bool bcrp = true;
    int32_t n = 0;
    int64_t m = 0;
    int32_t A = 0;
    const int32_t *src = nullptr, *act = nullptr, *dst = nullptr, *pi0 = nullptr;
    bool inputs_on_device = false;
    int64_t max_supersteps = BISIM_DEFAULT_GUARD;
    int32_t* block_out = nullptr;
    bool block_out_on_device = false;
    int32_t* splits_out = nullptr;
    int64_t splits_cap = 0;
    bisim_stats* st = nullptr;
    bisim_options opt{};
    // transition-sharded mode (sharded.cuh): reverse CSR over sources in
    // [src_lo, src_hi) only, double-buffered round state, and run() stops
    // after the setup, handing the loop parameters to the caller
    int32_t src_lo = 0, src_hi = -1;
    struct ShardPrep* prep = nullptr;
};

// What run() leaves for the sharded driver when Job::prep is set.
struct ShardPrep {
    SparseParams sp{};
    bisim_stats S{};
    int64_t guard = 0;
    int64_t splits_dev_cap = 0;
    int32_t* block = nullptr;
    int32_t* splits = nullptr;
    int32_t* leaders = nullptr;
    int64_t mark_words = 0, bm_words = 0;
};

template <typename T>
T* as(DevBuf& b) {
    return reinterpret_cast<T*>(b.p);
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// Status of a refinement-loop launch, mode independent.
struct LoopStatus {
    int64_t round = 0;
    int32_t done = 0, error = 0;
    int64_t guard_count = 0;
    unsigned long long work_edges = 0, work_members = 0, work_splits = 0, retired = 0;
};

// Algorithmic bytes of the refinement loop ("Roofline"): the
// bytes a round must move at minimum, each element counted once.
int64_t loop_bytes(bool bcrp, bool dense, int32_t n, int64_t L, int64_t R, const LoopStatus& ls) {
    const int64_t nwords = ((int64_t)n + 31) / 32;
    if (dense) {
        // per round: block[] twice, off[s], off[s+1], off[leader], mark words
        // of s and leader, unstable scan; per in-edge of C slot + mark set/clear
        const int64_t per_round = bcrp ? (int64_t)n * 20 + L / 8 * 2 + nwords * 4 : (int64_t)n * 8 + nwords * 12;
        return (R + 1) * per_round + (int64_t)ls.work_edges * 16 + (int64_t)ls.work_splits * 28;
    }
    // per round: C's range and control words; per in-edge of C: the packed
    // reverse edge, mark read-modify-write, source block id;
    // per member of a touched block: member id, mark bits, slot
    // offsets, compaction write and block id write.
    const int64_t per_edge = bcrp ? 8 + 8 + 4 : 4 + 8 + 4;
    const int64_t per_member = bcrp ? 4 + 4 + 8 + 4 + 4 + 4 : 4 + 4 + 4 + 4;
    return (R + 1) * 64 + (int64_t)ls.work_edges * per_edge + (int64_t)ls.work_members * per_member;
}

// Developer tuning knobs (kernel-variant sweeps, tracing): read only when
// BISIM_DEV=1, so a production call never depends on the environment.
const char* dev_env(const char* name) { return getenv("BISIM_DEV") ? getenv(name) : nullptr; }

// Label pre-partition (bcrp.py:144-184) into block[]: canonical grouping by
// a verified 64-bit hash of each state's label set (kernels_label.cuh); a
// hash collision -- or `literal` -- runs the literal |Act| mark-and-split
// rounds in one cooperative kernel instead.  Both give the same canonical
// pi0 (states grouped by outgoing label set, min-id leaders).
void label_partition_dev(Ctx& c, int32_t n, int32_t A, const unsigned long long* lmask, int32_t* block,
                         bool literal) {
    cudaStream_t st = c.stream;
    const int32_t W = (A + 63) / 64;
    const int TB = 256;
    CK(cudaMemsetAsync(block, 0, (int64_t)n * 4, st));
    if (A == 0) return;
    if (!literal) {
        uint64_t T = 1024;
        while (T < 2ull * (uint64_t)n) T <<= 1;
        auto* h = (unsigned long long*)c.lhash.ensure((int64_t)n * 8);
        auto* keys = (unsigned long long*)c.lkeys.ensure(T * 8);
        auto* mins = (int32_t*)c.lmins.ensure(T * 4 + 4);
        int32_t* mismatch = mins + T;
        CK(cudaMemsetAsync(keys, 0, T * 8, st));
        CK(cudaMemsetAsync(mins, 0x7f, T * 4 + 4, st));
        CK(cudaMemsetAsync(mismatch, 0, 4, st));
        k_label_hash<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, W, lmask, h);
        k_label_insert<<<c.sms * 2, 512, 0, st>>>(n, h, keys, mins, T - 1);
        k_label_assign<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, W, h, keys, mins, T - 1, lmask, block,
                                                              mismatch);
        c.launches += 3;
        int32_t hm = 0;
        CK(cudaMemcpyAsync(&hm, mismatch, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        literal = hm != 0;
        if (literal) CK(cudaMemsetAsync(block, 0, (int64_t)n * 4, st));
    }
    if (literal) {
        unsigned long long* nl = (unsigned long long*)c.nl.ensure((int64_t)n * 8);
        CK(cudaMemsetAsync(nl, 0, (int64_t)n * 8, st));
        int32_t nn = n, AA = A;
        const unsigned long long* lm = lmask;
        void* args[] = {&nn, &AA, (void*)&lm, &block, &nl};
        CK(cudaLaunchCooperativeKernel((const void*)k_label_rounds, c.grid_label, kThreads, args, 0, st));
        ++c.launches;
    }
}

// Error mapping for the table entry points (same codes as the loop calls).
template <typename F>
int guarded_call(F&& f) {
    try {
        g_last_error.clear();
        f();
        return BISIM_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BISIM_CUDA;
    }
}

// Device label tables of a host transition list: inputs copied, validated
// (read back BEFORE anything indexes by them), label masks, nr_marks and
// off = exclusive scan (bcrp.py:91-113).
struct LabelTables {
    const int32_t *src = nullptr, *act = nullptr, *dst = nullptr;
    unsigned long long* lmask = nullptr;
    int32_t* nr = nullptr;   // nr_marks[n]
    int32_t* off = nullptr;  // off[n+1]
    int64_t L = 0;
};

LabelTables label_tables(Ctx& c, int32_t n, int64_t m, int32_t A, const int32_t* src, const int32_t* act,
                         const int32_t* dst = nullptr) {
    if (n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
    if (m < 0 || m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
    if (A < 0) throw Error(BISIM_BAD_INPUT, "negative action count");
    if (n >= (1 << 30)) throw Error(BISIM_BAD_INPUT, "state count above 2^30 is not supported");
    if (m > 0 && (!src || !act)) throw Error(BISIM_BAD_INPUT, "null transition array");
    CK(cudaSetDevice(c.device));
    c.launches = 0;
    cudaStream_t st = c.stream;
    const int TB = 256;
    const int64_t mm = std::max<int64_t>(m, 1);
    const int32_t W = std::max((A + 63) / 64, 1);
    LabelTables t;
    int32_t* d_src = (int32_t*)c.src.ensure(mm * 4);
    int32_t* d_act = (int32_t*)c.act.ensure(mm * 4);
    int32_t* d_dst = dst ? (int32_t*)c.dst.ensure(mm * 4) : d_src;
    h2d(c, d_src, src, m * 4, st);
    h2d(c, d_act, act, m * 4, st);
    if (dst) h2d(c, d_dst, dst, m * 4, st);
    Ctrl* ctrl = (Ctrl*)c.ctrl.ensure(std::max(sizeof(Ctrl), sizeof(SCtrl)));
    t.lmask = (unsigned long long*)c.lmask.ensure((size_t)W * n * 8);
    CK(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), st));
    CK(cudaMemsetAsync(t.lmask, 0, (size_t)W * n * 8, st));
    // k_label_mask checks src/act/dst ranges (dst := src when not given)
    if (m) k_label_mask<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, A, d_src, d_act, d_dst, t.lmask, ctrl);
    int32_t bad = 0;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&bad, &ctrl->bad, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad) throw Error(BISIM_BAD_INPUT, "transition mentions a state or action outside range");
    t.nr = (int32_t*)c.nrm.ensure((int64_t)n * 4);
    t.off = (int32_t*)c.off.ensure(((int64_t)n + 1) * 4);
    k_nr_marks<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, W, t.lmask, t.off);
    CK(cudaMemcpyAsync(t.nr, t.off, (int64_t)n * 4, cudaMemcpyDeviceToDevice, st));
    scan_excl(c, t.off, n);
    int32_t L32 = 0;
    CK(cudaMemcpyAsync(&L32, t.off + n, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    t.L = L32;
    t.src = d_src;
    t.act = d_act;
    t.dst = dst ? d_dst : nullptr;
    return t;
}

// Host-input pipelining of large labelled systems (run_with): chunks of the
// src / act copies overlap the per-transition passes.
constexpr int64_t kPipeMin = 1 << 22;
constexpr int kPipeChunks = 8;
cudaEvent_t* pipe_events(Ctx& c) {
    if (c.pev.empty()) {
        c.pev.resize(kPipeChunks + 2);
        for (auto& e : c.pev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return c.pev.data();
}

// Host threads narrowing the caller's int32 actions to bytes in the
// context's pinned buffer, chunk by chunk in order (the pipelined input path
// DMAs chunk k as soon as its slices are done).
struct ActPacker {
    static constexpr int kSlices = 8;  // work units per chunk
    std::vector<std::thread> th;
    std::atomic<int> next{0};
    std::atomic<int> done[kPipeChunks];
    std::atomic<bool> bad_flag{false};
    bool bad = false;
    int64_t m = 0, chunk = 0;
    ActPacker() {
        for (auto& d : done) d.store(0);
    }
    void start(Ctx& c, const int32_t* act, int64_t m_, int64_t chunk_) {
        m = m_;
        chunk = chunk_;
        if (c.act8_cap < (size_t)m) {
            if (c.act8_host) CK(cudaFreeHost(c.act8_host));
            c.act8_host = nullptr;
            c.act8_cap = 0;
            CK(cudaHostAlloc((void**)&c.act8_host, (size_t)m, cudaHostAllocPortable));
            c.act8_cap = (size_t)m;
        }
        uint8_t* out = c.act8_host;
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        int T = (int)std::max(1u, std::min(8u, hw / 2));
        if (const char* e = dev_env("BISIM_PACK_THREADS")) T = std::max(1, atoi(e));
        for (int t = 0; t < T; ++t)
            th.emplace_back([this, act, out] {
                bool b = false;
                for (;;) {
                    const int u = next.fetch_add(1, std::memory_order_relaxed);
                    if (u >= kPipeChunks * kSlices) break;
                    const int k = u / kSlices, q = u % kSlices;
                    const int64_t c0 = k * chunk, c1 = std::min<int64_t>(c0 + chunk, m);
                    const int64_t per = (chunk + kSlices - 1) / kSlices;
                    const int64_t lo = std::min<int64_t>(c0 + q * per, c1), hi = std::min<int64_t>(lo + per, c1);
                    uint32_t any = 0;
                    for (int64_t i = lo; i < hi; ++i) {
                        const uint32_t v = (uint32_t)act[i];
                        any |= v;
                        out[i] = (uint8_t)v;
                    }
                    b |= (any >> 8) != 0;  // some action outside 0..255
                    done[k].fetch_add(1, std::memory_order_release);
                }
                if (b) bad_flag.store(true);
            });
    }
    void wait(int k) {
        while (done[k].load(std::memory_order_acquire) < kSlices) std::this_thread::yield();
    }
    void join() {
        for (auto& t : th) t.join();
        th.clear();
        bad = bad_flag.load();
    }
    ~ActPacker() {
        for (auto& t : th)
            if (t.joinable()) t.join();
    }
};

int run_with(Ctx& c, Job& j);

int run(Job& j) { return run_with(*get_ctx(j.opt.device), j); }

int run_with(Ctx& c, Job& j) {
    if (j.n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
    if (j.m < 0 || j.m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
    if (j.A < 0) throw Error(BISIM_BAD_INPUT, "negative action count");
    if (j.n >= (1 << 30)) throw Error(BISIM_BAD_INPUT, "state count above 2^30 is not supported");
    if (j.m > 0 && (!j.src || !j.dst || (j.bcrp && !j.act)))
        throw Error(BISIM_BAD_INPUT, "null transition array");
    if (!j.bcrp && !j.pi0) throw Error(BISIM_BAD_INPUT, "null pi0");
    if (!j.block_out) throw Error(BISIM_BAD_INPUT, "null block_out");

    std::lock_guard<std::mutex> lock(c.mu);
    CK(cudaSetDevice(c.device));
    c.launches = 0;
    cudaStream_t st = c.stream;
    const int32_t n = j.n;
    const int64_t m = j.m;
    const int32_t A = j.bcrp ? j.A : 0;
    const int32_t W = j.bcrp ? (A + 63) / 64 : 0;
    const int64_t guard = j.max_supersteps == BISIM_DEFAULT_GUARD
                              ? (j.bcrp ? 3LL * n + A + 8 : 3LL * n + 9)
                              : j.max_supersteps;
    const bool sharded = j.prep != nullptr;
    const bool stepped = !sharded && (j.opt.observer != nullptr || j.opt.mode == BISIM_MODE_STEPPED);
    const bool dense = !sharded && j.opt.mode == BISIM_MODE_DENSE;
    const int32_t src_lo = sharded ? j.src_lo : 0, src_hi = sharded ? j.src_hi : n;
    bisim_stats S{};
    S.label_rounds = A;
    S.mode = stepped ? BISIM_MODE_STEPPED : (dense ? BISIM_MODE_DENSE : BISIM_MODE_PERSISTENT);

    // ---- buffers
    const int64_t mm = std::max<int64_t>(m, 1);
    Ctrl* ctrl = (Ctrl*)c.ctrl.ensure(std::max(sizeof(Ctrl), sizeof(SCtrl)));
    unsigned long long* lmask =
        j.bcrp ? (unsigned long long*)c.lmask.ensure((size_t)std::max(W, 1) * n * 8) : nullptr;
    int32_t* off = j.bcrp ? (int32_t*)c.off.ensure(((int64_t)n + 1) * 4) : nullptr;
    int32_t* rev_ptr = (int32_t*)c.rev_ptr.ensure(((int64_t)n + 1) * 4);
    int32_t* cursor = (int32_t*)c.cursor.ensure(((int64_t)n + 1) * 4);
    int32_t* block = (int32_t*)c.block.ensure((int64_t)n * 4);
    const int64_t mark_bits = j.bcrp ? m : n;  // L <= m (bcrp.py:113)
    const int64_t mark_words = (mark_bits + 31) / 32 + 2;
    const int parities = sharded ? 2 : 1;  // sharded: one buffer per round parity
    uint32_t* mark = (uint32_t*)c.mark.ensure(parities * mark_words * 4);
    const int64_t nwords = ((int64_t)n + 31) / 32;
    // rounds can never exceed the guard nor the 3n bound of the paper
    const int64_t splits_dev_cap =
        std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(guard - A, 1), 3LL * n + 16));
    int32_t* splits = (int32_t*)c.splits.ensure(splits_dev_cap * 4);
    int32_t* rev_slot = nullptr;  // dense: slot per in-edge
    int2* rev2 = nullptr;         // sparse BCRP: (slot, source)
    int32_t* rev_src = nullptr;   // sparse RCPP: source
    if (dense) rev_slot = (int32_t*)c.rev_slot.ensure(mm * 4);
    else if (j.bcrp) rev2 = (int2*)c.rev2.ensure(mm * 8);
    else rev_src = (int32_t*)c.rev_slot.ensure(mm * 4);
    // sparse modes: reverse CSR through the bucketed staging array
    // (kernels_sparse.cuh k_rev_bucket / k_rev_place), <= 256 target buckets
    int shift = 0;
    while (((int64_t)n >> shift) >= 256) ++shift;
    const int32_t nb = (int32_t)(((int64_t)n - 1) >> shift) + 1;
    int32_t* bcur = dense ? nullptr : (int32_t*)c.bcur.ensure((int64_t)nb * 4);
    int4* stage = dense ? nullptr : (int4*)c.stage.ensure(mm * 16);
    auto bucket_pass = [&](int64_t len, const int32_t* s_, auto a_, const int32_t* d_, int32_t lo,
                           int32_t hi, bool slot_here, const int4* si, const int2* si2) {
        if (len <= 0) return;
        const int64_t tiles = (len + kBucketTile - 1) / kBucketTile;
        const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)c.sms * 4));
        k_rev_bucket<<<g1, kBucketThreads, 0, st>>>(len, s_, a_, d_, shift, nb, bcur, stage, lo, hi, slot_here, n,
                                                    si, lmask, off, si2);
        ++c.launches;
    };
    auto rev_ptr_scan = [&]() {
        scan_excl(c, rev_ptr, n);
        CK(cudaMemcpyAsync(cursor, rev_ptr, ((int64_t)n + 1) * 4, cudaMemcpyDeviceToDevice, st));
        if (!dense) {
            k_bucket_init<<<(nb + 255) / 256, 256, 0, st>>>(n, shift, nb, rev_ptr, bcur);
            ++c.launches;
        }
    };

    // ---- inputs + preprocessing (bcrp.py:49-126)
    const int TB = 256;
    const int32_t* d_src;
    const int32_t* d_act = nullptr;
    const int32_t* d_dst;
    const int32_t* d_pi0 = nullptr;
    // A large labelled system from host memory: the copies of src / act
    // overlap the per-transition passes (label sets, target buckets) of the
    // chunks already on the device; dst goes first, its in-degrees fix the
    // bucket layout.
    const bool pipe = j.bcrp && !j.inputs_on_device && !sharded && !dense && m >= kPipeMin;
    bool host_bad = false;  // the host narrowing of the actions met one outside 0..255
    CK(cudaEventRecord(c.ev[0], st));
    CK(cudaMemsetAsync(ctrl, 0, std::max(sizeof(Ctrl), sizeof(SCtrl)), st));
    CK(cudaMemsetAsync(rev_ptr, 0, ((int64_t)n + 1) * 4, st));
    if (j.bcrp) CK(cudaMemsetAsync(lmask, 0, (size_t)std::max(W, 1) * n * 8, st));
    if (pipe) {
        int32_t* ds = (int32_t*)c.src.ensure(mm * 4);
        int32_t* dd = (int32_t*)c.dst.ensure(mm * 4);
        int32_t* da = (int32_t*)c.act.ensure(mm * 4);
        d_src = ds;
        d_dst = dd;
        d_act = da;
        cudaStream_t cs = c.cstream;
        cudaEvent_t* pev = pipe_events(c);
        CK(cudaEventRecord(pev[0], st));  // the buffers' previous readers are done
        CK(cudaStreamWaitEvent(cs, pev[0], 0));
        h2d(c, dd, j.dst, m * 4, cs);
        CK(cudaEventRecord(pev[1], cs));
        CK(cudaStreamWaitEvent(st, pev[1], 0));
        CK(cudaEventRecord(c.ev[1], st));
        k_indeg_checked<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, dd, rev_ptr, ctrl);
        ++c.launches;
        rev_ptr_scan();
        const int64_t chunk = (m + kPipeChunks - 1) / kPipeChunks;
        // |Act| <= 256: host threads narrow the actions to bytes in pinned
        // memory, chunk by chunk ahead of the DMA, so a quarter of their
        // bytes cross PCIe (an action outside 0..255 is flagged here, one in
        // A..255 by k_label_mask, as before)
        const bool narrow = A <= 256 && !dev_env("BISIM_NO_NARROW");
        ActPacker pk;
        if (narrow) pk.start(c, j.act, m, chunk);
        uint8_t* da8 = narrow ? (uint8_t*)c.act8.ensure(mm) : nullptr;
        for (int k = 0; k < kPipeChunks; ++k) {
            const int64_t i0 = k * chunk, len = std::min<int64_t>(chunk, m - i0);
            if (len <= 0) break;
            h2d(c, ds + i0, j.src + i0, len * 4, cs);
            if (narrow) {
                pk.wait(k);
                CK(cudaMemcpyAsync(da8 + i0, c.act8_host + i0, len, cudaMemcpyHostToDevice, cs));
            } else {
                h2d(c, da + i0, j.act + i0, len * 4, cs);
            }
            CK(cudaEventRecord(pev[2 + k], cs));
            CK(cudaStreamWaitEvent(st, pev[2 + k], 0));
            if (narrow) {
                k_label_mask<<<grid_for(len, TB, c.sms), TB, 0, st>>>(n, len, A, ds + i0, (const uint8_t*)da8 + i0,
                                                                      dd + i0, lmask, ctrl);
                ++c.launches;
                bucket_pass(len, ds + i0, (const uint8_t*)da8 + i0, dd + i0, 0, n, false, nullptr, nullptr);
            } else {
                k_label_mask<<<grid_for(len, TB, c.sms), TB, 0, st>>>(n, len, A, ds + i0, (const int32_t*)da + i0,
                                                                      dd + i0, lmask, ctrl);
                ++c.launches;
                bucket_pass(len, ds + i0, (const int32_t*)da + i0, dd + i0, 0, n, false, nullptr, nullptr);
            }
        }
        if (narrow) {
            pk.join();
            if (pk.bad) host_bad = true;
        }
    } else {
        if (j.inputs_on_device) {
            d_src = j.src;
            d_act = j.act;
            d_dst = j.dst;
            d_pi0 = j.pi0;
        } else {
            d_src = (int32_t*)c.src.ensure(mm * 4);
            d_dst = (int32_t*)c.dst.ensure(mm * 4);
            h2d(c, (void*)d_src, j.src, m * 4, st);
            h2d(c, (void*)d_dst, j.dst, m * 4, st);
            if (j.bcrp) {
                d_act = (int32_t*)c.act.ensure(mm * 4);
                h2d(c, (void*)d_act, j.act, m * 4, st);
            } else {
                d_pi0 = (int32_t*)c.pi0.ensure((int64_t)n * 4);
                h2d(c, (void*)d_pi0, j.pi0, (int64_t)n * 4, st);
            }
        }
        CK(cudaEventRecord(c.ev[1], st));
        if (j.bcrp) {
            if (m) {
                k_label_mask<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, A, d_src, d_act, d_dst, lmask, ctrl);
                ++c.launches;
            }
        } else {
            if (m) {
                k_check_edges<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, d_src, d_dst, ctrl);
                ++c.launches;
            }
            k_check_pi0<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, d_pi0, ctrl);
            ++c.launches;
        }
    }
    // Validation must finish before anything indexes by a source or action
    // (in-degrees, slots, the reverse fill): read the flag back here.
    {
        int32_t bad = 0;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&bad, &ctrl->bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (bad || host_bad)
            throw Error(BISIM_BAD_INPUT, j.bcrp ? "transition mentions a state or action outside range"
                                                : "edge outside 0..n-1 or pi0 is not a leader-form partition");
    }
    int4* sinfo = nullptr;
    int2* sinfo2 = nullptr;
    if (j.bcrp) {
        k_nr_marks<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, W, lmask, off);
        ++c.launches;
        scan_excl(c, off, n);
        if (A <= 32 && !dense) {
            sinfo2 = (int2*)c.sinfo.ensure((int64_t)n * 8);
            k_pack_sinfo2<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, lmask, off, sinfo2);
            ++c.launches;
        } else if (W == 1 && !dense) {
            sinfo = (int4*)c.sinfo.ensure((int64_t)n * 16);
            k_pack_sinfo<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, lmask, off, sinfo);
            ++c.launches;
        }
    }
    // the mark slot goes into the staging array in pass 1 when the label
    // sets are already complete (every path but the pipelined one)
    const bool slot_staged = !pipe && j.bcrp;
    if (!pipe) {
        if (m) {
            k_indeg<<<grid_for(m, TB, c.sms), TB, 0, st>>>(m, d_dst, rev_ptr, sharded ? d_src : nullptr, src_lo,
                                                           src_hi);
            ++c.launches;
        }
        rev_ptr_scan();
        if (!dense) bucket_pass(m, d_src, d_act, d_dst, src_lo, src_hi, slot_staged, sinfo, sinfo2);
    }
    if (m) {
        if (dense) {
            const int g = grid_for(m, TB, c.sms);
            if (j.bcrp) k_rev_fill<true><<<g, TB, 0, st>>>(n, m, d_src, d_act, d_dst, lmask, off, cursor, rev_slot);
            else k_rev_fill<false><<<g, TB, 0, st>>>(n, m, d_src, d_act, d_dst, lmask, off, cursor, rev_slot);
        } else {
            // exactly the resident number of CTAs: the grid-stride sweep then
            // moves through the staging array as one wave, so the positions
            // being written stay within a few MB (an oversubscribed grid
            // sweeps twice, half a window each, and sectors leave L2
            // half-written)
            const void* fn = !j.bcrp    ? (const void*)k_rev_place<false, false>
                             : slot_staged ? (const void*)k_rev_place<true, true>
                                           : (const void*)k_rev_place<true, false>;
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0));
            const int g2 =
                (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.sms * std::max(occ, 1), (m + 255) / 256));
            if (!j.bcrp)
                k_rev_place<false, false><<<g2, 256, 0, st>>>(rev_ptr + n, stage, cursor, nullptr, rev_src, n, nullptr,
                                                              nullptr, nullptr);
            else if (slot_staged)
                k_rev_place<true, true><<<g2, 256, 0, st>>>(rev_ptr + n, stage, cursor, rev2, nullptr, n, lmask, off,
                                                            sinfo, sinfo2);
            else
                k_rev_place<true, false><<<g2, 256, 0, st>>>(rev_ptr + n, stage, cursor, rev2, nullptr, n, lmask,
                                                             off, sinfo, sinfo2);
        }
        ++c.launches;
    }
    CK(cudaGetLastError());
    int32_t L32 = n;
    if (j.bcrp) CK(cudaMemcpyAsync(&L32, off + n, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(c.ev[2], st));
    CK(cudaStreamSynchronize(st));
    S.mark_length = L32;

    // ---- label pre-partition (bcrp.py:144-184) / pi0 (rcpp.py:58-72)
    if (j.bcrp && A > 0 && guard < A) {
        // PramEngine.begin_superstep of label round guard+1 (pram.py:195-200)
        S.guard_count = std::max<int64_t>(guard + 1, 1);
        *j.st = S;
        throw Error(BISIM_GUARD, "superstep guard exceeded (" + std::to_string(S.guard_count) + " > " +
                                     std::to_string(guard) + ")");
    }
    unsigned long long* nl = (unsigned long long*)c.nl.ensure((int64_t)n * 8);
    if (j.bcrp) {
        label_partition_dev(c, n, A, lmask, block, (j.opt.flags & BISIM_FLAG_LITERAL_LABEL_ROUNDS) != 0);
    } else {
        CK(cudaMemcpyAsync(block, d_pi0, (int64_t)n * 4, cudaMemcpyDeviceToDevice, st));
    }
    // unstable := leaders of the initial partition (level 0 of the set)
    const int32_t nw0 = (int32_t)nwords, nw1 = (int32_t)((n + 32767) / 32768), nw2 = (int32_t)((n + (1 << 25) - 1) >> 25);
    uint32_t* U = (uint32_t*)c.unstable.ensure(((int64_t)nw0 + nw1 + nw2 + 3) * 4);
    CK(cudaMemsetAsync(U, 0, ((int64_t)nw0 + nw1 + nw2 + 3) * 4, st));
    k_init_unstable<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, block, U);
    int32_t* leaders = (int32_t*)c.counter.ensure(16);
    int32_t h_leaders = 0;
    CK(cudaMemsetAsync(leaders, 0, 4, st));
    k_count_leaders<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, block, leaders);
    c.launches += 2;
    CK(cudaMemcpyAsync(&h_leaders, leaders, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(mark, 0, parities * mark_words * 4, st));
    CK(cudaMemsetAsync(splits, 0, splits_dev_cap * 4, st));

    // ---- loop state
    SparseParams sp{};
    LoopParams lp{};
    if (dense) {
        int32_t* split_list = (int32_t*)c.split_list.ensure((int64_t)n * 4);
        int32_t* cmem = (int32_t*)c.cmem.ensure((int64_t)n * 4);
        CK(cudaMemsetAsync(nl, 0, (int64_t)n * 8, st));
        lp.n = n;
        lp.A = A;
        lp.reflag_c = j.bcrp ? 1 : 0;
        lp.has_guard = 1;
        lp.max_supersteps = guard;
        lp.round_limit = stepped ? 1 : INT64_MAX;
        lp.splits_cap = splits_dev_cap;
        lp.off = off;
        lp.rev_ptr = rev_ptr;
        lp.rev_slot = rev_slot;
        lp.block = block;
        lp.nl = nl;
        lp.mark = mark;
        lp.unstable = U;
        lp.split_list = split_list;
        lp.cmem = cmem;
        lp.splits = splits;
        lp.ctrl = ctrl;
    } else {
        // members grouped by block: counting sort of states by label
        MemberRec* members = (MemberRec*)c.members.ensure((int64_t)n * sizeof(MemberRec));
        int32_t* bstart = (int32_t*)c.bstart.ensure(((int64_t)n + 1) * 4);
        int32_t* bsize = (int32_t*)c.bsize.ensure((int64_t)n * 4);
        CK(cudaMemsetAsync(bstart, 0, ((int64_t)n + 1) * 4, st));
        const int ggrid = std::max(1, std::min(c.sms * 4, (int)((n + kGroupThreads - 1) / kGroupThreads)));
        k_group_states<false><<<ggrid, kGroupThreads, 0, st>>>(n, block, bstart, nullptr, nullptr, nullptr);
        ++c.launches;
        CK(cudaMemcpyAsync(bsize, bstart, (int64_t)n * 4, cudaMemcpyDeviceToDevice, st));
        scan_excl(c, bstart, n);
        CK(cudaMemcpyAsync(cursor, bstart, (int64_t)n * 4, cudaMemcpyDeviceToDevice, st));
        int2* brange = (int2*)c.brange.ensure((int64_t)n * 8);
        k_pack_ranges<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, bstart, bsize, brange);
        ++c.launches;
        k_group_states<true><<<ggrid, kGroupThreads, 0, st>>>(n, block, cursor, j.bcrp ? off : nullptr, rev_ptr,
                                                             members);
        ++c.launches;
        uint32_t* U1 = U + nw0;
        uint32_t* U2 = U1 + nw1 + 1;
        k_summary<<<grid_for((int64_t)nw1 * 32, TB, c.sms), TB, 0, st>>>(U, nw0, U1, nw1);
        k_summary<<<1, 64, 0, st>>>(U1, nw1, U2, nw2);
        c.launches += 2;
        uint32_t* tblock = (uint32_t*)c.tblock.ensure(parities * (nwords + 2) * 4);
        CK(cudaMemsetAsync(tblock, 0, parities * (nwords + 2) * 4, st));
        sp.n = n;
        sp.A = A;
        sp.reflag_c = j.bcrp ? 1 : 0;
        sp.has_guard = 1;
        sp.max_supersteps = guard;
        sp.round_limit = stepped ? 1 : INT64_MAX;
        sp.splits_cap = splits_dev_cap;
        sp.off = off;
        sp.rev_ptr = rev_ptr;
        sp.rev = rev2;
        sp.rev_src = rev_src;
        sp.block = block;
        sp.members = members;
        sp.brange = brange;
        sp.mark = mark;
        sp.tblock = tblock;
        sp.U0 = U;
        sp.U1 = U1;
        sp.U2 = U2;
        sp.nw0 = nw0;
        sp.nw1 = nw1;
        sp.nw2 = nw2;
        sp.small_list = (int4*)c.small_list.ensure((int64_t)n * 16);
        sp.big_list = (int4*)c.big_list.ensure(((int64_t)n / 32 + 2) * 16);
        sp.big_base = (int32_t*)c.big_base.ensure(((int64_t)n / 32 + 2) * 4);
        sp.big_list4 = (int4*)c.big_list4.ensure(((int64_t)n / 32 + 2) * 16);
        sp.big_base4 = (int32_t*)c.big_base4.ensure(((int64_t)n / 32 + 2) * 4);
        sp.big_info = (int2*)c.big_info.ensure(((int64_t)n / 32 + 2) * 8);
        sp.big_info4 = (int2*)c.big_info4.ensure(((int64_t)n / 32 + 2) * 8);
        // chunk-major two-pass records: at most n / 128 + (blocks of > 32
        // members < n / 32) chunks of 32 * kWide members
        sp.tmp = (MemberRec*)c.tmp.ensure(((int64_t)n / (32 * kWide) + (int64_t)n / 32 + 2) * 32 * kWide *
                                          (int64_t)sizeof(MemberRec));
        sp.srec = (SplitRec*)c.sarr.ensure((int64_t)n * sizeof(SplitRec));
        sp.scnt = (int32_t*)c.scnt.ensure((int64_t)n * 4);
        sp.kcur = (int32_t*)c.kcur.ensure((int64_t)n * 4);
        sp.scur = (int32_t*)c.scur.ensure((int64_t)n * 4);
        sp.splits = splits;
        sp.ctrl = (SCtrl*)ctrl;
        sp.bar = (GridBarrier*)c.bar.ensure(sizeof(GridBarrier));
        // schedule variants (bisim.h BISIM_FLAG_*); none changes a result
        sp.allow_skip = (j.opt.flags & BISIM_FLAG_NO_SKIP) ? 0 : 1;
        sp.cta_minor = (j.opt.flags & BISIM_FLAG_CTA_MAJOR) ? 0 : 1;
        sp.allow_solo = (j.opt.flags & BISIM_FLAG_NO_SOLO) ? 0 : 1;
        // developer: BISIM_MODE_B=1|2 forces the wide / two-pass phase-B layout
        sp.force_mode_b = dev_env("BISIM_MODE_B") ? atoi(dev_env("BISIM_MODE_B")) : -1;
        if (j.opt.flags & BISIM_FLAG_WIDE_LAYOUT) sp.force_mode_b = std::max(sp.force_mode_b, 1);
        if (j.opt.flags & BISIM_FLAG_TWO_PASS) sp.force_mode_b = 2;
        sp.batch_min_c = dev_env("BISIM_BATCH_C") ? atoi(dev_env("BISIM_BATCH_C")) : 8192;
        if (j.opt.flags & BISIM_FLAG_BATCH_WALK) sp.batch_min_c = 1;
        sp.onepass_major = dev_env("BISIM_ONEPASS_MINOR") != nullptr ? 0
                           : dev_env("BISIM_MAJOR") ? atoi(dev_env("BISIM_MAJOR")) : kSparseThreads / 32;
        sp.wide_major = dev_env("BISIM_WIDE_MAJOR") ? atoi(dev_env("BISIM_WIDE_MAJOR")) : 0;
        sp.prefetch_next = dev_env("BISIM_PREFETCH") ? atoi(dev_env("BISIM_PREFETCH")) : 2;
        // one-pass wide layout above 512 chunks of 32 per big block (A/B: 32 -> c5 +9 %, 128 -> neutral)
        sp.wide_min = dev_env("BISIM_WIDE_MIN") ? atoi(dev_env("BISIM_WIDE_MIN")) : 512;
        sp.solo_max_c = dev_env("BISIM_SOLO_C") ? atoi(dev_env("BISIM_SOLO_C")) : kSoloMaxC;
        sp.solo_max_items = dev_env("BISIM_SOLO_ITEMS") ? atoi(dev_env("BISIM_SOLO_ITEMS")) : kSoloMaxItems;
        // developer tracing: BISIM_TRACE=<rounds> BISIM_TRACE_FILE=<path>
        if (const char* tr = dev_env("BISIM_TRACE")) {
            sp.trace_rounds = atoll(tr);
            sp.trace = (unsigned long long*)c.trace.ensure(sp.trace_rounds * 8 * kTraceWords + 64);
            CK(cudaMemsetAsync(sp.trace, 0, sp.trace_rounds * 8 * kTraceWords, st));
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c.ev[3], st));
    CK(cudaStreamSynchronize(st));
    S.initial_blocks = h_leaders;
    if (sharded) {
        ShardPrep& P = *j.prep;
        sp.mark_stride = mark_words;
        sp.bm_stride = nwords + 2;
        sp.allow_skip = 0;  // skip steps read in-edges of other shards
        sp.allow_solo = 0;
        P.sp = sp;
        P.S = S;
        P.guard = guard;
        P.splits_dev_cap = splits_dev_cap;
        P.block = block;
        P.splits = splits;
        P.leaders = leaders;
        P.mark_words = mark_words;
        P.bm_words = nwords + 2;
        S.t_h2d_ms = elapsed(c.ev[0], c.ev[1]);
        S.t_pre_ms = elapsed(c.ev[1], c.ev[2]);
        S.t_label_ms = elapsed(c.ev[2], c.ev[3]);
        P.S = S;
        return BISIM_OK;
    }

    // ---- refinement loop
    const void* kfn;
    int kgrid, kthreads = kThreads;
    void* kargs[1];
    if (dense) {
        kfn = j.bcrp ? (const void*)k_refine<false> : (const void*)k_refine<true>;
        kgrid = j.bcrp ? c.grid_refine_bcrp : c.grid_refine_rcpp;
        kargs[0] = &lp;
    } else {
        kfn = j.bcrp ? (const void*)k_refine_sparse<false, false> : (const void*)k_refine_sparse<true, false>;
        kgrid = j.bcrp ? c.grid_sparse_bcrp : c.grid_sparse_rcpp;
        // developer: BISIM_SPARSE_GRID=<CTAs> (at most the resident grid)
        if (const char* g = dev_env("BISIM_SPARSE_GRID")) kgrid = std::max(1, std::min(kgrid, atoi(g)));
        kthreads = kSparseThreads;
        kargs[0] = &sp;
    }
    auto status = [&]() {
        LoopStatus ls;
        if (dense) {
            Ctrl h;
            CK(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ls.round = h.round; ls.done = h.done; ls.error = h.error; ls.guard_count = h.guard_count;
            ls.work_edges = h.work_edges; ls.work_splits = h.work_splits;
        } else {
            SCtrl h;
            CK(cudaMemcpyAsync(&h, ctrl, sizeof(SCtrl), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ls.round = h.round; ls.done = h.done; ls.error = h.error; ls.guard_count = h.guard_count;
            ls.work_edges = h.work_edges; ls.work_members = h.work_members; ls.retired = h.skipped_rounds;
        }
        return ls;
    };
    std::vector<int32_t> host_block;
    int64_t rounds = 0;
    int rc = BISIM_OK;
    for (;;) {
        if (dense) {
            k_ctrl_reset<<<1, 1, 0, st>>>(ctrl);
            ++c.launches;
        }
        if (!dense) CK(cudaMemsetAsync(sp.bar, 0, sizeof(GridBarrier), st));
        CK(cudaLaunchCooperativeKernel(kfn, kgrid, kthreads, kargs, 0, st));
        ++c.launches;
        if (!stepped) break;
        LoopStatus ls = status();
        if (ls.error || ls.done) break;
        if (ls.round > rounds) {
            rounds = ls.round;
            if (j.opt.observer) {
                host_block.resize(n);
                CK(cudaMemcpyAsync(host_block.data(), block, (int64_t)n * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (j.opt.observer(rounds, host_block.data(), n, j.opt.observer_user) != 0) {
                    rc = BISIM_ABORTED;
                    break;
                }
            }
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(c.ev[4], st));
    LoopStatus ls = status();
    S.supersteps = ls.round;
    if (rc == BISIM_ABORTED) {
        *j.st = S;
        throw Error(BISIM_ABORTED, "observer aborted the run");
    }
    if (ls.error == BISIM_GUARD) {
        S.guard_count = ls.guard_count;
        *j.st = S;
        throw Error(BISIM_GUARD, "superstep guard exceeded (" + std::to_string(ls.guard_count) + " > " +
                                     std::to_string(guard) + ")");
    }

    // ---- results
    CK(cudaMemsetAsync(leaders, 0, 4, st));
    k_count_leaders<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, block, leaders);
    ++c.launches;
    if (j.block_out_on_device)
        CK(cudaMemcpyAsync(j.block_out, block, (int64_t)n * 4, cudaMemcpyDeviceToDevice, st));
    else
        d2h(c, j.block_out, block, (int64_t)n * 4, st);
    const int64_t R = ls.round;
    const int64_t ncopy = std::min<int64_t>(std::min<int64_t>(R, j.splits_cap), splits_dev_cap);
    if (j.splits_out && ncopy > 0)
        CK(cudaMemcpyAsync(j.splits_out, splits, ncopy * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h_leaders, leaders, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(c.ev[5], st));
    CK(cudaStreamSynchronize(st));
    S.final_blocks = h_leaders;
    S.t_h2d_ms = elapsed(c.ev[0], c.ev[1]);
    S.t_pre_ms = elapsed(c.ev[1], c.ev[2]);
    S.t_label_ms = elapsed(c.ev[2], c.ev[3]);
    S.t_alg_ms = elapsed(c.ev[3], c.ev[4]);
    S.t_d2h_ms = elapsed(c.ev[4], c.ev[5]);
    S.bytes_alg = loop_bytes(j.bcrp, dense, n, L32, R, ls);
    if (!dense && sp.trace) {
        std::vector<unsigned long long> t(sp.trace_rounds * kTraceWords);
        CK(cudaMemcpy(t.data(), sp.trace, t.size() * 8, cudaMemcpyDeviceToHost));
        const char* path = dev_env("BISIM_TRACE_FILE");
        if (FILE* f = fopen(path ? path : "bisim_trace.csv", "w")) {
            fprintf(f, "round,phaseA_ns,barrierA_ns,phaseB_ns,csize,solo,n_small,big_chunks,n_big,"
                       "b_tag_ns,b_sync1_ns,b_arrive_ns,b_sync2_ns,b_place_ns,mode_b,a_walk0_ns,a_walkcta_ns,a_wave_ns\n");
            for (int64_t r = 0; r < std::min<int64_t>(sp.trace_rounds, R); ++r) {
                const unsigned long long* q = &t[r * kTraceWords];
                auto d = [&](int a, int b) -> long long { return (q[a] && q[b]) ? (long long)(q[a] - q[b]) : -1; };
                fprintf(f, "%lld,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%lld,%lld,%lld,%lld,%lld,%llu,%lld,%lld,%lld\n",
                        (long long)r, q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4], q[5], q[6],
                        q[7] & 0xffffffffull, q[7] >> 32, d(8, 2), d(9, 8), d(10, 9), d(11, 10), d(12, 11),
                        q[13], d(14, 0), d(15, 14), d(1, 15));
            }
            fclose(f);
        }
    }
    S.kernel_launches = c.launches;
    S.rounds_retired = (int64_t)ls.retired;
    *j.st = S;
    return BISIM_OK;
}

// ---- transition-sharded mode (kernels_shard.cuh) ------------------------------

// Per-shard resources, cached across calls with the same device list.
struct ShardSet {
    std::vector<int32_t> devices;
    std::vector<std::unique_ptr<Ctx>> ctx;
    std::vector<DevBuf> xlist, xcnt, xbar, go;
};
std::mutex g_shard_mu;
std::unique_ptr<ShardSet> g_shards;

ShardSet& shard_set(const int32_t* devices, int G) {
    std::vector<int32_t> want(devices, devices + G);
    if (!g_shards || g_shards->devices != want) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw Error(BISIM_CUDA, "no CUDA device available (libbisim has no CPU fallback)");
        auto S = std::make_unique<ShardSet>();
        S->devices = want;
        for (int g = 0; g < G; ++g) {
            if (want[g] < 0 || want[g] >= count) throw Error(BISIM_CUDA, "invalid CUDA device ordinal");
            S->ctx.push_back(make_ctx(want[g]));
        }
        S->xlist.resize(G);
        S->xcnt.resize(G);
        S->xbar.resize(G);
        S->go.resize(G);
        // peer access between distinct devices (NVLink / NVSwitch)
        for (int a = 0; a < G; ++a)
            for (int b = 0; b < G; ++b) {
                if (want[a] == want[b]) continue;
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, want[a], want[b]));
                if (!ok) throw Error(BISIM_CUDA, "devices cannot access each other's memory (no P2P)");
                CK(cudaSetDevice(want[a]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(want[b], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
        g_shards = std::move(S);
    }
    return *g_shards;
}

// Source ranges with about m / G transitions each (out-degree prefix sums on
// the first shard's device).
std::vector<int32_t> shard_bounds(Ctx& c, int32_t n, int64_t m, const int32_t* d_src, int G) {
    std::vector<int32_t> lo(G + 1, n);
    lo[0] = 0;
    if (m == 0) {
        for (int g = 1; g < G; ++g) lo[g] = (int32_t)((int64_t)n * g / G);
        return lo;
    }
    // validate src before scattering through it (the replicas check the rest)
    Ctrl* ctrl = (Ctrl*)c.ctrl.ensure(std::max(sizeof(Ctrl), sizeof(SCtrl)));
    CK(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), c.stream));
    k_check_edges<<<grid_for(m, 256, c.sms), 256, 0, c.stream>>>(n, m, d_src, d_src, ctrl);
    int32_t bad = 0;
    CK(cudaMemcpyAsync(&bad, &ctrl->bad, sizeof(bad), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (bad) throw Error(BISIM_BAD_INPUT, "transition mentions a state outside range");
    int32_t* deg = (int32_t*)c.cursor.ensure(((int64_t)n + 1) * 4);
    CK(cudaMemsetAsync(deg, 0, ((int64_t)n + 1) * 4, c.stream));
    k_indeg<<<grid_for(m, 256, c.sms), 256, 0, c.stream>>>(m, d_src, deg);
    scan_excl(c, deg, n);
    int32_t* dlo = (int32_t*)c.counter.ensure(4 * (kMaxShards + 2));
    k_shard_cuts<<<1, 32, 0, c.stream>>>(deg, n, G, dlo);
    CK(cudaMemcpyAsync(lo.data(), dlo, 4 * (G + 1), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return lo;
}

int run_sharded(Job& base, const int32_t* devices, int G, int32_t flags) {
    if (G < 1 || G > kMaxShards) throw Error(BISIM_BAD_INPUT, "shard count must be 1..8");
    if (!devices) throw Error(BISIM_BAD_INPUT, "null device list");
    if (base.n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
    std::lock_guard<std::mutex> lock(g_shard_mu);
    ShardSet& S = shard_set(devices, G);
    const int32_t n = base.n;
    const int64_t m = base.m;
    // shard bounds: copy src to shard 0 once to find them
    Ctx& c0 = *S.ctx[0];
    CK(cudaSetDevice(c0.device));
    std::vector<int32_t> lo;
    {
        const int64_t mm = std::max<int64_t>(m, 1);
        int32_t* d_src = (int32_t*)c0.src.ensure(mm * 4);
        h2d(c0, d_src, base.src, m * 4, c0.stream);
        lo = shard_bounds(c0, n, m, d_src, G);
    }
    // every replica: inputs, preprocessing, label partition, loop state
    std::vector<ShardPrep> prep(G);
    for (int g = 0; g < G; ++g) {
        Ctx& c = *S.ctx[g];
        Job j = base;
        j.prep = &prep[g];
        j.src_lo = lo[g];
        j.src_hi = lo[g + 1];
        j.opt.device = c.device;
        bisim_stats st{};
        j.st = &st;
        run_with(c, j);
    }
    for (int g = 0; g < G; ++g) {
        Ctx& c = *S.ctx[g];
        CK(cudaSetDevice(c.device));
        int32_t* xl = (int32_t*)S.xlist[g].ensure(2 * (int64_t)n * 4);
        (void)xl;
        CK(cudaMemsetAsync(S.xcnt[g].ensure(16), 0, 16, c.stream));
        CK(cudaMemsetAsync(S.xbar[g].ensure(128), 0, 128, c.stream));
        CK(cudaMemsetAsync(S.go[g].ensure(128), 0, 128, c.stream));
        CK(cudaMemsetAsync(prep[g].sp.bar, 0, sizeof(GridBarrier), c.stream));
    }
    for (int g = 0; g < G; ++g) {
        SparseParams& sp = prep[g].sp;
        sp.nshard = G;
        sp.shard = g;
        sp.xlist = (int32_t*)S.xlist[g].p;
        sp.go = (unsigned*)S.go[g].p;
        sp.timeout_ns = 20ull * 1000 * 1000 * 1000;
        for (int r = 0; r < G; ++r) {
            sp.peer_mark[r] = prep[r].sp.mark;
            sp.peer_xlist[r] = (int32_t*)S.xlist[r].p;
            sp.peer_xcnt[r] = (int32_t*)S.xcnt[r].p;
            sp.peer_xbar[r] = (unsigned*)S.xbar[r].p;
        }
    }
    for (int g = 0; g < G; ++g) CK(cudaStreamSynchronize(S.ctx[g]->stream));
    // launch every replica; a device holding several replicas (testing on
    // one GPU) splits its SMs between them and uses plain launches
    std::vector<cudaEvent_t> t0(G), t1(G);
    for (int g = 0; g < G; ++g) {
        Ctx& c = *S.ctx[g];
        CK(cudaSetDevice(c.device));
        const int same = (int)std::count(S.devices.begin(), S.devices.end(), c.device);
        const void* kfn = base.bcrp ? (const void*)k_refine_sparse<false, true> : (const void*)k_refine_sparse<true, true>;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kSparseThreads, 0));
        if (occ < 1) throw Error(BISIM_CUDA, "sharded kernel cannot be resident");
        t0[g] = c.ev[3];
        t1[g] = c.ev[4];
        CK(cudaEventRecord(t0[g], c.stream));
        void* args[] = {&prep[g].sp};
        if (same == 1) {
            CK(cudaLaunchCooperativeKernel(kfn, c.sms, kSparseThreads, args, 0, c.stream));
        } else {
            const int grid = std::max(1, c.sms / same);
            CK(cudaLaunchKernel(kfn, grid, kSparseThreads, args, 0, c.stream));
        }
        CK(cudaEventRecord(t1[g], c.stream));
        ++c.launches;
    }
    std::vector<SCtrl> hc(G);
    for (int g = 0; g < G; ++g) {
        Ctx& c = *S.ctx[g];
        CK(cudaSetDevice(c.device));
        CK(cudaMemcpyAsync(&hc[g], prep[g].sp.ctrl, sizeof(SCtrl), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    }
    for (int g = 0; g < G; ++g) {
        if (hc[g].error == kShardTimeout)
            throw Error(BISIM_CUDA, "sharded replicas did not run concurrently (cross-replica wait timed out)");
        if (hc[g].round != hc[0].round || hc[g].error != hc[0].error)
            throw Error(BISIM_CUDA, "sharded replicas diverged");
    }
    ShardPrep& P = prep[0];
    bisim_stats St = P.S;
    St.supersteps = hc[0].round;
    St.mode = BISIM_MODE_PERSISTENT;
    if (hc[0].error == BISIM_GUARD) {
        St.guard_count = hc[0].guard_count;
        if (base.st) *base.st = St;
        throw Error(BISIM_GUARD, "superstep guard exceeded (" + std::to_string(hc[0].guard_count) + " > " +
                                     std::to_string(P.guard) + ")");
    }
    float alg = 0.f;
    for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(S.ctx[g]->device));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, t0[g], t1[g]));
        alg = std::max(alg, ms);
    }
    // results from replica 0 (optionally checked against every replica)
    CK(cudaSetDevice(c0.device));
    CK(cudaMemsetAsync(P.leaders, 0, 4, c0.stream));
    k_count_leaders<<<grid_for(n, 256, c0.sms), 256, 0, c0.stream>>>(n, P.block, P.leaders);
    CK(cudaMemcpyAsync(base.block_out, P.block, (int64_t)n * 4, cudaMemcpyDeviceToHost, c0.stream));
    const int64_t R = hc[0].round;
    const int64_t ncopy = std::min<int64_t>(std::min<int64_t>(R, base.splits_cap), P.splits_dev_cap);
    if (base.splits_out && ncopy > 0)
        CK(cudaMemcpyAsync(base.splits_out, P.splits, ncopy * 4, cudaMemcpyDeviceToHost, c0.stream));
    int32_t fin = 0;
    CK(cudaMemcpyAsync(&fin, P.leaders, 4, cudaMemcpyDeviceToHost, c0.stream));
    CK(cudaStreamSynchronize(c0.stream));
    if (flags & BISIM_SHARD_VERIFY) {
        std::vector<int32_t> other(n);
        for (int g = 1; g < G; ++g) {
            CK(cudaSetDevice(S.ctx[g]->device));
            CK(cudaMemcpy(other.data(), prep[g].block, (int64_t)n * 4, cudaMemcpyDeviceToHost));
            if (memcmp(other.data(), base.block_out, (size_t)n * 4) != 0)
                throw Error(BISIM_CUDA, "sharded replicas hold different partitions");
        }
    }
    St.final_blocks = fin;
    St.t_alg_ms = alg;
    LoopStatus ls;
    for (int g = 0; g < G; ++g) {
        ls.work_edges += hc[g].work_edges;
        ls.work_members = std::max(ls.work_members, hc[g].work_members);
    }
    ls.round = R;
    St.bytes_alg = loop_bytes(base.bcrp, false, n, St.mark_length, R, ls);
    St.kernel_launches = G;
    if (base.st) *base.st = St;
    return BISIM_OK;
}

int guarded(Job& j) {
    bisim_stats dummy{};
    if (!j.st) j.st = &dummy;
    try {
        g_last_error.clear();
        return run(j);
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BISIM_CUDA;
    }
}

int sharded_guarded(Job& j, const int32_t* devices, int G, int32_t flags) {
    bisim_stats dummy{};
    if (!j.st) j.st = &dummy;
    try {
        g_last_error.clear();
        if (j.n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
        if (j.m < 0 || j.m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
        if (j.m > 0 && (!j.src || !j.dst || (j.bcrp && !j.act)))
            throw Error(BISIM_BAD_INPUT, "null transition array");
        if (!j.block_out) throw Error(BISIM_BAD_INPUT, "null block_out");
        return run_sharded(j, devices, G, flags);
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BISIM_CUDA;
    }
}

bisim_options opts_or_default(const bisim_options* o, int device) {
    bisim_options r{};
    if (o) r = *o;
    else r.device = device;
    return r;
}

}  // namespace
}  // namespace bisim

namespace bisim {
// used by aut.cpp (host-only translation unit)
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace bisim

using namespace bisim;

extern "C" {

int bisim_bcrp_ex(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                  const int32_t* dst, int64_t max_supersteps, int32_t* block_out, int32_t* splits_out,
                  int64_t splits_cap, bisim_stats* st, const bisim_options* opt) {
    Job j;
    j.bcrp = true;
    j.n = n;
    j.m = m;
    j.A = num_actions;
    j.src = src;
    j.act = act;
    j.dst = dst;
    j.max_supersteps = max_supersteps;
    j.block_out = block_out;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    j.opt = opts_or_default(opt, 0);
    return guarded(j);
}

int bisim_bcrp(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
               const int32_t* dst, int64_t max_supersteps, int32_t* block_out, int32_t* splits_out,
               int64_t splits_cap, bisim_stats* st, int device) {
    bisim_options o{};
    o.device = device;
    return bisim_bcrp_ex(n, m, num_actions, src, act, dst, max_supersteps, block_out, splits_out, splits_cap,
                         st, &o);
}

int bisim_rcpp_ex(int32_t n, int64_t m, const int32_t* src, const int32_t* dst, const int32_t* pi0_leader,
                  int64_t max_supersteps, int32_t* block_out, int32_t* splits_out, int64_t splits_cap,
                  bisim_stats* st, const bisim_options* opt) {
    Job j;
    j.bcrp = false;
    j.n = n;
    j.m = m;
    j.src = src;
    j.dst = dst;
    j.pi0 = pi0_leader;
    j.max_supersteps = max_supersteps;
    j.block_out = block_out;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    j.opt = opts_or_default(opt, 0);
    return guarded(j);
}

int bisim_rcpp(int32_t n, int64_t m, const int32_t* src, const int32_t* dst, const int32_t* pi0_leader,
               int64_t max_supersteps, int32_t* block_out, int32_t* splits_out, int64_t splits_cap,
               bisim_stats* st, int device) {
    bisim_options o{};
    o.device = device;
    return bisim_rcpp_ex(n, m, src, dst, pi0_leader, max_supersteps, block_out, splits_out, splits_cap, st,
                         &o);
}

int bisim_bcrp_device(int32_t n, int64_t m, int32_t num_actions, const int32_t* d_src, const int32_t* d_act,
                      const int32_t* d_dst, int64_t max_supersteps, int32_t* d_block_out, int32_t* splits_out,
                      int64_t splits_cap, bisim_stats* st, const bisim_options* opt) {
    Job j;
    j.bcrp = true;
    j.n = n;
    j.m = m;
    j.A = num_actions;
    j.src = d_src;
    j.act = d_act;
    j.dst = d_dst;
    j.inputs_on_device = true;
    j.max_supersteps = max_supersteps;
    j.block_out = d_block_out;
    j.block_out_on_device = true;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    j.opt = opts_or_default(opt, 0);
    return guarded(j);
}

int bisim_rcpp_device(int32_t n, int64_t m, const int32_t* d_src, const int32_t* d_dst,
                      const int32_t* d_pi0_leader, int64_t max_supersteps, int32_t* d_block_out,
                      int32_t* splits_out, int64_t splits_cap, bisim_stats* st, const bisim_options* opt) {
    Job j;
    j.bcrp = false;
    j.n = n;
    j.m = m;
    j.src = d_src;
    j.dst = d_dst;
    j.pi0 = d_pi0_leader;
    j.inputs_on_device = true;
    j.max_supersteps = max_supersteps;
    j.block_out = d_block_out;
    j.block_out_on_device = true;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    j.opt = opts_or_default(opt, 0);
    return guarded(j);
}

int bisim_bcrp_sharded(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                       const int32_t* dst, int64_t max_supersteps, int32_t* block_out, int32_t* splits_out,
                       int64_t splits_cap, bisim_stats* st, const int32_t* devices, int32_t nshards,
                       int32_t flags) {
    Job j;
    j.bcrp = true;
    j.n = n;
    j.m = m;
    j.A = num_actions;
    j.src = src;
    j.act = act;
    j.dst = dst;
    j.max_supersteps = max_supersteps;
    j.block_out = block_out;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    return sharded_guarded(j, devices, nshards, flags);
}

int bisim_rcpp_sharded(int32_t n, int64_t m, const int32_t* src, const int32_t* dst, const int32_t* pi0_leader,
                       int64_t max_supersteps, int32_t* block_out, int32_t* splits_out, int64_t splits_cap,
                       bisim_stats* st, const int32_t* devices, int32_t nshards, int32_t flags) {
    Job j;
    j.bcrp = false;
    j.n = n;
    j.m = m;
    j.src = src;
    j.dst = dst;
    j.pi0 = pi0_leader;
    j.max_supersteps = max_supersteps;
    j.block_out = block_out;
    j.splits_out = splits_out;
    j.splits_cap = splits_cap;
    j.st = st;
    return sharded_guarded(j, devices, nshards, flags);
}

int bisim_preprocess(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                     int32_t* order_out, int32_t* nr_marks_out, int32_t* off_out, int64_t* mark_length,
                     int device) {
    return guarded_call([&]() {
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        LabelTables t = label_tables(c, n, m, num_actions, src, act);
        cudaStream_t st = c.stream;
        const int TB = 256;
        int32_t* d_order = (int32_t*)c.rev_slot.ensure(std::max<int64_t>(m, 1) * 4);
        if (m) k_order<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, t.src, t.act, t.lmask, d_order);
        CK(cudaGetLastError());
        if (nr_marks_out) CK(cudaMemcpyAsync(nr_marks_out, t.nr, (int64_t)n * 4, cudaMemcpyDeviceToHost, st));
        if (off_out) CK(cudaMemcpyAsync(off_out, t.off, (int64_t)n * 4, cudaMemcpyDeviceToHost, st));
        if (order_out && m) CK(cudaMemcpyAsync(order_out, d_order, m * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (mark_length) *mark_length = t.L;
    });
}

int bisim_preprocess_sorted(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                            const int32_t* dst, int32_t* perm_out, int32_t* src_out, int32_t* act_out,
                            int32_t* dst_out, int32_t* action_switch_out, int32_t* order_out,
                            int32_t* nr_marks_out, int32_t* off_out, int64_t* mark_length, int device) {
    return guarded_call([&]() {
        if (m > 0 && !dst && dst_out) throw Error(BISIM_BAD_INPUT, "null dst with dst_out");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        LabelTables t = label_tables(c, n, m, num_actions, src, act, m ? dst : nullptr);
        cudaStream_t st = c.stream;
        const int TB = 256;
        const int64_t mm = std::max<int64_t>(m, 1);
        // stable sort by (source, action): radix sort of the key
        // source * |Act| + action carrying the transition index (bcrp.py:49-52)
        auto* keys = (unsigned long long*)c.lkeys.ensure(mm * 8 * 2);
        unsigned long long* keys_sorted = keys + mm;
        int32_t* idx = (int32_t*)c.cursor.ensure(mm * 4 * 2);
        int32_t* perm = idx + mm;
        if (m) {
            k_sort_keys<<<grid_for(m, TB, c.sms), TB, 0, st>>>(m, num_actions, t.src, t.act, keys, idx);
            const unsigned long long maxkey = (unsigned long long)n * (unsigned long long)std::max(num_actions, 1);
            int bits = 1;
            while (bits < 64 && (1ull << bits) < maxkey) ++bits;
            size_t tmp_bytes = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_sorted, idx, perm, (int)m, 0, bits,
                                               st));
            void* tmp = c.scan_tmp.ensure(tmp_bytes);
            CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_sorted, idx, perm, (int)m, 0, bits, st));
            c.launches += 2;
        }
        // per sorted transition: columns, action_switch (bcrp.py:55-65), order
        int32_t* cols = (int32_t*)c.rev2.ensure(mm * 4 * 5);
        int32_t *s_src = cols, *s_act = cols + mm, *s_dst = cols + 2 * mm, *s_sw = cols + 3 * mm,
                *s_ord = cols + 4 * mm;
        const int32_t* d_dst = t.dst;
        if (m)
            k_sorted_tables<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, perm, t.src, t.act, d_dst, t.lmask, s_src,
                                                                   s_act, s_dst, s_sw, s_ord);
        CK(cudaGetLastError());
        auto d2h = [&](int32_t* out, const int32_t* d, int64_t cnt) {
            if (out && cnt) CK(cudaMemcpyAsync(out, d, cnt * 4, cudaMemcpyDeviceToHost, st));
        };
        d2h(perm_out, perm, m);
        d2h(src_out, s_src, m);
        d2h(act_out, s_act, m);
        if (d_dst) d2h(dst_out, s_dst, m);
        d2h(action_switch_out, s_sw, m);
        d2h(order_out, s_ord, m);
        d2h(nr_marks_out, t.nr, n);
        d2h(off_out, t.off, n);
        CK(cudaStreamSynchronize(st));
        if (mark_length) *mark_length = t.L;
    });
}

int bisim_label_partition(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                          int32_t* block_out, int device) {
    return guarded_call([&]() {
        if (!block_out) throw Error(BISIM_BAD_INPUT, "null block_out");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        LabelTables t = label_tables(c, n, m, num_actions, src, act);
        int32_t* block = (int32_t*)c.block.ensure((int64_t)n * 4);
        label_partition_dev(c, n, num_actions, t.lmask, block, false);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(block_out, block, (int64_t)n * 4, cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int bisim_label_rounds_common(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                              int32_t* conflict_round, int32_t* conflict_leader, int32_t* conflict_winner,
                              int32_t* block_out, int device) {
    return guarded_call([&]() {
        if (!block_out || !conflict_round || !conflict_leader || !conflict_winner)
            throw Error(BISIM_BAD_INPUT, "null output");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        LabelTables t = label_tables(c, n, m, num_actions, src, act);
        cudaStream_t st = c.stream;
        int32_t* block = (int32_t*)c.block.ensure((int64_t)n * 4);
        auto* nl = (unsigned long long*)c.nl.ensure((int64_t)n * 8);
        int32_t* moved = (int32_t*)c.bsize.ensure((int64_t)n * 4);
        int32_t* conf = (int32_t*)c.counter.ensure(16);
        auto* conf_key = (unsigned long long*)c.sarr.ensure(8);
        CK(cudaMemsetAsync(block, 0, (int64_t)n * 4, st));
        CK(cudaMemsetAsync(nl, 0, (int64_t)n * 8, st));
        CK(cudaMemsetAsync(moved, 0, (int64_t)n * 4, st));
        CK(cudaMemsetAsync(conf, 0x7f, 4, st));
        CK(cudaMemsetAsync(conf_key, 0xff, 8, st));
        if (num_actions > 0) {
            int32_t nn = n, AA = num_actions;
            const unsigned long long* lm = t.lmask;
            void* args[] = {&nn, &AA, (void*)&lm, &block, &nl, &moved, &conf, &conf_key};
            CK(cudaLaunchCooperativeKernel((const void*)k_label_rounds_common, c.grid_label_common, kThreads, args, 0,
                                           st));
        }
        int32_t h_conf = 0;
        unsigned long long h_key = 0;
        CK(cudaMemcpyAsync(&h_conf, conf, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&h_key, conf_key, 8, cudaMemcpyDeviceToHost, st));
        d2h(c, block_out, block, (int64_t)n * 4, st);
        CK(cudaStreamSynchronize(st));
        const bool hit = h_conf != 0x7f7f7f7f;
        *conflict_round = hit ? h_conf : -1;
        *conflict_winner = hit ? (int32_t)(h_key >> 32) : -1;
        *conflict_leader = hit ? (int32_t)(h_key & 0xffffffffu) : -1;
    });
}

const char* bisim_last_error(void) { return g_last_error.c_str(); }

int bisim_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

void* bisim_stream(int device) {
    try {
        return (void*)get_ctx(device)->stream;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return nullptr;
    }
}

const char* bisim_version(void) { return "libbisim 0.2 (sm_100a: work-efficient persistent refinement loop, sharded replicas, GPU quotient/stability, C++ .aut reader)"; }

}  // extern "C"

#include "post.cuh"
