// Error state, launch accounting and kernel timing for the C ABI.
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "sc_common.cuh"

namespace sc {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? SC_ERR_NO_MEMORY : SC_ERR_CUDA;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaStream_t& tl_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}

void ensure_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        // keep freed blocks cached (per-step temporaries must not re-map
        // memory after every synchronisation); the pipeline returns the
        // cache to the driver between stages with sc_trim_pool(), so the
        // multi-GB stage buffers (candidate lists, Krylov basis) do not stay
        // reserved against PyTorch's allocator
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    (void)cudaGetLastError();
    done = true;
}

cudaError_t d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    struct Staging {
        void* p = nullptr;
        size_t cap = 0;
        ~Staging() {
            if (p) cudaFreeHost(p);
        }
    };
    static thread_local Staging sb;
    if (bytes > ((size_t)8 << 20)) {  // bulk results: the plain copy
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
        return e != cudaSuccess ? e : cudaStreamSynchronize(st);
    }
    if (bytes > sb.cap) {
        if (sb.p) cudaFreeHost(sb.p);
        sb.p = nullptr;
        sb.cap = 0;
        const size_t want = std::max<size_t>(bytes, 1 << 16);
        cudaError_t e = cudaMallocHost(&sb.p, want);
        if (e != cudaSuccess) {  // no pinned memory: the plain copy
            sb.p = nullptr;
            e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
            return e != cudaSuccess ? e : cudaStreamSynchronize(st);
        }
        sb.cap = want;
    }
    cudaError_t e = cudaMemcpyAsync(sb.p, src, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) std::memcpy(dst, sb.p, bytes);
    return e;
}

void trim_pool() {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceSynchronize();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    (void)cudaGetLastError();
}

// ---- profiling ---------------------------------------------------------------
struct ProfSlot {
    std::string name;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    double ms = 0.0;
    int64_t launches = 0;
    double work = 0.0;
};
static bool g_prof = false;
static std::mutex g_prof_mu;
static std::vector<ProfSlot> g_slots;
static thread_local int g_prof_mute = 0;
ProfMute::ProfMute() { ++g_prof_mute; }
ProfMute::~ProfMute() { --g_prof_mute; }

static int slot_of(const char* name) {
    for (size_t i = 0; i < g_slots.size(); ++i)
        if (g_slots[i].name == name) return (int)i;
    g_slots.push_back(ProfSlot{});
    g_slots.back().name = name;
    return (int)g_slots.size() - 1;
}

ProfScope::ProfScope(const char* name, cudaStream_t s, double work) {
    if (!g_prof || g_prof_mute) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    slot = slot_of(name);
    stream = s;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    g_slots[slot].pending.push_back({a, b});
    g_slots[slot].launches += 1;
    g_slots[slot].work += work;
}
ProfScope::~ProfScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_slots[slot].pending.back().second, stream);
}

static void drain(ProfSlot& s) {
    for (auto& ev : s.pending) {
        cudaEventSynchronize(ev.second);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev.first, ev.second);
        s.ms += ms;
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    s.pending.clear();
}

}  // namespace sc

using namespace sc;

extern "C" {

const char* sc_last_error(void) { return g_last_error.c_str(); }
int sc_version(void) { return 100; }
int64_t sc_launch_count(void) { return g_launches; }
void sc_trim_pool(void) { trim_pool(); }
void sc_launch_count_reset(void) { g_launches = 0; }

void sc_profile_enable(int on) { g_prof = on != 0; }
void sc_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& s : g_slots) drain(s);
    g_slots.clear();
}
int sc_profile_query(const char* name, double* ms, int64_t* launches, double* work) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& s : g_slots) {
        if (s.name == name) {
            drain(s);
            if (ms) *ms = s.ms;
            if (launches) *launches = s.launches;
            if (work) *work = s.work;
            return SC_OK;
        }
    }
    if (ms) *ms = 0.0;
    if (launches) *launches = 0;
    if (work) *work = 0.0;
    return SC_ERR_VALUE;
}

}  // extern "C"
