// Kernel launch counter and optional per-phase CUDA-event timing (spc_profile_*), used by
// bench.py to time the dominant kernel live on the stream the library launches it on.
#include "spc_internal.cuh"

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace spc {

namespace {
struct Pending {
    std::string name;
    cudaEvent_t a, b;
};
struct Acc {
    double ms = 0.0;
    int64_t n = 0;
};
struct Prof {
    std::mutex m;
    bool on = false;
    std::vector<Pending> pend;
    std::map<std::string, Acc> acc;
};
Prof& prof() {
    static Prof p;
    return p;
}
std::atomic<long long> g_launches{0};

void drain_locked(Prof& p) {
    for (auto& q : p.pend) {
        float ms = 0.f;
        if (cudaEventSynchronize(q.b) == cudaSuccess && cudaEventElapsedTime(&ms, q.a, q.b) == cudaSuccess) {
            Acc& a = p.acc[q.name];
            a.ms += ms;
            a.n += 1;
        }
        cudaEventDestroy(q.a);
        cudaEventDestroy(q.b);
    }
    p.pend.clear();
}
}  // namespace

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

PhaseScope::PhaseScope(const char* name, cudaStream_t s) : name_(name), s_(s), a_(nullptr), b_(nullptr) {
    Prof& p = prof();
    if (!p.on) return;
    if (cudaEventCreate(&a_) != cudaSuccess || cudaEventCreate(&b_) != cudaSuccess) {
        a_ = b_ = nullptr;
        return;
    }
    cudaEventRecord(a_, s_);
}

PhaseScope::~PhaseScope() {
    if (!a_) return;
    cudaEventRecord(b_, s_);
    Prof& p = prof();
    std::lock_guard<std::mutex> g(p.m);
    p.pend.push_back(Pending{name_, a_, b_});
}

}  // namespace spc

extern "C" {

spc_status_t spc_profile_enable(int on) {
    spc::Prof& p = spc::prof();
    std::lock_guard<std::mutex> g(p.m);
    p.on = on != 0;
    return SPC_OK;
}

spc_status_t spc_profile_reset(void) {
    spc::Prof& p = spc::prof();
    std::lock_guard<std::mutex> g(p.m);
    spc::drain_locked(p);
    p.acc.clear();
    return SPC_OK;
}

int spc_profile_read(char* names, size_t names_len, double* ms, int64_t* counts, int max_phases) {
    spc::Prof& p = spc::prof();
    std::lock_guard<std::mutex> g(p.m);
    spc::drain_locked(p);
    int i = 0;
    size_t used = 0;
    for (auto& kv : p.acc) {
        if (i >= max_phases) break;
        const size_t L = kv.first.size() + 1;
        if (names && used + L <= names_len) {
            memcpy(names + used, kv.first.c_str(), L);
            used += L;
        }
        if (ms) ms[i] = kv.second.ms;
        if (counts) counts[i] = kv.second.n;
        ++i;
    }
    return i;
}

int64_t spc_kernel_launches(void) { return spc::g_launches.load(); }

}  // extern "C"

namespace spc {

namespace {
constexpr int kMaxDev = 64;
int g_sms[kMaxDev];
int g_clk_khz[kMaxDev];
int cur_dev() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) d = 0;
    return d;
}
}  // namespace

int num_sms() {
    const int d = cur_dev();
    if (g_sms[d] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
        g_sms[d] = v;
    }
    return g_sms[d];
}

double sm_clock_hz() {
    const int d = cur_dev();
    if (g_clk_khz[d] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, d) != cudaSuccess || v <= 0) v = 1965000;
        g_clk_khz[d] = v;
    }
    return 1e3 * (double)g_clk_khz[d];
}

}  // namespace spc
